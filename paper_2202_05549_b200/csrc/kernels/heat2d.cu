// Stencil kernels: the 2D 5-point heat step (BASELINE configs C1/C2/C5) and the reference's
// stencil1d (proj/src/kernels.cpp:147-165).
//
// heat2d semantics (restated for the CPU oracle in oracle/ref_shim.cpp make_heat2d):
//   out[i,j] = c + a*(((up + dn) + (lf + rt)) - 4c),  a = (float)alpha,
// f32 arithmetic in exactly that order, zero padding outside [0,rows)x[0,cols). Every op is
// an explicitly rounded intrinsic (__fadd_rn/__fsub_rn/__fmul_rn), so the result is bit-exact
// against the CPU oracle (4c is exact).
//
// The kernel is HBM-bound: 8 algorithmic bytes per cell update (one f32 read, one f32 write).
// Layout of the fast path: a CTA of 256 threads owns a 1024-column strip and walks a segment
// of kSegRows rows top to bottom. Each thread owns 4 consecutive columns (one 128-bit load and
// one 128-bit streaming store per row); the vertical neighbours stay in registers as the
// window slides, the horizontal neighbours come from warp shuffles, and only two edge lanes
// per warp issue a scalar load per row. Rows are fetched kBatch at a time so every thread has
// kBatch independent 128-bit loads in flight. Input bytes are read once from HBM except the 2
// halo rows per segment (2/kSegRows extra, mostly L2 hits).
#include <cuda.h>
#include <cstdlib>
#include <mutex>

#include "../executor.hpp"
#include "common.cuh"

namespace mtb {
namespace kern {

constexpr int kThreads = 256;
constexpr int kColsPerCta = kThreads * 4;
constexpr int kSegRows = 128;
constexpr int kBatch = 4;

struct heat_args {
	const float* in;   // element (i, j) at in[(i - in_r0) * in_ld + (j - in_c0)]
	float* out;        // element (i, j) at out[(i - out_r0) * out_ld + (j - out_c0)]
	int64_t in_r0, in_c0, in_ld;
	int64_t out_r0, out_c0, out_ld;
	int64_t rows, cols; // domain (zero padding outside)
	int64_t r0, r1;     // output rows [r0, r1)
	int64_t c0, c1;     // vectorised output columns [c0, c1), (c1 - c0) % 4 == 0
	int64_t seg;        // rows per CTA segment (kSegRows, fewer for small superblocks)
	float a;
};

__device__ __forceinline__ float heat_point(float c, float up, float dn, float lf, float rt, float a) {
	const float s = __fsub_rn(__fadd_rn(__fadd_rn(up, dn), __fadd_rn(lf, rt)), __fmul_rn(4.0f, c));
	return __fadd_rn(c, __fmul_rn(a, s));
}

__device__ __forceinline__ float4 load_row4(const heat_args& p, int64_t i, int64_t j, bool active) {
	if(!active || i < 0 || i >= p.rows) return make_float4(0.f, 0.f, 0.f, 0.f);
	return __ldg(reinterpret_cast<const float4*>(p.in + (i - p.in_r0) * p.in_ld + (j - p.in_c0)));
}

__device__ __forceinline__ float load_one(const heat_args& p, int64_t i, int64_t j) {
	if(i < 0 || i >= p.rows || j < 0 || j >= p.cols) return 0.f;
	return __ldg(p.in + (i - p.in_r0) * p.in_ld + (j - p.in_c0));
}

// 4 CTAs (32 warps) per SM: <= 64 registers. Measured alternatives (B200, 65536^2): 64- or
// 256-row segments, 8-row batches (125 registers, 2 CTAs/SM: 0.74 of peak) and 5-8 CTAs/SM
// (register caps with small spills) are all equal or slower.
__global__ void __launch_bounds__(kThreads, 4) heat2d_vec_kernel(heat_args p) {
	const int lane = threadIdx.x & 31;
	const int64_t j = p.c0 + static_cast<int64_t>(blockIdx.x) * kColsPerCta + threadIdx.x * 4;
	const bool active = j < p.c1;
	// last active lane of this warp (right edge of the strip)
	const int64_t warp_j0 = j - lane * 4;
	const int64_t rem = (p.c1 - warp_j0) / 4 - 1;
	const int last_lane = rem < 31 ? static_cast<int>(rem) : 31;
	const int64_t r0 = p.r0 + static_cast<int64_t>(blockIdx.y) * p.seg;
	const int64_t r1 = p.r1 < r0 + p.seg ? p.r1 : r0 + p.seg;
	if(r0 >= r1) return;

	float4 up = load_row4(p, r0 - 1, j, active);
	float4 c = load_row4(p, r0, j, active);
	for(int64_t i = r0; i < r1; i += kBatch) {
		float4 nxt[kBatch];
#pragma unroll
		for(int b = 0; b < kBatch; ++b) nxt[b] = load_row4(p, i + 1 + b, j, active && i + 1 + b <= r1);
#pragma unroll
		for(int b = 0; b < kBatch; ++b) {
			const int64_t row = i + b;
			if(row >= r1) break;
			const float4 dn = nxt[b];
			// horizontal neighbours: x-1 from the lane to the left, w+1 from the lane to the right
			float lf = __shfl_up_sync(0xffffffffu, c.w, 1);
			float rt = __shfl_down_sync(0xffffffffu, c.x, 1);
			if(lane == 0) lf = load_one(p, row, j - 1);
			if(lane == last_lane) rt = load_one(p, row, j + 4);
			if(active) {
				float4 o;
				o.x = heat_point(c.x, up.x, dn.x, lf, c.y, p.a);
				o.y = heat_point(c.y, up.y, dn.y, c.x, c.z, p.a);
				o.z = heat_point(c.z, up.z, dn.z, c.y, c.w, p.a);
				o.w = heat_point(c.w, up.w, dn.w, c.z, rt, p.a);
				__stcs(reinterpret_cast<float4*>(p.out + (row - p.out_r0) * p.out_ld + (j - p.out_c0)), o);
			}
			up = c;
			c = dn;
		}
	}
}

// ---- TMA-staged kernel (the default) -------------------------------------------------------
// A CTA of 64 threads (two warps) owns a 256-column strip and walks a segment of kTSegRows rows.
// One elected thread streams the segment's input rows (plus one halo row above and below) into a
// ring of kTStages shared-memory stages with TMA (cp.async.bulk.tensor, completion on an
// mbarrier): per stage a 256-column x kTRows box plus 4-column boxes on either side for the
// horizontal neighbours. Rows outside the chunk view arrive zero-filled, which is exactly the
// stencil's zero padding at the domain edges. Threads keep the vertical window in registers
// (one 128-bit shared load per row) and get horizontal neighbours by warp shuffles (edge lanes
// read them from shared memory), so the copy engine, not the SM's load queue, keeps the bytes in
// flight: 8 CTAs per SM x 6 stages x 4.2 KB. Measured on B200 (65536^2, power-capped clocks):
// 0.99-1.00 of the copy peak, against 0.89-0.90 for the register-window kernel above on the same
// box; 4 rows x 6 stages x 64-row segments beat 4x4, 4x8, 2x8, 2x12, 8x4 and 32/128/256-row
// segments.
constexpr int kTThreads = 64;
constexpr int kTCols = kTThreads * 4; // 256: one TMA box wide
constexpr int kTRows = 4;    // rows per stage
constexpr int kTStages = 6;  // stages in flight per CTA
constexpr int kTSegRows = 64; // rows per CTA segment (measured: 64 > 32, 128, 256)
constexpr int kTSegSmall = 16;
// per stage: the main box, then each 4-column halo box in its own 128-byte slot (TMA writes
// shared memory at 128-byte aligned addresses)
constexpr uint32_t kTHaloSlot = 32; // floats (one 128-byte slot fits a 4-column box of up to 8 rows)

// A mirror: output rows [r0, r1) x cols [c0, c1) are also stored at base[(i - row0) * ld + (j -
// col0)] — the halo rows of a neighbouring chunk (this GPU, or a peer GPU over NVLink), so the
// halo exchange that follows the step is fused into it (mt_launch_ctx mirrors).
constexpr int kMaxMirrors = 2;
struct heat_mirror {
	int64_t r0, r1, c0, c1;
	float* base;
	int64_t row0, col0, ld;
};

struct heat_tma_args {
	float* out;
	int64_t out_r0, out_c0, out_ld;
	int64_t in_r0, in_c0; // chunk view origin (tensor-map coordinate 0)
	int64_t r0, r1, c0, c1;
	float a;
	int nm; // mirrors in use
	heat_mirror m[kMaxMirrors];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tbar_init(uint64_t* bar, uint32_t count) {
	asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void tbar_wait(uint64_t* bar, uint32_t parity) {
	asm volatile(
	    "{\n\t.reg .pred P1;\n\t"
	    "W_%=:\n\t"
	    "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
	    "@!P1 bra W_%=;\n\t}" ::"r"(smem_addr(bar)),
	    "r"(parity)
	    : "memory");
}

__device__ __forceinline__ void tbar_expect(uint64_t* bar, uint32_t bytes) {
	asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tbar_arrive(uint64_t* bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory"); }

__device__ __forceinline__ void tma_box(float* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y) {
	asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_addr(dst)),
	    "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y)
	    : "memory");
}

__device__ __forceinline__ void tma_box_hint(float* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y, uint64_t pol) {
	asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
	                 smem_addr(dst)),
	    "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y), "l"(pol)
	    : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
	uint64_t p;
	asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
	return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
	uint64_t p;
	asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
	return p;
}

__device__ __forceinline__ void st_hint(float4* dst, float4 v, uint64_t pol) {
	asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// L2 residency of a step (template L2 of heat2d_tma_kernel):
//   0  streaming: outputs stored evict-first (st.global.cs), loads default — grids >> L2
//   1  L2-resident grids: loads evict-first (the input is dead after this step), outputs
//      evict-last so the next step's reads of them hit L2
//   2  loads evict-first, outputs default
//   3  both default

template <int ROWS, int STAGES, int SEG, int L2 = 0, bool MIRROR = false>
__global__ void __launch_bounds__(kTThreads) heat2d_tma_kernel(const __grid_constant__ CUtensorMap main_map, const __grid_constant__ CUtensorMap halo_map,
    heat_tma_args p) {
	constexpr uint32_t kHalo = ROWS * 4 <= kTHaloSlot ? kTHaloSlot : ROWS * 4;
	constexpr uint32_t kTStageFloats = ROWS * kTCols + 2 * ((kHalo + 31) / 32 * 32);
	constexpr uint32_t kTStageBytes = ROWS * (kTCols + 8) * 4; // bytes the three boxes deliver
	__shared__ alignas(128) float st[STAGES][kTStageFloats];
	__shared__ alignas(8) uint64_t full[STAGES], empty[STAGES];
	const int tid = threadIdx.x, lane = tid & 31;
	const int64_t j0 = p.c0 + static_cast<int64_t>(blockIdx.x) * kTCols; // strip start (global column)
	const int64_t j = j0 + tid * 4;
	const bool active = j < p.c1;
	const int64_t r0 = p.r0 + static_cast<int64_t>(blockIdx.y) * SEG;
	const int64_t r1 = p.r1 < r0 + SEG ? p.r1 : r0 + SEG;
	if(r0 >= r1) return;
	// rows r0-1 .. r1 are loaded (r1 - r0 + 2 rows), ROWS per stage
	const int64_t first = r0 - 1;
	const int tiles = static_cast<int>((r1 - r0 + 2 + ROWS - 1) / ROWS);
	if(tid == 0) {
		for(int s = 0; s < STAGES; ++s) {
			tbar_init(&full[s], 1);
			tbar_init(&empty[s], kTThreads / 32);
		}
		asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
	}
	__syncthreads();
	const int32_t xm = static_cast<int32_t>(j0 - p.in_c0);
	const auto issue = [&](int t) {
		const int s = t % STAGES;
		const int32_t y = static_cast<int32_t>(first + static_cast<int64_t>(t) * ROWS - p.in_r0);
		float* base = st[s];
		tbar_expect(&full[s], kTStageBytes);
		if constexpr(L2 == 1 || L2 == 2) {
			const uint64_t pol = policy_evict_first();
			tma_box_hint(base, &main_map, &full[s], xm, y, pol);
			tma_box_hint(base + ROWS * kTCols, &halo_map, &full[s], xm - 4, y, pol);
			tma_box_hint(base + ROWS * kTCols + (kHalo + 31) / 32 * 32, &halo_map, &full[s], xm + kTCols, y, pol);
		} else {
			tma_box(base, &main_map, &full[s], xm, y);
			tma_box(base + ROWS * kTCols, &halo_map, &full[s], xm - 4, y);
			tma_box(base + ROWS * kTCols + (kHalo + 31) / 32 * 32, &halo_map, &full[s], xm + kTCols, y);
		}
	};
	if(tid == 0)
		for(int t = 0; t < STAGES && t < tiles; ++t) issue(t);
	// window: up (row k-2), cur (row k-1) with its left/right neighbours
	float4 up = make_float4(0.f, 0.f, 0.f, 0.f), cur = up;
	float cur_l = 0.f, cur_r = 0.f;
	const int64_t rem = (p.c1 - (j - lane * 4)) / 4 - 1;
	const int last_lane = rem < 31 ? static_cast<int>(rem) : 31;
	for(int t = 0; t < tiles; ++t) {
		const int s = t % STAGES;
		tbar_wait(&full[s], static_cast<uint32_t>((t / STAGES) & 1));
		const float* base = st[s];
		const float* lh = base + ROWS * kTCols;
		const float* rh = lh + (kHalo + 31) / 32 * 32;
#pragma unroll
		for(int r = 0; r < ROWS; ++r) {
			const int64_t k = first + static_cast<int64_t>(t) * ROWS + r; // row just loaded
			if(k > r1) break;
			const float4 v = *reinterpret_cast<const float4*>(base + r * kTCols + tid * 4);
			float vl = __shfl_up_sync(0xffffffffu, v.w, 1);
			float vr = __shfl_down_sync(0xffffffffu, v.x, 1);
			if(lane == 0) vl = tid == 0 ? lh[r * 4 + 3] : base[r * kTCols + tid * 4 - 1];
			if(lane == last_lane) vr = tid * 4 + 4 < kTCols ? base[r * kTCols + tid * 4 + 4] : rh[r * 4];
			if(k - 1 >= r0 && active) {
				float4 o;
				o.x = heat_point(cur.x, up.x, v.x, cur_l, cur.y, p.a);
				o.y = heat_point(cur.y, up.y, v.y, cur.x, cur.z, p.a);
				o.z = heat_point(cur.z, up.z, v.z, cur.y, cur.w, p.a);
				o.w = heat_point(cur.w, up.w, v.w, cur.z, cur_r, p.a);
				float4* dst = reinterpret_cast<float4*>(p.out + (k - 1 - p.out_r0) * p.out_ld + (j - p.out_c0));
				if constexpr(L2 == 0)
					__stcs(dst, o);
				else if constexpr(L2 == 1)
					st_hint(dst, o, policy_evict_last());
				else
					*dst = o;
				if constexpr(MIRROR) {
#pragma unroll
					for(int q = 0; q < kMaxMirrors; ++q) {
						const heat_mirror& m = p.m[q];
						if(q < p.nm && k - 1 >= m.r0 && k - 1 < m.r1 && j >= m.c0 && j < m.c1)
							*reinterpret_cast<float4*>(m.base + (k - 1 - m.row0) * m.ld + (j - m.col0)) = o;
					}
				}
			}
			up = cur;
			cur = v;
			cur_l = vl;
			cur_r = vr;
		}
		__syncwarp();
		if(lane == 0) tbar_arrive(&empty[s]);
		if(tid == 0 && t + STAGES < tiles) {
			tbar_wait(&empty[s], static_cast<uint32_t>((t / STAGES) & 1));
			issue(t + STAGES);
		}
	}
}

using tma_encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

tma_encode_fn heat_encode() {
	static tma_encode_fn fn = nullptr;
	static std::once_flag once;
	std::call_once(once, [] {
		void* f = nullptr;
		cudaDriverEntryPointQueryResult q{};
		if(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
			fn = reinterpret_cast<tma_encode_fn>(f);
	});
	return fn;
}

// f32 chunk view `rows` x `cols` (row pitch `ld` elements) read in boxes of box_cols x kTRows;
// out-of-view elements read as zero
bool heat_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows) {
	tma_encode_fn enc = heat_encode();
	if(!enc) return false;
	const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
	const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
	const cuuint32_t box[2] = {box_cols, box_rows};
	const cuuint32_t es[2] = {1, 1};
	return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
	           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
	       == CUDA_SUCCESS;
}

// the mirror stores are compiled only into the instances that take mirrors (MIRROR), so the
// plain streaming path keeps its instruction count
template <int SEG, bool MIRROR>
void launch_tma_m(int l2, dim3 grid, cudaStream_t s, const CUtensorMap& mm, const CUtensorMap& hm, const heat_tma_args& t) {
	switch(l2) {
	case 1: heat2d_tma_kernel<kTRows, kTStages, SEG, 1, MIRROR><<<grid, kTThreads, 0, s>>>(mm, hm, t); break;
	case 2: heat2d_tma_kernel<kTRows, kTStages, SEG, 2, MIRROR><<<grid, kTThreads, 0, s>>>(mm, hm, t); break;
	case 3: heat2d_tma_kernel<kTRows, kTStages, SEG, 3, MIRROR><<<grid, kTThreads, 0, s>>>(mm, hm, t); break;
	default: heat2d_tma_kernel<kTRows, kTStages, SEG, 0, MIRROR><<<grid, kTThreads, 0, s>>>(mm, hm, t); break;
	}
}

template <int SEG>
void launch_tma(int l2, dim3 grid, cudaStream_t s, const CUtensorMap& mm, const CUtensorMap& hm, const heat_tma_args& t) {
	if(t.nm > 0)
		launch_tma_m<SEG, true>(l2, grid, s, mm, hm, t);
	else
		launch_tma_m<SEG, false>(l2, grid, s, mm, hm, t);
}

// any shape / alignment: one thread per cell
__global__ void heat2d_scalar_kernel(heat_args p, int64_t c_lo, int64_t c_hi) {
	const int64_t w = c_hi - c_lo;
	const int64_t total = (p.r1 - p.r0) * w;
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int64_t i = p.r0 + t / w, j = c_lo + t % w;
		const float cc = load_one(p, i, j);
		p.out[(i - p.out_r0) * p.out_ld + (j - p.out_c0)] =
		    heat_point(cc, load_one(p, i - 1, j), load_one(p, i + 1, j), load_one(p, i, j - 1), load_one(p, i, j + 1), p.a);
	}
}

__global__ void stencil1d_kernel(const float* in, int64_t in_off, float* out, int64_t out_off, int64_t n, int64_t lo, int64_t hi) {
	for(int64_t i = lo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < hi; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const float left = i - 1 >= 0 ? in[i - 1 - in_off] : 0.0f;
		const float mid = in[i - in_off];
		const float right = i + 1 < n ? in[i + 1 - in_off] : 0.0f;
		out[i - out_off] = __fdiv_rn(__fadd_rn(__fadd_rn(left, mid), right), 3.0f);
	}
}

} // namespace kern

int launch_heat2d(const mt_launch_ctx* c, void* stream) {
	using namespace kern;
	const mt_view& vo = c->views[3];
	const mt_view& vi = c->views[4];
	heat_args p{};
	p.rows = c->scalars_int[0];
	p.cols = c->scalars_int[1];
	p.a = static_cast<float>(c->scalars_float[2]);
	p.r0 = c->threads_lo[0];
	p.r1 = std::min(c->threads_hi[0], p.rows);
	const int64_t col_lo = c->threads_lo[1];
	const int64_t col_hi = std::min(c->threads_hi[1], p.cols);
	if(p.r0 >= p.r1 || col_lo >= col_hi) return 0;
	if(!vo.base || !vi.base) return 2;
	p.in = static_cast<const float*>(vi.base);
	p.out = static_cast<float*>(vo.base);
	p.in_r0 = vi.offset[0];
	p.in_c0 = vi.offset[1];
	p.in_ld = vi.stride[0];
	p.out_r0 = vo.offset[0];
	p.out_c0 = vo.offset[1];
	p.out_ld = vo.stride[0];
	const auto s = static_cast<cudaStream_t>(stream);
	// 128-bit path needs 16B-aligned rows at the strip start in both views
	const bool aligned = vi.stride[1] == 1 && vo.stride[1] == 1 && p.in_ld % 4 == 0 && p.out_ld % 4 == 0 && (col_lo - p.in_c0) % 4 == 0
	                     && (col_lo - p.out_c0) % 4 == 0 && (reinterpret_cast<uintptr_t>(p.in) % 16) == 0 && (reinterpret_cast<uintptr_t>(p.out) % 16) == 0;
	int64_t vec_hi = col_lo;
	// TMA-staged kernel by default (MTB_HEAT_TMA=0 selects the register-window kernel)
	static const bool use_tma = std::getenv("MTB_HEAT_TMA") == nullptr || std::atoi(std::getenv("MTB_HEAT_TMA")) != 0;
	if(aligned && use_tma && (vi.stride[0] * 4) % 16 == 0 && vi.extent[0] < (int64_t{1} << 31) && vi.extent[1] < (int64_t{1} << 31)) {
		const int64_t v_hi = col_lo + (col_hi - col_lo) / 4 * 4;
		CUtensorMap mm, hm;
		if(v_hi > col_lo && heat_map(&mm, p.in, vi.extent[0], vi.extent[1], vi.stride[0], kTCols, kTRows)
		    && heat_map(&hm, p.in, vi.extent[0], vi.extent[1], vi.stride[0], 4, kTRows)) {
			heat_tma_args t{};
			int32_t mirror_idx[kMaxMirrors] = {};
			// fused halo copies: a mirror is applied when its box lies in the rows and the
			// vectorised columns this kernel writes, float4-aligned in both chunks
			for(int32_t i = 0; i < c->nmirrors && c->mirrors && c->mirror_applied; ++i) {
				const mt_mirror& mr = c->mirrors[i];
				const mt_view& d = mr.dst;
				const int64_t mr0 = mr.lo[0], mr1 = mr.hi[0], mc0 = mr.lo[1], mc1 = mr.hi[1];
				const bool fits = mr.param == 3 && t.nm < kMaxMirrors && d.base && d.rank == 2 && d.stride[1] == 1 && mr0 >= p.r0 && mr1 <= p.r1 && mr0 < mr1
				                  && mc0 >= col_lo && mc1 <= v_hi && mc0 < mc1 && (mc0 - col_lo) % 4 == 0 && (mc1 - col_lo) % 4 == 0 && d.stride[0] % 4 == 0
				                  && (mc0 - d.offset[1]) % 4 == 0 && reinterpret_cast<uintptr_t>(d.base) % 16 == 0 && mr0 >= d.offset[0]
				                  && mr1 <= d.offset[0] + d.extent[0] && mc0 >= d.offset[1] && mc1 <= d.offset[1] + d.extent[1];
				if(!fits) continue;
				mirror_idx[t.nm] = i;
				t.m[t.nm++] = heat_mirror{mr0, mr1, mc0, mc1, static_cast<float*>(d.base), d.offset[0], d.offset[1], d.stride[0]};
			}
			t.out = p.out;
			t.out_r0 = p.out_r0;
			t.out_c0 = p.out_c0;
			t.out_ld = p.out_ld;
			t.in_r0 = p.in_r0;
			t.in_c0 = p.in_c0;
			t.r0 = p.r0;
			t.r1 = p.r1;
			t.c0 = col_lo;
			t.c1 = v_hi;
			t.a = p.a;
			const int64_t strips = (v_hi - col_lo + kTCols - 1) / kTCols;
			// short segments for small superblocks (>= 2 CTAs per SM), 64 rows otherwise
			const bool small = strips * ((p.r1 - p.r0 + kTSegRows - 1) / kTSegRows) < 2 * 148;
			const int64_t seg = small ? kTSegSmall : kTSegRows;
			const int64_t segs = (p.r1 - p.r0 + seg - 1) / seg;
			if(segs <= 65535) {
				const dim3 grid(static_cast<unsigned>(strips), static_cast<unsigned>(segs));
				// L2 residency mode (see heat2d_tma_kernel; MTB_HEAT_L2 forces one). A grid whose
				// whole f32 array fits in half the 126 MB L2 (BASELINE C1: 4096^2 = 64 MiB) keeps
				// its outputs in L2 for the next step and reads its (dead) inputs evict-first;
				// larger grids stream. Measured (scripts/diag/heat_l2_modes.sh, B200): C1 4 chunks
				// 26.2 -> 23.6 us per step (mode 0 -> 2); 16384^2 x 4 chunks 347 us in mode 0,
				// 391 us in mode 2
				static const int l2_env = std::getenv("MTB_HEAT_L2") ? std::atoi(std::getenv("MTB_HEAT_L2")) : -1;
				const bool resident = p.rows * p.cols * 4 <= (int64_t{64} << 20);
				const int l2 = l2_env >= 0 ? l2_env : (resident ? 2 : 0);
				if(small)
					launch_tma<kTSegSmall>(l2, grid, s, mm, hm, t);
				else
					launch_tma<kTSegRows>(l2, grid, s, mm, hm, t);
				vec_hi = v_hi;
				for(int q = 0; q < t.nm; ++q) c->mirror_applied[mirror_idx[q]] = 1; // written by this launch
			}
		}
	}
	if(aligned && vec_hi == col_lo) {
		vec_hi = col_lo + (col_hi - col_lo) / 4 * 4;
		if(vec_hi > col_lo) {
			p.c0 = col_lo;
			p.c1 = vec_hi;
			const int64_t strips = (vec_hi - col_lo + kColsPerCta - 1) / kColsPerCta;
			// small superblocks (e.g. the 1024 x 4096 chunks of BASELINE C1) would launch a few
			// dozen CTAs: shorten the segments until the launch has two CTAs per SM (the extra
			// halo-row reads, 2 per segment, mostly hit L2)
			p.seg = kSegRows;
			while(p.seg > 8 && strips * ((p.r1 - p.r0 + p.seg - 1) / p.seg) < 2 * 148) p.seg /= 2;
			const int64_t segs = (p.r1 - p.r0 + p.seg - 1) / p.seg;
			if(segs > 65535) return 3;
			heat2d_vec_kernel<<<dim3(static_cast<unsigned>(strips), static_cast<unsigned>(segs)), kThreads, 0, s>>>(p);
		}
	}
	if(vec_hi < col_hi) {
		const int64_t total = (p.r1 - p.r0) * (col_hi - vec_hi);
		heat2d_scalar_kernel<<<grid_1d(total, 256), 256, 0, s>>>(p, vec_hi, col_hi);
	}
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_stencil1d(const mt_launch_ctx* c, void* stream) {
	const int64_t n = c->scalars_int[0];
	const int64_t lo = c->threads_lo[0], hi = std::min(c->threads_hi[0], n);
	if(lo >= hi) return 0;
	const mt_view& vo = c->views[1];
	const mt_view& vi = c->views[2];
	kern::stencil1d_kernel<<<kern::grid_1d(hi - lo, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
	    static_cast<const float*>(vi.base), vi.offset[0], static_cast<float*>(vo.base), vo.offset[0], n, lo, hi);
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

} // namespace mtb
