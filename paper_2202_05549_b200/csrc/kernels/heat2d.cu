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
	if(aligned) {
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
