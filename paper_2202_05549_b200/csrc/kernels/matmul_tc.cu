// Dense contraction on the 5th-generation tensor cores: C (f32) = A (bf16) x Bt^T (bf16).
//
// BASELINE config C3 (dense matmul with tiled distribution). The reference's `matmul`
// (kernels.cpp:167-193) is a scalar f32 loop; this is the tensor-core contraction the
// north_star asks for, registered as kernel `matmul_nt_bf16`:
//   params  (m, n, k : i64, C : f32[2] writable, A : bf16[2], Bt : bf16[2])
//   annot.  global [i, j] => write C[i,j], read A[i,:], read Bt[j,:]
//   C[i,j] = sum_l A[i,l] * Bt[j,l]   (products exact in f32, f32 accumulation)
// Both operands are K-major (Bt is B transposed), the layout UMMA consumes natively.
//
// Kernel structure (persistent, one CTA per SM, 192 threads, 6 warps):
//   warp 0   TMA producer: 128x64 A and 256x64 Bt bf16 boxes (128B swizzle) into a 4-stage
//            smem ring, completion counted on `full` mbarriers (expect_tx)
//   warp 1   TMEM allocator + MMA issuer: one elected lane issues tcgen05.mma.cta_group::1
//            .kind::f16, M=128 N=256 K=16, 4 per stage, accumulating in TMEM; tcgen05.commit
//            frees the smem stage (`empty`) and, after the last K block, signals `tmem_full`
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 (each warp its 32 TMEM lanes = rows), f32
//            stores to C with edge masking, then arrive `tmem_empty`
// TMEM holds two 128x256 f32 accumulators (512 columns), so the epilogue of tile t overlaps
// the MMAs of tile t+1. Tiles are rasterised in groups of 16 M-blocks so the ~148 tiles in
// flight share A/B K-slices through L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>

#include "../executor.hpp"
#include "../registry.hpp"
#include "common.cuh"

namespace mtb {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, UMMA_K = 16;
constexpr int NUM_THREADS = 192;
constexpr uint32_t A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_STAGE_BYTES = BN * BK * 2;  // 32 KB
constexpr uint32_t STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr uint32_t TMEM_COLS = 512;                // two 256-column f32 accumulators
constexpr int GROUP_M = 16;
// epilogue staging: per epilogue warp a 32 x 32 f32 block, rows padded to 36 floats (16-byte
// aligned rows, conflict-free 128-bit shared stores and loads); the C stores then go out as whole
// 128-byte row segments (see the epilogues)
constexpr int kEpiPitch = 36;
constexpr size_t kEpiBytes = 4 * 32 * kEpiPitch * sizeof(float);
constexpr size_t SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/ + kEpiBytes;
// CTA pair (cta_group::2): a 256x256 tile per pair; per CTA per stage its 128 A rows and its
// 128 of the 256 Bt rows, so 32 KB per stage and 6 stages in flight
constexpr int STAGES2 = 6;
constexpr uint32_t B2_STAGE_BYTES = (BN / 2) * BK * 2; // 16 KB
constexpr uint32_t STAGE2_BYTES = A_STAGE_BYTES + B2_STAGE_BYTES;
constexpr size_t SMEM2_BYTES = 1024 + STAGES2 * STAGE2_BYTES + 256;
constexpr int kTileRing = 4; // dynamic scheduler: tile ids in flight per CTA
// Wide CTA pair (NSUB = 2): a 256x512 tile per pair, two M256 N256 MMAs per K step into the two
// halves of the 512 TMEM columns (one accumulator, no double buffering); per CTA a stage holds
// 128 A rows and 2 x 128 Bt rows = 48 KB, so 4 stages. Per flop it moves half the operand bytes
// of the single-CTA kernel from L2 (the tile shape cuBLAS picks at 32768^3,
// nvjet_tst_256x256_64x4_2x1_2cta).
__host__ __device__ constexpr int pair_stages(int nsub) { return nsub == 1 ? STAGES2 : 4; }
__host__ __device__ constexpr size_t pair_smem_bytes(int nsub) {
	return 1024 + static_cast<size_t>(pair_stages(nsub)) * (A_STAGE_BYTES + nsub * B2_STAGE_BYTES) + 256 + kEpiBytes;
}
static_assert(pair_smem_bytes(2) <= 227 * 1024, "wide pair stages");
static_assert((2 * STAGES2 + 4 + 2 * kTileRing) * 8 + 4 * kTileRing + 4 <= 256, "barrier area");
static_assert((2 * STAGES + 4 + 2 * kTileRing) * 8 + 4 * kTileRing + 4 <= 256, "barrier area");

struct gemm_args {
	float* c;
	int64_t ldc;       // elements
	int64_t m, n, k;   // problem (rows of C, cols of C, reduction)
	int64_t a_row0;    // A tensor-map row of output row 0
	int64_t b_row0;    // Bt tensor-map row of output col 0
	int m_blocks, n_blocks, k_blocks;
	int group_m; // rasterisation group (M units)
	uint64_t hint_a, hint_b; // L2 cache policies of the operand loads
	int no_store;            // diagnostics (MTB_GEMM_NOSTORE): skip the C stores
	int n_major;             // diagnostics (MTB_GEMM_NMAJOR): rasterise N-first
	int epi_rowwise;         // A/B (MTB_GEMM_EPI=0): the per-row epilogue stores instead of the transposed ones
	unsigned* sched;         // dynamic tile counter (zeroed per launch); null: static round robin
	unsigned long long* trace; // diagnostics (MTB_GEMM_TRACE): per tile {cluster, start ns, end ns} of the MMA issue
};

// ---- PTX wrappers -------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
	asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
	float4 f;
	asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w) : "r"(addr) : "memory");
	return f;
}

// one 32 x 32 f32 block of C from the epilogue warp's registers (lane = row, r = its 32 columns)
// through its shared staging block (32 rows of kEpiPitch floats at `epi`, a shared address), so
// that every 128-bit global store writes four whole 128-byte row segments
__device__ __forceinline__ void store_block_transposed(uint32_t epi, const uint32_t (&r)[32], float* c, int64_t ldc, int64_t row0, int64_t col0, int lane, int pitch) {
#pragma unroll
	for(int v = 0; v < 8; ++v) sts128(epi + static_cast<uint32_t>((lane * pitch + 4 * v) * 4), r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
	__syncwarp();
	const int rr = lane >> 3, cc = (lane & 7) * 4;
	float4 f[8];
#pragma unroll
	for(int v = 0; v < 8; ++v) f[v] = lds128(epi + static_cast<uint32_t>(((4 * v + rr) * pitch + cc) * 4));
#pragma unroll
	for(int v = 0; v < 8; ++v) *reinterpret_cast<float4*>(c + (row0 + 4 * v + rr) * ldc + col0 + cc) = f[v];
	__syncwarp();
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
	asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
	asm volatile(
	    "{\n\t.reg .pred P1;\n\t"
	    "WAIT_%=:\n\t"
	    "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
	    "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
	    "r"(parity)
	    : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
	asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
	asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y) {
	asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
	    "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
	    : "memory");
}


// cta_group::2 load: data into this CTA's smem, completion on the LEADER CTA's mbarrier (the
// peer bit of the shared::cluster address cleared)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y, uint64_t hint) {
	asm volatile(
	    "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
	        smem_u32(dst)),
	    "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y), "l"(hint)
	    : "memory");
}

__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
	asm volatile(
	    "{\n\t.reg .pred p;\n\t"
	    "setp.ne.b32 p, %4, 0;\n\t"
	    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
	    "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tc_mma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
	asm volatile(
	    "{\n\t.reg .pred p;\n\t"
	    "setp.ne.b32 p, %4, 0;\n\t"
	    "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
	    "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tc_commit2_mc(uint64_t* bar, uint16_t mask) {
	asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
	    : "memory");
}

// arrive on the mbarrier at `bar`'s offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
	asm volatile(
	    "{\n\t.reg .b32 ra;\n\t"
	    "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
	    "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
	    "r"(rank)
	    : "memory");
}

// acquire at cluster scope: the data guarded by the barrier was written by the peer CTA
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
	asm volatile(
	    "{\n\t.reg .pred P1;\n\t"
	    "WAIT_%=:\n\t"
	    "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
	    "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
	    "r"(parity)
	    : "memory");
}

// store `v` at `dst`'s offset in CTA `rank`'s shared memory
__device__ __forceinline__ void st_cluster_u32(uint32_t* dst, uint32_t rank, uint32_t v) {
	asm volatile(
	    "{\n\t.reg .b32 ra;\n\t"
	    "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
	    "st.shared::cluster.u32 [ra], %2;\n\t}" ::"r"(smem_u32(dst)),
	    "r"(rank), "r"(v)
	    : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
	uint32_t r;
	asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
	return r;
}

__device__ __forceinline__ void cluster_sync_all() {
	asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
	asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
	asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}


__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
	asm volatile(
	    "{\n\t.reg .pred p;\n\t"
	    "setp.ne.b32 p, %4, 0;\n\t"
	    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
	    "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::tf32: f32 operands read as TF32 (the low 13 mantissa bits are not used), K = 8 per MMA
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
	asm volatile(
	    "{\n\t.reg .pred p;\n\t"
	    "setp.ne.b32 p, %4, 0;\n\t"
	    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
	    "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// K-major operand, 128-byte swizzle: 8-row atoms of 1024 B (SBO), version 1, layout type 2
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
	uint64_t d = 0;
	d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
	d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
	d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
	d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
	d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
	return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N = `m` x 256
__host__ __device__ constexpr uint32_t instr_desc(int m = BM) {
	return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// kind::tf32 instruction descriptor: tf32 x tf32 -> f32 (formats 2), both K-major, 128 x 256
__host__ __device__ constexpr uint32_t instr_desc_tf32(int m = BM) {
	return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
	asm volatile(
	    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%"
	    "28,%29,%30,%31}, [%32];"
	    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
	    "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
	    "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
	    : "r"(taddr));
	asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tile t -> (M unit, N block), rasterised in groups of GROUP_M M units (units = M blocks, or
// M block pairs for the CTA-pair kernel)
__device__ __forceinline__ void tile_coords(int t, const gemm_args& p, int& mb, int& nb, int m_units, int n_units) {
	if(p.n_major) { // diagnostics: groups of group_m N blocks, M fastest across the group
		const int group = p.group_m * m_units;
		const int g = t / group;
		const int first_n = g * p.group_m;
		const int cols = min(p.group_m, n_units - first_n);
		const int r = t % group;
		nb = first_n + r % cols;
		mb = r / cols;
		return;
	}
	const int group = p.group_m * n_units;
	const int g = t / group;
	const int first_m = g * p.group_m;
	const int rows = min(p.group_m, m_units - first_m);
	const int r = t % group;
	mb = first_m + r % rows;
	nb = r / rows;
}

// TF32: f32 operands (kind::tf32). A stage is still one 128-byte swizzle row per operand row,
// i.e. 32 f32 instead of 64 bf16 of K, and each of its 4 MMAs covers 32 bytes of K (8 f32).
template <bool TF32>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_nt_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b, gemm_args p) {
	constexpr int BKE = TF32 ? BK / 2 : BK; // K elements per stage
	extern __shared__ uint8_t smem_raw[];
	uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
	uint8_t* a_smem = smem;
	uint8_t* b_smem = smem + STAGES * A_STAGE_BYTES;
	uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
	uint64_t* full = bars;
	uint64_t* empty = bars + STAGES;
	uint64_t* tmem_full = bars + 2 * STAGES;
	uint64_t* tmem_empty = bars + 2 * STAGES + 2;
	uint64_t* tile_full = bars + 2 * STAGES + 4; // dynamic scheduler ring (see the CTA-pair kernel)
	uint64_t* tile_empty = tile_full + kTileRing;
	uint32_t* tile_ring = reinterpret_cast<uint32_t*>(tile_empty + kTileRing);
	uint32_t* tmem_slot = tile_ring + kTileRing;

	const int warp = threadIdx.x / 32;
	const int lane = threadIdx.x % 32;
	const int num_tiles = p.m_blocks * p.n_blocks;
	const bool dyn = p.sched != nullptr;
	const auto next_tile = [&](int i, int t_static) -> int {
		if(!dyn) return t_static;
		const int slot = i % kTileRing;
		mbar_wait(&tile_full[slot], static_cast<uint32_t>((i / kTileRing) & 1));
		const int t = static_cast<int>(tile_ring[slot]);
		mbar_arrive(&tile_empty[slot]);
		return t;
	};

	if(warp == 0 && lane == 0) {
		for(int s = 0; s < STAGES; ++s) {
			mbar_init(&full[s], 1);
			mbar_init(&empty[s], 1);
		}
		for(int a = 0; a < 2; ++a) {
			mbar_init(&tmem_full[a], 1);
			mbar_init(&tmem_empty[a], 4);
		}
		for(int r = 0; r < kTileRing; ++r) {
			mbar_init(&tile_full[r], 1);
			mbar_init(&tile_empty[r], 5); // MMA + 4 epilogue warps
		}
		asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
		asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
		asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
	}
	if(warp == 1) {
		asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
		asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
	}
	tc_fence_before();
	__syncthreads();
	tc_fence_after();
	const uint32_t tmem_base = *tmem_slot;

	if(warp == 0) {
		if(lane == 0) {
			// ---- TMA producer ----
			int stage = 0;
			uint32_t phase = 0;
			for(int i = 0, ts = blockIdx.x;; ++i, ts += gridDim.x) {
				int t = ts;
				if(dyn) {
					const int slot = i % kTileRing;
					mbar_wait(&tile_empty[slot], static_cast<uint32_t>(((i / kTileRing) & 1) ^ 1));
					t = static_cast<int>(atomicAdd(p.sched, 1u));
					tile_ring[slot] = static_cast<uint32_t>(t);
					mbar_arrive(&tile_full[slot]); // release (cta): the ring entry is visible to the waiters
				}
				if(t >= num_tiles) break;
				int mb, nb;
				tile_coords(t, p, mb, nb, p.m_blocks, p.n_blocks);
				const int32_t arow = static_cast<int32_t>(p.a_row0 + static_cast<int64_t>(mb) * BM);
				const int32_t brow = static_cast<int32_t>(p.b_row0 + static_cast<int64_t>(nb) * BN);
				for(int kb = 0; kb < p.k_blocks; ++kb) {
					mbar_wait(&empty[stage], phase ^ 1);
					mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
					tma_load_2d(a_smem + stage * A_STAGE_BYTES, &tmap_a, &full[stage], kb * BKE, arow);
					tma_load_2d(b_smem + stage * B_STAGE_BYTES, &tmap_b, &full[stage], kb * BKE, brow);
					if(++stage == STAGES) {
						stage = 0;
						phase ^= 1;
					}
				}
			}
		}
	} else if(warp == 1) {
		if(lane == 0) {
			// ---- MMA issuer ----
			constexpr uint32_t idesc = TF32 ? instr_desc_tf32() : instr_desc();
			int stage = 0;
			uint32_t phase = 0;
			for(int local = 0, ts = blockIdx.x;; ++local, ts += gridDim.x) {
				const int t = next_tile(local, ts);
				if(t >= num_tiles) break;
				const int acc = local & 1;
				mbar_wait(&tmem_empty[acc], ((local >> 1) & 1) ^ 1);
				tc_fence_after();
				const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
				for(int kb = 0; kb < p.k_blocks; ++kb) {
					mbar_wait(&full[stage], phase);
					tc_fence_after();
					const uint32_t a0 = smem_u32(a_smem + stage * A_STAGE_BYTES);
					const uint32_t b0 = smem_u32(b_smem + stage * B_STAGE_BYTES);
#pragma unroll
					for(int k = 0; k < BK / UMMA_K; ++k) {
						if constexpr(TF32)
							tc_mma_tf32(d, smem_desc(a0 + k * UMMA_K * 2), smem_desc(b0 + k * UMMA_K * 2), idesc, (kb | k) != 0 ? 1u : 0u);
						else
							tc_mma(d, smem_desc(a0 + k * UMMA_K * 2), smem_desc(b0 + k * UMMA_K * 2), idesc, (kb | k) != 0 ? 1u : 0u);
					}
					tc_commit(&empty[stage]);
					if(++stage == STAGES) {
						stage = 0;
						phase ^= 1;
					}
				}
				tc_commit(&tmem_full[acc]);
			}
		}
	} else {
		// ---- epilogue: warps 2..5, TMEM lanes 32*(warp%4) .. +31 ----
		const int quarter = warp & 3;
		const uint32_t epi = smem_u32(smem + STAGES * STAGE_BYTES + 256) + static_cast<uint32_t>(quarter * 32 * kEpiPitch * 4);
		for(int local = 0, ts = blockIdx.x;; ++local, ts += gridDim.x) {
			int t = ts;
			if(dyn) {
				if(lane == 0) t = next_tile(local, ts);
				t = __shfl_sync(0xffffffffu, t, 0);
			}
			if(t >= num_tiles) break;
			int mb, nb;
			tile_coords(t, p, mb, nb, p.m_blocks, p.n_blocks);
			const int acc = local & 1;
			mbar_wait(&tmem_full[acc], (local >> 1) & 1);
			tc_fence_after();
			const int64_t row0 = static_cast<int64_t>(mb) * BM + quarter * 32; // this warp's first row
			const int64_t row = row0 + lane;
			const bool row_ok = row < p.m;
			float* crow = p.c + row * p.ldc;
			const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN);
			const bool block_rows = !p.epi_rowwise && !p.no_store && row0 + 32 <= p.m && (p.ldc & 3) == 0
			                        && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
#pragma unroll 1
			for(int c = 0; c < BN; c += 32) {
				uint32_t r[32];
				tmem_ld32(taddr + static_cast<uint32_t>(c), r);
				const int64_t col0 = static_cast<int64_t>(nb) * BN + c;
				if(block_rows && col0 + 32 <= p.n) { // transposed through shared memory (CTA-pair kernel)
store_block_transposed(epi, r, p.c, p.ldc, row0, col0, lane, kEpiPitch);
					continue;
				}
				if(!row_ok || p.no_store) continue;
				if(col0 + 32 <= p.n && ((reinterpret_cast<uintptr_t>(crow + col0) & 15) == 0)) {
#pragma unroll
					for(int v = 0; v < 8; ++v) {
						float4 f = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
						*reinterpret_cast<float4*>(crow + col0 + 4 * v) = f;
					}
				} else {
					for(int v = 0; v < 32; ++v)
						if(col0 + v < p.n) crow[col0 + v] = __uint_as_float(r[v]);
				}
			}
			tc_fence_before();
			__syncwarp();
			if(lane == 0) mbar_arrive(&tmem_empty[acc]);
		}
	}
	__syncthreads();
	if(warp == 1) {
		tc_fence_after();
		asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
	}
}

// ---- CTA pair: tcgen05.mma.cta_group::2, 256x256 tiles -----------------------------------
//
// The two CTAs of a cluster (one TPC) compute one 256x256 tile: each holds 128 rows of A and
// 128 of the 256 Bt rows per stage and the leader (rank 0) issues M=256 N=256 K=16 MMAs that
// read both CTAs' shared memory; each CTA's TMEM receives its own 128 rows. Per CTA a stage is
// 32 KB instead of 48 KB, so 6 stages are in flight and the L2->SM operand traffic per flop is
// a third lower. Both CTAs' TMA loads complete on the leader's `full` barrier (expect_tx set by
// the leader for both); the leader's MMA commit frees the stage in both CTAs and signals both
// CTAs' `tmem_full`; both CTAs' epilogue warps release the accumulator on the leader's
// `tmem_empty` (count 8).
template <bool TF32, int NSUB>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_nt_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b, gemm_args p) {
	constexpr int BKE = TF32 ? BK / 2 : BK; // K elements per stage
	constexpr int kStages = pair_stages(NSUB);
	constexpr uint32_t kBStage = NSUB * B2_STAGE_BYTES;   // this CTA's Bt rows of every N sub-tile
	constexpr uint32_t kStageBytes = A_STAGE_BYTES + kBStage;
	constexpr int kAcc = NSUB == 1 ? 2 : 1;               // accumulators in the 512 TMEM columns
	constexpr int kAccCols = BN * NSUB;                   // columns of one accumulator (= tile N)
	extern __shared__ uint8_t smem_raw[];
	uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
	uint8_t* a_smem = smem;
	uint8_t* b_smem = smem + kStages * A_STAGE_BYTES;
	uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
	uint64_t* full = bars;
	uint64_t* empty = bars + kStages;
	uint64_t* tmem_full = bars + 2 * kStages;
	uint64_t* tmem_empty = bars + 2 * kStages + 2;
	uint64_t* tile_full = bars + 2 * kStages + 4;  // dynamic scheduler ring (kTileRing slots)
	uint64_t* tile_empty = tile_full + kTileRing;
	uint32_t* tile_ring = reinterpret_cast<uint32_t*>(tile_empty + kTileRing);
	uint32_t* tmem_slot = tile_ring + kTileRing;

	const int warp = threadIdx.x / 32;
	const int lane = threadIdx.x % 32;
	const uint32_t rank = cluster_rank();
	const bool leader = rank == 0;
	const int m_pairs = (p.m_blocks + 1) / 2;
	const int n_units = (p.n_blocks + NSUB - 1) / NSUB;
	const int num_units = m_pairs * n_units;
	const int first_unit = static_cast<int>(blockIdx.x) / 2;
	const int unit_stride = static_cast<int>(gridDim.x) / 2;
	constexpr uint16_t kPair = 0x3;
	// Tile sequence of this cluster. Static: first_unit, += unit_stride. Dynamic (p.sched): the
	// leader's producer thread takes the next tile from a global counter and publishes it in both
	// CTAs' rings; every other role reads it from its own ring. Tiles then start in id order as
	// clusters free up, so the tiles in flight stay a window of consecutive ids: panels shared by
	// neighbouring tiles are read at nearly the same K and stay in L2. With a static round robin
	// the clusters drift apart over a long kernel (221 tiles each at 32768^3) and the shared
	// panels are re-read from DRAM (ncu: 274 GB of DRAM reads against 73 GB lockstep).
	const bool dyn = p.sched != nullptr;
	// consumer side: the i-th tile of this role (sentinel >= num_units ends the loop)
	const auto next_tile = [&](int i, int t_static, bool release) -> int {
		if(!dyn) return t_static;
		const int slot = i % kTileRing;
		mbar_wait_cluster(&tile_full[slot], static_cast<uint32_t>((i / kTileRing) & 1));
		const int t = static_cast<int>(tile_ring[slot]);
		if(release) mbar_arrive_remote(&tile_empty[slot], 0);
		return t;
	};

	if(warp == 0 && lane == 0) {
		for(int s = 0; s < kStages; ++s) {
			mbar_init(&full[s], 1);
			mbar_init(&empty[s], 1);
		}
		for(int a = 0; a < 2; ++a) {
			mbar_init(&tmem_full[a], 1);
			mbar_init(&tmem_empty[a], 8);
		}
		for(int r = 0; r < kTileRing; ++r) {
			mbar_init(&tile_full[r], 1);
			mbar_init(&tile_empty[r], 10); // leader: MMA + 4 epilogue warps; peer: producer + 4 epilogue warps
		}
		asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
		asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
		asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
	}
	if(warp == 1) {
		asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
		asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
	}
	tc_fence_before();
	__syncthreads();
	cluster_sync_all();
	tc_fence_after();
	const uint32_t tmem_base = *tmem_slot;

	if(warp == 0) {
		if(lane == 0) {
			// ---- TMA producer (both CTAs) ----
			int stage = 0;
			uint32_t phase = 0;
			for(int i = 0, ts = first_unit;; ++i, ts += unit_stride) {
				int t = ts;
				if(dyn && leader) {
					// take the next tile and publish it to both CTAs' rings
					const int slot = i % kTileRing;
					mbar_wait(&tile_empty[slot], static_cast<uint32_t>(((i / kTileRing) & 1) ^ 1));
					t = static_cast<int>(atomicAdd(p.sched, 1u));
					for(uint32_t r = 0; r < 2; ++r) {
						st_cluster_u32(&tile_ring[slot], r, static_cast<uint32_t>(t));
						mbar_arrive_remote(&tile_full[slot], r);
					}
				} else if(dyn) {
					t = next_tile(i, ts, true);
				}
				if(t >= num_units) break;
				int mu, nb;
				tile_coords(t, p, mu, nb, m_pairs, n_units);
				const int32_t arow = static_cast<int32_t>(p.a_row0 + static_cast<int64_t>(mu) * 2 * BM + rank * BM);
				// sub-tile s of the tile's N: Bt rows [s*BN, (s+1)*BN), this CTA holds half of each
				const int32_t brow = static_cast<int32_t>(p.b_row0 + static_cast<int64_t>(nb) * kAccCols + rank * (BN / 2));
				for(int kb = 0; kb < p.k_blocks; ++kb) {
					mbar_wait(&empty[stage], phase ^ 1);
					if(leader) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
					tma_load_2d_2sm(a_smem + stage * A_STAGE_BYTES, &tmap_a, &full[stage], kb * BKE, arow, p.hint_a);
#pragma unroll
					for(int sub = 0; sub < NSUB; ++sub)
						tma_load_2d_2sm(b_smem + stage * kBStage + sub * B2_STAGE_BYTES, &tmap_b, &full[stage], kb * BKE, brow + sub * BN, p.hint_b);
					if(++stage == kStages) {
						stage = 0;
						phase ^= 1;
					}
				}
			}
		}
	} else if(warp == 1) {
		if(lane == 0 && leader) {
			// ---- MMA issuer (leader only) ----
			constexpr uint32_t idesc = TF32 ? instr_desc_tf32(2 * BM) : instr_desc(2 * BM);
			int stage = 0;
			uint32_t phase = 0;
			for(int local = 0, ts = first_unit;; ++local, ts += unit_stride) {
				const int t = next_tile(local, ts, true);
				if(t >= num_units) break;
				const int acc = local % kAcc;
				mbar_wait(&tmem_empty[acc], ((local / kAcc) & 1) ^ 1);
				tc_fence_after();
				const uint32_t d = tmem_base + static_cast<uint32_t>(acc * kAccCols);
				uint64_t t_start = 0;
				if(p.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
				for(int kb = 0; kb < p.k_blocks; ++kb) {
					mbar_wait(&full[stage], phase);
					tc_fence_after();
					const uint32_t a0 = smem_u32(a_smem + stage * A_STAGE_BYTES);
					const uint32_t b0 = smem_u32(b_smem + stage * kBStage);
#pragma unroll
					for(int k = 0; k < BK / UMMA_K; ++k) {
#pragma unroll
						for(int sub = 0; sub < NSUB; ++sub) {
							const uint32_t dd = d + static_cast<uint32_t>(sub * BN);
							const uint64_t bd = smem_desc(b0 + sub * B2_STAGE_BYTES + k * UMMA_K * 2);
							if constexpr(TF32)
								tc_mma2_tf32(dd, smem_desc(a0 + k * UMMA_K * 2), bd, idesc, (kb | k) != 0 ? 1u : 0u);
							else
								tc_mma2(dd, smem_desc(a0 + k * UMMA_K * 2), bd, idesc, (kb | k) != 0 ? 1u : 0u);
						}
					}
					tc_commit2_mc(&empty[stage], kPair);
					if(++stage == kStages) {
						stage = 0;
						phase ^= 1;
					}
				}
				tc_commit2_mc(&tmem_full[acc], kPair);
				if(p.trace) {
					uint64_t t_end;
					asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
					p.trace[3 * t] = blockIdx.x / 2;
					p.trace[3 * t + 1] = t_start;
					p.trace[3 * t + 2] = t_end;
				}
			}
		}
	} else {
		// ---- epilogue (both CTAs): warps 2..5, own TMEM lanes = own 128 rows ----
		const int quarter = warp & 3;
		const uint32_t epi = smem_u32(smem + kStages * kStageBytes + 256) + static_cast<uint32_t>(quarter * 32 * kEpiPitch * 4);
		for(int local = 0, ts = first_unit;; ++local, ts += unit_stride) {
			int t = ts;
			if(dyn) {
				if(lane == 0) t = next_tile(local, ts, true);
				t = __shfl_sync(0xffffffffu, t, 0);
			}
			if(t >= num_units) break;
			int mu, nb;
			tile_coords(t, p, mu, nb, m_pairs, n_units);
			const int acc = local % kAcc;
			mbar_wait(&tmem_full[acc], (local / kAcc) & 1);
			tc_fence_after();
			const int64_t row0 = static_cast<int64_t>(mu) * 2 * BM + rank * BM + quarter * 32; // this warp's first row
			const int64_t row = row0 + lane;
			const bool row_ok = row < p.m && !p.no_store;
			float* crow = p.c + row * p.ldc;
			const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kAccCols);
			// transposed stores: a 32 x 32 block goes through shared memory so that each 128-bit
			// store instruction writes four whole 128-byte row segments (lanes 8r..8r+7 one row)
			// instead of one 16-byte piece of 32 different rows
			const bool block_rows = !p.epi_rowwise && !p.no_store && row0 + 32 <= p.m && (p.ldc & 3) == 0
			                        && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
#pragma unroll 1
			for(int c = 0; c < kAccCols; c += 32) {
				uint32_t r[32];
				tmem_ld32(taddr + static_cast<uint32_t>(c), r);
				const int64_t col0 = static_cast<int64_t>(nb) * kAccCols + c;
				if(block_rows && col0 + 32 <= p.n) {
store_block_transposed(epi, r, p.c, p.ldc, row0, col0, lane, kEpiPitch);
					continue;
				}
				if(!row_ok) continue;
				if(col0 + 32 <= p.n && ((reinterpret_cast<uintptr_t>(crow + col0) & 15) == 0)) {
#pragma unroll
					for(int v = 0; v < 8; ++v) {
						float4 f = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
						*reinterpret_cast<float4*>(crow + col0 + 4 * v) = f;
					}
				} else {
					for(int v = 0; v < 32; ++v)
						if(col0 + v < p.n) crow[col0 + v] = __uint_as_float(r[v]);
				}
			}
			tc_fence_before();
			__syncwarp();
			if(lane == 0) mbar_arrive_remote(&tmem_empty[acc], 0);
		}
	}
	__syncthreads();
	// the peer may still read this CTA's smem (MMA) or arrive on its barriers
	cluster_sync_all();
	if(warp == 1) {
		tc_fence_after();
		asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
	}
}

// ---- host side -------------------------------------------------------------------------------

using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn get_encode() {
	static encode_fn fn = nullptr;
	static std::once_flag once;
	std::call_once(once, [] {
		void* p = nullptr;
		cudaDriverEntryPointQueryResult q{};
		if(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
			fn = reinterpret_cast<encode_fn>(p);
	});
	return fn;
}

// 2D K-major operand (bf16, or f32 for TF32): `rows` x `cols` (cols contiguous), row pitch `ld`
// elements; boxes of one 128-byte row of K
bool make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows, bool f32 = false) {
	encode_fn enc = get_encode();
	if(!enc) return false;
	const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
	const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * (f32 ? 4 : 2)};
	const cuuint32_t box[2] = {static_cast<cuuint32_t>(f32 ? BK / 2 : BK), box_rows};
	const cuuint32_t estride[2] = {1, 1};
	return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
	           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
	       == CUDA_SUCCESS;
}

std::atomic<uint64_t> g_tc_launches{0}; // tcgen05 contraction launches in this process (mt_tensor_core_launches)

int num_sms() {
	int dev = 0, sms = 148;
	cudaGetDevice(&dev);
	cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
	return sms;
}

// a: rows [a_row0, a_row0 + m) of an (a_rows x k) matrix; bt likewise for n.
int run_gemm(const void* a, int64_t a_rows, int64_t lda, int64_t a_row0, const void* bt, int64_t b_rows, int64_t ldb, int64_t b_row0, float* c,
    int64_t ldc, int64_t m, int64_t n, int64_t k, cudaStream_t s, bool tf32 = false) {
	if(m <= 0 || n <= 0) return 0;
	if(k <= 0) return 5;
	const int64_t es = tf32 ? 4 : 2;
	if((lda * es) % 16 || (ldb * es) % 16 || (reinterpret_cast<uintptr_t>(a) % 16) || (reinterpret_cast<uintptr_t>(bt) % 16)) return 6;
	gemm_args p{};
	p.c = c;
	p.ldc = ldc;
	p.m = m;
	p.n = n;
	p.k = k;
	p.a_row0 = a_row0;
	p.b_row0 = b_row0;
	p.m_blocks = static_cast<int>((m + BM - 1) / BM);
	p.n_blocks = static_cast<int>((n + BN - 1) / BN);
	const int64_t bke = tf32 ? BK / 2 : BK;
	p.k_blocks = static_cast<int>((k + bke - 1) / bke);
	const int sms = num_sms();
	// L2 policies (the CUTLASS encodings): normal 0x1000000000000000, evict-first 0x12F0..., evict-last 0x14F0...
	p.hint_a = p.hint_b = 0x1000000000000000ull;
	if(const char* e = std::getenv("MTB_GEMM_HINT_A")) p.hint_a = std::strtoull(e, nullptr, 16);
	if(const char* e = std::getenv("MTB_GEMM_HINT_B")) p.hint_b = std::strtoull(e, nullptr, 16);
	// Kernel choice (measured on B200 under sustained load, interleaved launches,
	// scripts/diag/gemm_interleaved_ab.py; profiles/round2/gemm_scheduling.md):
	//  * CTA pairs (256x256 tiles, static raster in groups of 16 M units) once there are enough
	//    tiles to fill the machine: best up to 16384^3 (bf16 1532 vs 1214 TFLOP/s single-CTA;
	//    TF32 735 vs 652);
	//  * wide CTA pairs (256x512 tiles) with the dynamic tile counter in groups of 4 M units when
	//    M*N > 16384^2 and K > 16384: 32768^3 bf16 1355 vs 1282 median (single-CTA), TF32 736 vs
	//    630. The wide tile halves the L2->SM operand bytes per flop; cold in ncu it matches
	//    cuBLAS (41.4 vs 41.5 ms, 108 vs 115 GB of DRAM reads), while the 256x256 pair kernel
	//    reads 132-301 GB there whatever its schedule.
	//  * single CTAs (128x256) otherwise.
	const bool big = static_cast<double>(m) * static_cast<double>(n) > 16384.0 * 16384.0 && k > 16384;
	p.no_store = std::getenv("MTB_GEMM_NOSTORE") != nullptr;
	p.epi_rowwise = std::getenv("MTB_GEMM_EPI") && std::atoi(std::getenv("MTB_GEMM_EPI")) == 0;
	if(const char* e = std::getenv("MTB_GEMM_TRACE")) p.trace = reinterpret_cast<unsigned long long*>(std::strtoull(e, nullptr, 0));
	p.n_major = std::getenv("MTB_GEMM_NMAJOR") != nullptr;
	const bool force_pair = std::getenv("MTB_GEMM_FORCE_PAIR") != nullptr;
	const bool no_pair = std::getenv("MTB_GEMM_NO_PAIR") != nullptr;
	// MTB_GEMM_WIDE=1 forces the wide pair kernel, =0 disables it
	const char* we = std::getenv("MTB_GEMM_WIDE");
	const bool wide_ok = p.m_blocks >= 2 && ((p.m_blocks + 1) / 2) * ((p.n_blocks + 1) / 2) * 2 >= sms && !no_pair;
	const bool wide = wide_ok && (we ? std::atoi(we) != 0 : big && !force_pair);
	const bool pair = wide || (p.m_blocks >= 2 && ((p.m_blocks + 1) / 2) * p.n_blocks * 2 >= sms && (!big || force_pair) && !no_pair);
	p.group_m = wide ? 4 : GROUP_M;
	if(const char* e = std::getenv("MTB_GEMM_GROUP")) p.group_m = std::max(1, std::atoi(e));
	CUtensorMap ma, mb;
	if(!make_map(&ma, a, a_rows, k, lda, BM, tf32) || !make_map(&mb, bt, b_rows, k, ldb, pair ? BN / 2 : BN, tf32)) return 7;
	g_tc_launches.fetch_add(1, std::memory_order_relaxed);
	// dynamic tile scheduling (default for the wide kernel, MTB_GEMM_DYNAMIC=1 for the others,
	// MTB_GEMM_STATIC=1 turns it off): a counter per launch (round robin over a per-device pool,
	// so concurrent launches on other streams never share one), zeroed on the stream before the
	// launch. It keeps the tiles in flight a window of consecutive ids (tiles sharing a B panel
	// start within 38 us instead of 985 us at 32768^3 with the static round robin), which the wide
	// kernel needs to keep its shared panels in L2; on the other kernels it is not faster.
	if(std::getenv("MTB_GEMM_DYNAMIC") || wide) {
		constexpr unsigned kCounters = 1024;
		static unsigned* counters[64] = {};
		static unsigned next_counter[64] = {};
		int dev = 0;
		cudaGetDevice(&dev);
		const char* ds = std::getenv("MTB_GEMM_DYN_SINGLE");
		const bool want = !std::getenv("MTB_GEMM_STATIC") && (pair || !ds || std::atoi(ds) != 0);
		if(want && dev < 64) {
			if(!counters[dev] && cudaMalloc(&counters[dev], kCounters * sizeof(unsigned)) != cudaSuccess) counters[dev] = nullptr;
			unsigned* c = counters[dev] ? counters[dev] + (next_counter[dev]++ % kCounters) : nullptr;
			if(c && cudaMemsetAsync(c, 0, sizeof(unsigned), s) == cudaSuccess) p.sched = c;
		}
	}
	if(!pair) {
		const int grid = std::min(p.m_blocks * p.n_blocks, sms);
		if(tf32) {
			kern::ensure_smem(gemm_bf16_nt_kernel<true>, static_cast<int>(SMEM_BYTES));
			gemm_bf16_nt_kernel<true><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ma, mb, p);
		} else {
			kern::ensure_smem(gemm_bf16_nt_kernel<false>, static_cast<int>(SMEM_BYTES));
			gemm_bf16_nt_kernel<false><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ma, mb, p);
		}
		return cudaGetLastError() == cudaSuccess ? 0 : 1;
	}
	const auto pair_kernel = wide ? (tf32 ? gemm_bf16_nt_2sm_kernel<true, 2> : gemm_bf16_nt_2sm_kernel<false, 2>)
	                              : (tf32 ? gemm_bf16_nt_2sm_kernel<true, 1> : gemm_bf16_nt_2sm_kernel<false, 1>);
	const size_t smem2 = pair_smem_bytes(wide ? 2 : 1);
	kern::ensure_smem(pair_kernel, static_cast<int>(smem2));
	cudaLaunchConfig_t cfg{};
	cudaLaunchAttribute attr[1];
	attr[0].id = cudaLaunchAttributeClusterDimension;
	attr[0].val.clusterDim.x = 2;
	attr[0].val.clusterDim.y = 1;
	attr[0].val.clusterDim.z = 1;
	cfg.blockDim = dim3(NUM_THREADS);
	cfg.dynamicSmemBytes = smem2;
	cfg.stream = s;
	cfg.attrs = attr;
	cfg.numAttrs = 1;
	static int max_clusters_by_kind[4] = {0, 0, 0, 0};
	int& max_clusters = max_clusters_by_kind[(tf32 ? 1 : 0) + (wide ? 2 : 0)];
	if(max_clusters == 0) {
		cfg.gridDim = dim3(static_cast<unsigned>(sms & ~1));
		int n_cl = 0;
		if(cudaOccupancyMaxActiveClusters(&n_cl, pair_kernel, &cfg) != cudaSuccess || n_cl <= 0) n_cl = sms / 2;
		cudaGetLastError();
		max_clusters = n_cl;
		if(const char* e = std::getenv("MTB_GEMM_CLUSTERS")) max_clusters = std::max(1, std::atoi(e));
		if(std::getenv("MTB_GEMM_VERBOSE")) std::fprintf(stderr, "[gemm] max active clusters %d (occupancy query %d)\n", max_clusters, n_cl);
	}
	const int units = ((p.m_blocks + 1) / 2) * (wide ? (p.n_blocks + 1) / 2 : p.n_blocks);
	cfg.gridDim = dim3(static_cast<unsigned>(2 * std::min(units, max_clusters)));

	if(cudaLaunchKernelEx(&cfg, pair_kernel, ma, mb, p) != cudaSuccess) return 1;
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// ---- TF32 operand preparation ----------------------------------------------------------------
//
// kind::tf32 reads only the top 19 bits of each f32 operand, i.e. it truncates the mantissa to
// 10 bits; on same-signed data the truncation error is one-sided and a K-long dot product
// inherits a bias of about -2^-11 (measured -7e-4 relative at 32768^3). The operands are
// therefore rounded to nearest-even TF32 once per launch into packed scratch (K-major, row pitch
// a multiple of 4 elements), so the MMA sees unbiased operands: 2 reads + 2 writes of the
// operand bytes (about 2.6 ms at 32768^3 against a 110 ms contraction). The reference-id
// `matmul` (B row-major, K x N) is transposed in the same pass.

__device__ __forceinline__ float tf32_rne(float x) {
	uint32_t u = __float_as_uint(x);
	if((u & 0x7f800000u) == 0x7f800000u) return x; // inf / nan
	u += 0xfffu + ((u >> 13) & 1u);
	return __uint_as_float(u & 0xffffe000u);
}

// dst[r][c] = rne(src[r][c]) for r < rows, c < cols; gridDim.y walks rows
__global__ void round_rows_tf32_k(const float* __restrict__ src, int64_t ld_src, float* __restrict__ dst, int64_t ld_dst, int64_t rows, int64_t cols) {
	for(int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
		const float* sr = src + r * ld_src;
		float* dr = dst + r * ld_dst;
		for(int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols; c += static_cast<int64_t>(gridDim.x) * blockDim.x)
			dr[c] = tf32_rne(__ldg(sr + c));
	}
}

// dst[j][l] = rne(src[l][j]) (src: k x n row-major with pitch ld_src; dst: n x k, pitch ld_dst)
__global__ void transpose_round_tf32_k(const float* __restrict__ src, int64_t ld_src, float* __restrict__ dst, int64_t ld_dst, int64_t k, int64_t n) {
	__shared__ float tile[32][33];
	const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32, l0 = static_cast<int64_t>(blockIdx.y) * 32;
	for(int y = threadIdx.y; y < 32; y += blockDim.y) {
		const int64_t l = l0 + y, j = j0 + threadIdx.x;
		tile[y][threadIdx.x] = (l < k && j < n) ? tf32_rne(__ldg(src + l * ld_src + j)) : 0.0f;
	}
	__syncthreads();
	for(int y = threadIdx.y; y < 32; y += blockDim.y) {
		const int64_t j = j0 + y, l = l0 + threadIdx.x;
		if(j < n && l < k) dst[j * ld_dst + l] = tile[threadIdx.x][y];
	}
}

// scratch for prepared operands: stream-ordered allocations from the device's default pool,
// which keeps up to 32 GiB cached between launches instead of returning it at every sync
void* scratch_alloc(size_t bytes, cudaStream_t s) {
	static bool raised[64] = {};
	int dev = 0;
	cudaGetDevice(&dev);
	if(dev < 64 && !raised[dev]) {
		cudaMemPool_t pool;
		if(cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
			uint64_t thr = 32ull << 30;
			cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
		}
		raised[dev] = true;
	}
	void* p = nullptr;
	if(cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
	return p;
}

bool tf32_truncate() {
	static const bool on = std::getenv("MTB_TF32_TRUNCATE") != nullptr;
	return on;
}

int64_t pad4(int64_t k) { return (k + 3) / 4 * 4; }

// 16-byte form: every row start 16-byte aligned, cols a multiple of 4; each thread moves four
// float4 per row (independent loads in flight), CTAs stride over rows
__global__ void round_rows_tf32_v4_k(const float4* __restrict__ src, int64_t ld4_src, float4* __restrict__ dst, int64_t ld4_dst, int64_t rows, int64_t cols4) {
	for(int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
		const float4* sr = src + r * ld4_src;
		float4* dr = dst + r * ld4_dst;
		for(int64_t c0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * 4 + threadIdx.x; c0 < cols4; c0 += static_cast<int64_t>(gridDim.x) * blockDim.x * 4) {
			float4 v[4];
#pragma unroll
			for(int u = 0; u < 4; ++u)
				if(c0 + u * blockDim.x < cols4) v[u] = __ldcs(sr + c0 + u * blockDim.x);
#pragma unroll
			for(int u = 0; u < 4; ++u)
				if(c0 + u * blockDim.x < cols4) {
					const float4 t = v[u];
					dr[c0 + u * blockDim.x] = make_float4(tf32_rne(t.x), tf32_rne(t.y), tf32_rne(t.z), tf32_rne(t.w));
				}
		}
	}
}

void round_rows(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int64_t rows, int64_t cols, cudaStream_t s) {
	const bool v4 = cols % 4 == 0 && ld_src % 4 == 0 && ld_dst % 4 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0;
	if(v4) {
		const int64_t cols4 = cols / 4;
		const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((cols4 + 1023) / 1024, 64)));
		const unsigned gy = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(rows, 148 * 16 / gx + 1)));
		round_rows_tf32_v4_k<<<dim3(gx, gy), 256, 0, s>>>(reinterpret_cast<const float4*>(src), ld_src / 4, reinterpret_cast<float4*>(dst), ld_dst / 4, rows,
		    cols4);
		return;
	}
	const unsigned gx = static_cast<unsigned>(std::min<int64_t>((cols + 255) / 256, 64));
	const unsigned gy = static_cast<unsigned>(std::min<int64_t>(rows, 65535));
	round_rows_tf32_k<<<dim3(gx, gy), 256, 0, s>>>(src, ld_src, dst, ld_dst, rows, cols);
}

// C (rows r of A x cols of Bt) with both operands f32, rounded to TF32 first (unless
// MTB_TF32_TRUNCATE); `b_kn` true: b is K x N row-major (the reference `matmul` layout)
int run_gemm_tf32(const float* a, int64_t lda, const float* b, int64_t ldb, bool b_kn, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
    cudaStream_t s) {
	if(m <= 0 || n <= 0) return 0;
	if(k <= 0) return 5;
	if(tf32_truncate() && !b_kn) return run_gemm(a, m, lda, 0, b, n, ldb, 0, c, ldc, m, n, k, s, true);
	const int64_t kp = pad4(k);
	float* sa = static_cast<float*>(scratch_alloc(static_cast<size_t>((m + n) * kp) * 4, s));
	if(!sa) return 8;
	float* sb = sa + m * kp;
	round_rows(a, lda, sa, kp, m, k, s);
	if(b_kn) {
		const dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32));
		transpose_round_tf32_k<<<grid, dim3(32, 8), 0, s>>>(b, ldb, sb, kp, k, n);
	} else {
		round_rows(b, ldb, sb, kp, n, k, s);
	}
	const int rc = run_gemm(sa, m, kp, 0, sb, n, kp, 0, c, ldc, m, n, k, s, true);
	cudaFreeAsync(sa, s);
	return rc;
}

} // namespace tc

// the reference-id `matmul` (kernels.cpp:167-193: C = A x B, B row-major K x N) on the tensor
// cores: A rows and B columns of the superblock are rounded to TF32 (B transposed to K-major)
// and contracted by the tcgen05 kernel. Returns -1 when the views do not allow it (the caller
// falls back to the scalar reference-order kernel).
int matmul_tc_reference(const mt_launch_ctx* c, void* stream) {
	const int64_t m = c->scalars_int[0], n = c->scalars_int[1], k = c->scalars_int[2];
	const int64_t r0 = c->threads_lo[0], r1 = std::min(c->threads_hi[0], m);
	const int64_t c0 = c->threads_lo[1], c1 = std::min(c->threads_hi[1], n);
	if(r0 >= r1 || c0 >= c1) return 0;
	const mt_view& vc = c->views[3];
	const mt_view& va = c->views[4];
	const mt_view& vb = c->views[5];
	if(!vc.base || !va.base || !vb.base) return -1;
	if(vc.stride[1] != 1 || va.stride[1] != 1 || vb.stride[1] != 1) return -1;
	if(va.offset[1] > 0 || va.offset[1] + va.extent[1] < k || vb.offset[0] > 0 || vb.offset[0] + vb.extent[0] < k) return -1;
	if(r0 < va.offset[0] || r1 > va.offset[0] + va.extent[0] || c0 < vb.offset[1] || c1 > vb.offset[1] + vb.extent[1]) return -1;
	const float* a = static_cast<const float*>(va.base) + (r0 - va.offset[0]) * va.stride[0] - va.offset[1];
	const float* b = static_cast<const float*>(vb.base) - vb.offset[0] * vb.stride[0] + (c0 - vb.offset[1]);
	float* cp = static_cast<float*>(vc.base) + (r0 - vc.offset[0]) * vc.stride[0] + (c0 - vc.offset[1]);
	return tc::run_gemm_tf32(a, va.stride[0], b, vb.stride[0], true, cp, vc.stride[0], r1 - r0, c1 - c0, k, static_cast<cudaStream_t>(stream));
}

static int launch_matmul_nt(const mt_launch_ctx* c, void* stream, bool tf32) {
	const int64_t m = c->scalars_int[0], n = c->scalars_int[1], k = c->scalars_int[2];
	const int64_t r0 = c->threads_lo[0], r1 = std::min(c->threads_hi[0], m);
	const int64_t c0 = c->threads_lo[1], c1 = std::min(c->threads_hi[1], n);
	if(r0 >= r1 || c0 >= c1) return 0;
	const mt_view& vc = c->views[3];
	const mt_view& va = c->views[4];
	const mt_view& vb = c->views[5];
	if(!vc.base || !va.base || !vb.base) return 2;
	if(va.offset[1] != 0 || vb.offset[1] != 0 || va.extent[1] < k || vb.extent[1] < k) return 3; // whole K rows staged
	float* cp = static_cast<float*>(vc.base) + (r0 - vc.offset[0]) * vc.stride[0] + (c0 - vc.offset[1]) * vc.stride[1];
	if(tf32) {
		const float* a = static_cast<const float*>(va.base) + (r0 - va.offset[0]) * va.stride[0];
		const float* b = static_cast<const float*>(vb.base) + (c0 - vb.offset[0]) * vb.stride[0];
		return tc::run_gemm_tf32(a, va.stride[0], b, vb.stride[0], false, cp, vc.stride[0], r1 - r0, c1 - c0, k, static_cast<cudaStream_t>(stream));
	}
	return tc::run_gemm(va.base, va.extent[0], va.stride[0], r0 - va.offset[0], vb.base, vb.extent[0], vb.stride[0], c0 - vb.offset[0], cp, vc.stride[0],
	    r1 - r0, c1 - c0, k, static_cast<cudaStream_t>(stream), tf32);
}

int launch_matmul_nt_bf16(const mt_launch_ctx* c, void* stream) { return launch_matmul_nt(c, stream, false); }
int launch_matmul_nt_tf32(const mt_launch_ctx* c, void* stream) { return launch_matmul_nt(c, stream, true); }

void register_matmul_kernels(kernel_table& t) {
	t.add({"matmul_nt_bf16",
	    {param_sig{"m", false, dtype::i64, 0, false}, param_sig{"n", false, dtype::i64, 0, false}, param_sig{"k", false, dtype::i64, 0, false},
	        param_sig{"C", true, dtype::f32, 2, true}, param_sig{"A", true, dtype::bf16, 2, false}, param_sig{"Bt", true, dtype::bf16, 2, false}},
	    launch_matmul_nt_bf16});
	// the fp32 form of C3 on the tensor cores: f32 operands multiplied as TF32, f32 accumulation
	t.add({"matmul_nt_tf32",
	    {param_sig{"m", false, dtype::i64, 0, false}, param_sig{"n", false, dtype::i64, 0, false}, param_sig{"k", false, dtype::i64, 0, false},
	        param_sig{"C", true, dtype::f32, 2, true}, param_sig{"A", true, dtype::f32, 2, false}, param_sig{"Bt", true, dtype::f32, 2, false}},
	    launch_matmul_nt_tf32});
}

} // namespace mtb

// direct entry for tests and the bench's contraction line (device pointers, row-major)
extern "C" int mt_gemm_bf16_nt(const void* a, const void* bt, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream) {
	return mtb::tc::run_gemm(a, m, lda, 0, bt, n, ldb, 0, c, ldc, m, n, k, static_cast<cudaStream_t>(stream));
}

extern "C" int mt_gemm_tf32_nt(const float* a, const float* bt, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream) {
	return mtb::tc::run_gemm_tf32(a, lda, bt, ldb, false, c, ldc, m, n, k, static_cast<cudaStream_t>(stream));
}

// C = A x B with B row-major (K x N): the reference `matmul` layout on the tensor cores
extern "C" int mt_gemm_tf32_nn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream) {
	return mtb::tc::run_gemm_tf32(a, lda, b, ldb, true, c, ldc, m, n, k, static_cast<cudaStream_t>(stream));
}

extern "C" uint64_t mt_tensor_core_launches(void) { return mtb::tc::g_tc_launches.load(); }
