// Reduce-annotated kernels: histogram and int32 k-means (BASELINE config C4).
//
// Both accumulate into the superblock's identity-filled reduce partial (planner.cpp:298-309);
// the planner's reduce tree then combines partials across devices and workers. Integer sums
// wrap exactly like the reference's (runtime.cpp:481-494), so the atomics' arbitrary order
// is invisible: results are bit-exact against the CPU oracle (oracle/ref_shim.cpp).
//
// histogram: HBM-bound streaming read of 4 B per element; counts are privatised in shared
// memory (u32, one bank-spread copy per CTA) and flushed once per CTA with 64-bit atomics.
// kmeans_assign_i32: centroids staged in shared memory, one point per thread, distances in
// int64 (the reference computes in int64), strict '<' so ties go to the lowest centroid.
// kmeans_update_i32: per-CTA shared-memory sums/counts, flushed with 64-bit atomics.
#include "../executor.hpp"
#include "common.cuh"

namespace mtb {
namespace kern {

constexpr int kHistSmemBins = 16384; // 64 KB of u32 counters

__global__ void histogram_smem_kernel(const int32_t* x, int64_t lo, int64_t n_local, int64_t bins, unsigned long long* hist) {
	extern __shared__ uint32_t cnt[];
	for(int64_t b = threadIdx.x; b < bins; b += blockDim.x) cnt[b] = 0;
	__syncthreads();
	const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
	// x is 16B-aligned at `lo` when the host picked this path; vector body + scalar tail
	const int64_t nvec = n_local / 4;
	const int4* xv = reinterpret_cast<const int4*>(x);
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nvec; t += stride) {
		const int4 v = __ldcs(xv + t);
		if(static_cast<uint64_t>(v.x) < static_cast<uint64_t>(bins)) atomicAdd(&cnt[v.x], 1u);
		if(static_cast<uint64_t>(v.y) < static_cast<uint64_t>(bins)) atomicAdd(&cnt[v.y], 1u);
		if(static_cast<uint64_t>(v.z) < static_cast<uint64_t>(bins)) atomicAdd(&cnt[v.z], 1u);
		if(static_cast<uint64_t>(v.w) < static_cast<uint64_t>(bins)) atomicAdd(&cnt[v.w], 1u);
	}
	for(int64_t t = nvec * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_local; t += stride) {
		const int32_t v = x[t];
		if(static_cast<uint64_t>(v) < static_cast<uint64_t>(bins)) atomicAdd(&cnt[v], 1u);
	}
	__syncthreads();
	for(int64_t b = threadIdx.x; b < bins; b += blockDim.x)
		if(cnt[b]) atomicAdd(hist + b, static_cast<unsigned long long>(cnt[b]));
	(void)lo;
}

__global__ void histogram_global_kernel(const int32_t* x, int64_t n_local, int64_t bins, unsigned long long* hist) {
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n_local; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int32_t v = x[t];
		if(static_cast<uint64_t>(v) < static_cast<uint64_t>(bins)) atomicAdd(hist + v, 1ull);
	}
}

constexpr int kKmMaxSmem = 48 * 1024;

__global__ void kmeans_assign_i32_kernel(range r, int64_t k, int64_t d, dview assign, dview points, dview cents) {
	extern __shared__ int32_t cs[]; // k*d centroids, row-major
	for(int64_t e = threadIdx.x; e < k * d; e += blockDim.x) cs[e] = *at2<int32_t>(cents, e / d, e % d);
	__syncthreads();
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < r.total; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int64_t i = r.lo[0] + t;
		int32_t p[16];
		const int dd = static_cast<int>(d);
		for(int q = 0; q < dd && q < 16; ++q) p[q] = *at2<int32_t>(points, i, q);
		int64_t best = 0, best_dist = INT64_MAX;
		for(int64_t c = 0; c < k; ++c) {
			const int32_t* cc = cs + c * d;
			int64_t dist = 0;
			if(dd <= 16) {
#pragma unroll
				for(int q = 0; q < 16; ++q) {
					if(q < dd) {
						const int64_t diff = static_cast<int64_t>(p[q]) - cc[q];
						dist += diff * diff;
					}
				}
			} else {
				for(int64_t q = 0; q < d; ++q) {
					const int64_t diff = static_cast<int64_t>(*at2<int32_t>(points, i, q)) - cc[q];
					dist += diff * diff;
				}
			}
			if(dist < best_dist) {
				best_dist = dist;
				best = c;
			}
		}
		*at1<int32_t>(assign, i) = static_cast<int32_t>(best);
	}
}

// centroid table too large for shared memory: read it through L1/L2
__global__ void kmeans_assign_i32_global_kernel(range r, int64_t k, int64_t d, dview assign, dview points, dview cents) {
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < r.total; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int64_t i = r.lo[0] + t;
		int64_t best = 0, best_dist = INT64_MAX;
		for(int64_t c = 0; c < k; ++c) {
			int64_t dist = 0;
			for(int64_t q = 0; q < d; ++q) {
				const int64_t diff = static_cast<int64_t>(*at2<int32_t>(points, i, q)) - *at2<int32_t>(cents, c, q);
				dist += diff * diff;
			}
			if(dist < best_dist) {
				best_dist = dist;
				best = c;
			}
		}
		*at1<int32_t>(assign, i) = static_cast<int32_t>(best);
	}
}

__global__ void kmeans_update_i32_kernel(range r, int64_t k, int64_t d, dview points, dview assign, dview sums, dview counts, int use_smem) {
	extern __shared__ unsigned long long acc[]; // k*d sums then k counts
	if(use_smem) {
		for(int64_t e = threadIdx.x; e < k * d + k; e += blockDim.x) acc[e] = 0;
		__syncthreads();
	}
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < r.total; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int64_t i = r.lo[0] + t;
		const int64_t c = *at1<int32_t>(assign, i);
		for(int64_t q = 0; q < d; ++q) {
			const auto v = static_cast<unsigned long long>(static_cast<int64_t>(*at2<int32_t>(points, i, q)));
			if(use_smem && c >= 0 && c < k)
				atomicAdd(acc + c * d + q, v);
			else
				atomicAdd(reinterpret_cast<unsigned long long*>(at2<int64_t>(sums, c, q)), v);
		}
		if(use_smem && c >= 0 && c < k)
			atomicAdd(acc + k * d + c, 1ull);
		else
			atomicAdd(reinterpret_cast<unsigned long long*>(at1<int64_t>(counts, c)), 1ull);
	}
	if(!use_smem) return;
	__syncthreads();
	for(int64_t e = threadIdx.x; e < k * d; e += blockDim.x)
		if(acc[e]) atomicAdd(reinterpret_cast<unsigned long long*>(at2<int64_t>(sums, e / d, e % d)), acc[e]);
	for(int64_t c = threadIdx.x; c < k; c += blockDim.x)
		if(acc[k * d + c]) atomicAdd(reinterpret_cast<unsigned long long*>(at1<int64_t>(counts, c)), acc[k * d + c]);
}

} // namespace kern

int launch_histogram(const mt_launch_ctx* c, void* stream) {
	using namespace kern;
	const int64_t n = c->scalars_int[0], bins = c->scalars_int[1];
	const int64_t lo = c->threads_lo[0], hi = std::min(c->threads_hi[0], n);
	if(lo >= hi || bins <= 0) return 0;
	const mt_view& vx = c->views[2];
	const mt_view& vh = c->views[3];
	// every bin a value can hit must lie inside the bound partial (the CPU body's
	// bounds-checked view would throw; the GPU path refuses to launch)
	if(vh.offset[0] > 0 || vh.offset[0] + vh.extent[0] < bins) return 4;
	const int32_t* x = static_cast<const int32_t*>(vx.base) + (lo - vx.offset[0]);
	auto* hist = static_cast<unsigned long long*>(vh.base) - vh.offset[0];
	const int64_t n_local = hi - lo;
	const auto s = static_cast<cudaStream_t>(stream);
	if(bins <= kHistSmemBins && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
		const size_t smem = static_cast<size_t>(bins) * sizeof(uint32_t);
		ensure_smem(histogram_smem_kernel, kHistSmemBins * 4);
		int64_t blocks = (n_local / 4 + 511) / 512;
		blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 4));
		histogram_smem_kernel<<<static_cast<unsigned>(blocks), 512, smem, s>>>(x, lo, n_local, bins, hist);
	} else {
		histogram_global_kernel<<<grid_1d(n_local, 256), 256, 0, s>>>(x, n_local, bins, hist);
	}
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_kmeans_assign_i32(const mt_launch_ctx* c, void* stream) {
	using namespace kern;
	const int64_t lim[3] = {c->scalars_int[0], 0, 0};
	const range r = clip_range(c, lim);
	if(r.total <= 0) return 0;
	const int64_t k = c->scalars_int[1], d = c->scalars_int[2];
	const auto s = static_cast<cudaStream_t>(stream);
	const size_t smem = static_cast<size_t>(k * d) * sizeof(int32_t);
	if(smem <= static_cast<size_t>(kKmMaxSmem) && d <= 16) {
		kmeans_assign_i32_kernel<<<grid_1d(r.total, 256), 256, smem, s>>>(r, k, d, make_view(c->views[3]), make_view(c->views[4]), make_view(c->views[5]));
	} else {
		kmeans_assign_i32_global_kernel<<<grid_1d(r.total, 256), 256, 0, s>>>(r, k, d, make_view(c->views[3]), make_view(c->views[4]), make_view(c->views[5]));
	}
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_kmeans_update_i32(const mt_launch_ctx* c, void* stream) {
	using namespace kern;
	const int64_t lim[3] = {c->scalars_int[0], 0, 0};
	const range r = clip_range(c, lim);
	if(r.total <= 0) return 0;
	const int64_t d = c->scalars_int[1];
	const mt_view& vs = c->views[4];
	const int64_t k = vs.extent[0];
	// shared-memory privatisation only when the partial starts at centroid 0 (whole table)
	const bool smem_ok = vs.offset[0] == 0 && vs.offset[1] == 0 && vs.extent[1] == d && static_cast<size_t>(k * d + k) * 8 <= 96 * 1024;
	const size_t smem = smem_ok ? static_cast<size_t>(k * d + k) * 8 : 0;
	ensure_smem(kmeans_update_i32_kernel, 96 * 1024);
	const unsigned blocks = std::min<unsigned>(grid_1d(r.total, 256), 148 * 2);
	kmeans_update_i32_kernel<<<blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(r, k, d, make_view(c->views[2]), make_view(c->views[3]),
	    make_view(c->views[4]), make_view(c->views[5]), smem_ok ? 1 : 0);
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

} // namespace mtb
