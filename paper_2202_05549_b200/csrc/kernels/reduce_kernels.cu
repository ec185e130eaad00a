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

#include <climits>
#include <cstdlib>

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

// Up to ~110K bins: two u16 counters per u32 shared word (65536 bins = 128 KB). The word only
// ever receives additions, and every wrap is accounted from the old value its own atomic
// returned, so no thread can misread a transient state: a low half that wraps adds 65536 to its
// bin in the global partial and -1 to the high bin (its carry landed in the high half, and the
// end-of-kernel flush will count it), and if that carry also wrapped the high half, 65536 to the
// high bin; a high half that wraps adds 65536 to its bin. (Taking the carry back with a shared
// atomicSub instead would leave a window in which a concurrent high-bin increment reads the
// carried value and misses its own wrap.) With uniformly spread values the kernel is bound by
// shared-memory atomic throughput under random bank conflicts, not by HBM.
constexpr int kHistPairMaxBins = 110000;
constexpr int kHistQuadMaxBins = 220000; // u8 counters: 55000 words = 220 KB of shared memory

__global__ void __launch_bounds__(1024, 1) histogram_pair_kernel(const int32_t* x, int64_t n_local, int bins, unsigned long long* hist) {
	extern __shared__ uint32_t w[];
	const int words = (bins + 1) / 2;
	for(int b = threadIdx.x; b < words; b += blockDim.x) w[b] = 0;
	__syncthreads();
	const auto fixup = [&](int32_t v, uint32_t old) {
		const uint32_t sh = (v & 1) * 16;
		if(((old >> sh) & 0xFFFFu) == 0xFFFFu) { // this add wrapped its half (rare)
			atomicAdd(hist + v, 65536ull);
			if(sh == 0 && v + 1 < bins) {
				atomicAdd(hist + v + 1, ~0ull); // -1: the carry is counted by the flush of the high half
				if((old >> 16) == 0xFFFFu) atomicAdd(hist + v + 1, 65536ull); // and it wrapped the high half
			}
		}
	};
	const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
	const int64_t nvec = n_local / 4;
	const int4* xv = reinterpret_cast<const int4*>(x);
	// one CTA of 32 warps per SM: four 16-byte loads in flight per thread keep ~64 KB per SM
	// outstanding, enough to cover HBM latency at full bandwidth
	constexpr int U = 4;
	int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
	for(; t + (U - 1) * stride < nvec; t += U * stride) {
		int32_t v[4 * U];
#pragma unroll
		for(int u = 0; u < U; ++u) {
			const int4 q = __ldcs(xv + t + u * stride);
			v[4 * u] = q.x;
			v[4 * u + 1] = q.y;
			v[4 * u + 2] = q.z;
			v[4 * u + 3] = q.w;
		}
#pragma unroll
		for(int e = 0; e < 4 * U; ++e)
			if(static_cast<uint32_t>(v[e]) < static_cast<uint32_t>(bins)) fixup(v[e], atomicAdd(&w[v[e] >> 1], 1u << ((v[e] & 1) * 16)));
	}
	for(; t < nvec; t += stride) {
		const int4 q = __ldcs(xv + t);
		const int32_t v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
		for(int e = 0; e < 4; ++e)
			if(static_cast<uint32_t>(v[e]) < static_cast<uint32_t>(bins)) fixup(v[e], atomicAdd(&w[v[e] >> 1], 1u << ((v[e] & 1) * 16)));
	}
	for(int64_t e = nvec * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_local; e += stride) {
		const int32_t v = x[e];
		if(static_cast<uint32_t>(v) < static_cast<uint32_t>(bins)) fixup(v, atomicAdd(&w[v >> 1], 1u << ((v & 1) * 16)));
	}
	__syncthreads();
	for(int b = threadIdx.x; b < words; b += blockDim.x) {
		const uint32_t v = w[b];
		if(v & 0xFFFFu) atomicAdd(hist + 2 * b, static_cast<unsigned long long>(v & 0xFFFFu));
		if((v >> 16) && 2 * b + 1 < bins) atomicAdd(hist + 2 * b + 1, static_cast<unsigned long long>(v >> 16));
	}
}

// Four u8 counters per u32 shared word (65536 bins = 64 KB), so two 1024-thread CTAs share an
// SM. As with the u16 kernel the word only receives additions and every wrap is booked from the
// old value the thread's own atomic returned: adding 1 to byte b of `old` changes bytes b..3 by
// the carry chain, and each bin k in that chain gets (its true increment) - (its stored change)
// added to the global partial, which is 0 except when a byte wraps.
template <int U>
__global__ void __launch_bounds__(1024, 2) histogram_quad_kernel(const int32_t* x, int64_t n_local, int bins, unsigned long long* hist) {
	extern __shared__ uint32_t w[];
	const int words = (bins + 3) / 4;
	for(int b = threadIdx.x; b < words; b += blockDim.x) w[b] = 0;
	__syncthreads();
	const auto add = [&](int32_t v) {
		if(static_cast<uint32_t>(v) >= static_cast<uint32_t>(bins)) return;
		const uint32_t sh = (v & 3) * 8;
		const uint32_t old = atomicAdd(&w[v >> 2], 1u << sh);
		if(((old >> sh) & 0xFFu) == 0xFFu) { // this add wrapped its byte (rare): book the carry chain
			const uint32_t nw = old + (1u << sh);
			for(int kb = v & 3; kb < 4; ++kb) {
				const int bin = (v & ~3) + kb;
				const int delta = static_cast<int>((nw >> (8 * kb)) & 0xFFu) - static_cast<int>((old >> (8 * kb)) & 0xFFu);
				const long long fix = (kb == (v & 3) ? 1 : 0) - delta;
				if(fix != 0 && bin < bins) atomicAdd(hist + bin, static_cast<unsigned long long>(fix));
				if(delta != -255) break; // the carry stops at the first byte that did not wrap
			}
		}
	};
	// the common case without per-element branches: one range test per four values (unsigned
	// max), four atomics, their wrap tests folded into one predicate (byte k of `old` is 0xFF iff
	// ~old has no bit of the byte's mask), and one rarely taken branch that books the wraps
	const auto add4 = [&](const int4 q) {
		const uint32_t v[4] = {static_cast<uint32_t>(q.x), static_cast<uint32_t>(q.y), static_cast<uint32_t>(q.z), static_cast<uint32_t>(q.w)};
		if(max(max(v[0], v[1]), max(v[2], v[3])) >= static_cast<uint32_t>(bins)) {
			add(q.x);
			add(q.y);
			add(q.z);
			add(q.w);
			return;
		}
		uint32_t old[4];
		bool wrap = false;
#pragma unroll
		for(int e = 0; e < 4; ++e) {
			const uint32_t inc = 1u << ((v[e] & 3u) << 3);
			old[e] = atomicAdd(&w[v[e] >> 2], inc);
			wrap |= (~old[e] & (inc * 0xFFu)) == 0;
		}
		if(__builtin_expect(wrap, 0)) {
#pragma unroll
			for(int e = 0; e < 4; ++e) {
				const uint32_t sh = (v[e] & 3u) * 8;
				if(((old[e] >> sh) & 0xFFu) != 0xFFu) continue;
				const uint32_t nw = old[e] + (1u << sh);
				for(int kb = v[e] & 3; kb < 4; ++kb) {
					const int bin = static_cast<int>(v[e] & ~3u) + kb;
					const int delta = static_cast<int>((nw >> (8 * kb)) & 0xFFu) - static_cast<int>((old[e] >> (8 * kb)) & 0xFFu);
					const long long fix = (kb == static_cast<int>(v[e] & 3) ? 1 : 0) - delta;
					if(fix != 0 && bin < bins) atomicAdd(hist + bin, static_cast<unsigned long long>(fix));
					if(delta != -255) break;
				}
			}
		}
	};
	const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
	const int64_t nvec = n_local / 4;
	const int4* xv = reinterpret_cast<const int4*>(x);
	int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
	for(; t + (U - 1) * stride < nvec; t += U * stride) {
		int4 q[U];
#pragma unroll
		for(int u = 0; u < U; ++u) q[u] = __ldcs(xv + t + u * stride);
#pragma unroll
		for(int u = 0; u < U; ++u) add4(q[u]);
	}
	for(; t < nvec; t += stride) {
		const int4 q = __ldcs(xv + t);
		add(q.x);
		add(q.y);
		add(q.z);
		add(q.w);
	}
	for(int64_t e = nvec * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_local; e += stride) add(x[e]);
	__syncthreads();
	for(int b = threadIdx.x; b < words; b += blockDim.x) {
		const uint32_t v = w[b];
#pragma unroll
		for(int kb = 0; kb < 4; ++kb) {
			const uint32_t c = (v >> (8 * kb)) & 0xFFu;
			if(c && 4 * b + kb < bins) atomicAdd(hist + 4 * b + kb, static_cast<unsigned long long>(c));
		}
	}
}

// k-means assignment, fast paths. FP32 tier: when sum_q |x_q| * max|c| <= 2^24 for a thread's
// points (checked on the fly; BASELINE C4 data, values < 1000, qualifies), x.c is accumulated
// with FFMA — every partial sum is an integer below 2^24, so each FFMA is exact — converted to
// int, and the argmin is taken over the exact integer criterion |c|^2 - 2 x.c (|x|^2 is common to
// all centroids of a point). The FP32 pipe issues these faster than IMAD (14 % on C4).
// u32 tier: when every |coordinate| < 8192 (checked on the fly: the
// block checks its centroid table, each thread its points) the squared distance over d <= 16
// dimensions lies in [0, 2^32), so it is computed exactly in wrapping u32 arithmetic as
// |x|^2 + |c|^2 - 2 x.c: the table holds -2c (and |c|^2 per row), so each (point, centroid)
// costs 16 IMADs on the FMA pipe plus one IADD3 / compare / select on the ALU pipe (the
// direct (x-c)^2 form costs 32 FMA-pipe ops, because ptxas moves the subtractions there too).
// The exact distance makes the argmin (first minimum, strict '<') identical to the int64
// reference (kernels.cpp:283-292). Four points per thread share each broadcast centroid load.
// Points outside the range take the int64 path.
//
// Centred FP32 tier (tried first). The argmin is translation invariant, so points and centroids
// are moved by a per-dimension offset o (the midpoint of the centroid table's range) and the
// criterion becomes: maximise v = x'.c' - |c'|^2 / 2 (x' = x - o, c' = c - o), the first maximum
// being the first minimum of the squared distance. One FFMA chain per (point, centroid) starts at
// -|c'|^2/2 and adds the 16 products: every partial sum is a half-integer of magnitude below
// sum|x'_q| max|c'| + max|c'|^2/2, checked < 2^23 per point, so each FFMA is exact and the
// comparison needs no conversion: 16 FFMA + FSETP + 2 SEL per pair (the uncentred tier needs a
// second chain's FADD, an F2I and integer compare on top). BASELINE C4 data (values < 1000)
// qualifies after centring (|x'|, |c'| ~ 500).
template <int kKmPts, int kMinBlocks, int kCU = 1>
__global__ void __launch_bounds__(256, kMinBlocks) kmeans_assign_fast_kernel(const int32_t* __restrict__ points, int64_t pld, int64_t n_local, int k, int d,
    const int32_t* __restrict__ cents, int64_t cld, int32_t* __restrict__ assign) {
	// k rows of 16 values -2c (padded to 16 columns), k |c|^2, k rows of c as f32, k rows of c' as
	// f32, k values -|c'|^2/2
	extern __shared__ int4 cs4[];
	int32_t* cs = reinterpret_cast<int32_t*>(cs4);
	uint32_t* cn = reinterpret_cast<uint32_t*>(cs + k * 16);
	float* cf = reinterpret_cast<float*>(cn + ((k + 3) / 4) * 4);
	float* cz = cf + k * 16;
	float* hneg = cz + k * 16;
	__shared__ int cmax;        // max |c| over the table (f32 tier bound)
	__shared__ int omin[16], omax[16], off[16];
	__shared__ int czmax;       // max |c'|
	__shared__ unsigned long long hmax; // max |c'|^2
	if(threadIdx.x == 0) {
		cmax = 0;
		czmax = 0;
		hmax = 0;
	}
	if(threadIdx.x < 16) {
		omin[threadIdx.x] = INT_MAX;
		omax[threadIdx.x] = INT_MIN;
	}
	__syncthreads();
	int big = 0, mymax = 0;
	for(int e = threadIdx.x; e < k * 16; e += blockDim.x) {
		const int c = e / 16, q = e % 16;
		const int32_t v = q < d ? cents[static_cast<int64_t>(c) * cld + q] : 0;
		const bool b = (v >= 8192 || v <= -8192);
		big |= b;
		cs[e] = b ? 0 : -2 * v;
		cf[e] = b ? 0.f : static_cast<float>(v);
		mymax = max(mymax, b ? 8192 : abs(v));
		atomicMin(&omin[q], v);
		atomicMax(&omax[q], v);
	}
	atomicMax(&cmax, mymax);
	const int cent_big = __syncthreads_or(big);
	const uint64_t mc = static_cast<uint64_t>(cmax);
	if(threadIdx.x < 16) off[threadIdx.x] = cent_big ? 0 : (omin[threadIdx.x] + omax[threadIdx.x]) >> 1;
	for(int c = threadIdx.x; c < k; c += blockDim.x) {
		uint32_t s = 0;
		for(int q = 0; q < 16; ++q) {
			const uint32_t h = static_cast<uint32_t>(cs[c * 16 + q] / -2);
			s += h * h;
		}
		cn[c] = s;
	}
	__syncthreads();
	int myz = 0;
	for(int e = threadIdx.x; e < k * 16; e += blockDim.x) {
		const int q = e % 16;
		const int z = q < d && !cent_big ? static_cast<int>(cf[e]) - off[q] : 0;
		cz[e] = static_cast<float>(z);
		myz = max(myz, abs(z));
	}
	atomicMax(&czmax, myz);
	__syncthreads();
	for(int c = threadIdx.x; c < k; c += blockDim.x) {
		unsigned long long s = 0;
		for(int q = 0; q < 16; ++q) {
			const long long z = static_cast<long long>(cz[c * 16 + q]);
			s += static_cast<unsigned long long>(z * z);
		}
		hneg[c] = -0.5f * static_cast<float>(s); // exact whenever the tier's bound holds (s < 2^24)
		atomicMax(&hmax, s);
	}
	__syncthreads();
	const uint64_t zc = static_cast<uint64_t>(czmax);
	const uint64_t hm = hmax;
	const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * kKmPts;
	for(int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kKmPts; base < n_local; base += stride) {
		int bi[kKmPts];
		// centred tier first: its bound, sum|x'_q| max|c'| + max|c'|^2/2 < 2^23 for every point of
		// the thread (half-integers below 2^23 are exact floats); the point registers of the other
		// tiers are loaded only when it fails, so the two register sets are never live together
		bool zok = !cent_big && hm < (uint64_t{1} << 24);
		float pz[kKmPts][16];
#pragma unroll
		for(int j = 0; j < kKmPts; ++j) {
			const int64_t i = base + j;
			uint32_t sz = 0;
#pragma unroll
			for(int q = 0; q < 16; ++q) {
				const int32_t v = (i < n_local && q < d) ? points[i * pld + q] : 0;
				const bool in = v < 8192 && v > -8192;
				const int32_t z = in ? v - (q < d ? off[q] : 0) : 0;
				zok &= in;
				pz[j][q] = static_cast<float>(z);
				sz += static_cast<uint32_t>(abs(z));
			}
			zok &= static_cast<uint64_t>(sz) * zc * 2 + hm < (uint64_t{1} << 24);
		}
		if(zok) {
			float bv[kKmPts];
#pragma unroll
			for(int j = 0; j < kKmPts; ++j) {
				bv[j] = -INFINITY;
				bi[j] = 0;
			}
			const float4* cz4 = reinterpret_cast<const float4*>(cz);
#pragma unroll kCU
			for(int c = 0; c < k; ++c) {
				float cv[16];
#pragma unroll
				for(int v4 = 0; v4 < 4; ++v4) {
					const float4 t = cz4[c * 4 + v4];
					cv[4 * v4] = t.x;
					cv[4 * v4 + 1] = t.y;
					cv[4 * v4 + 2] = t.z;
					cv[4 * v4 + 3] = t.w;
				}
				const float h = hneg[c];
#pragma unroll
				for(int j = 0; j < kKmPts; ++j) {
					float v = h;
#pragma unroll
					for(int q = 0; q < 16; ++q) v = fmaf(pz[j][q], cv[q], v);
					if(v > bv[j]) {
						bv[j] = v;
						bi[j] = c;
					}
				}
			}
#pragma unroll
			for(int j = 0; j < kKmPts; ++j)
				if(base + j < n_local) assign[base + j] = bi[j];
			continue;
		}
		uint32_t p[kKmPts][16];
		uint32_t xx[kKmPts];
		bool ok = !cent_big;
		bool f32ok = !cent_big;
#pragma unroll
		for(int j = 0; j < kKmPts; ++j) {
			const int64_t i = base + j;
			xx[j] = 0;
			uint32_t sx = 0;
#pragma unroll
			for(int q = 0; q < 16; ++q) {
				const int32_t v = (i < n_local && q < d) ? points[i * pld + q] : 0;
				p[j][q] = static_cast<uint32_t>(v);
				ok &= (v < 8192 && v > -8192);
				xx[j] += static_cast<uint32_t>(v) * static_cast<uint32_t>(v);
				sx += static_cast<uint32_t>(abs(v < 8192 && v > -8192 ? v : 8192));
			}
			// f32 tier: every partial sum of x.c is an integer of magnitude <= sum|x_q| max|c|;
			// below 2^24 each FFMA is exact
			f32ok &= static_cast<uint64_t>(sx) * mc <= (uint64_t{1} << 24);
		}
		uint32_t best[kKmPts];
#pragma unroll
		for(int j = 0; j < kKmPts; ++j) {
			best[j] = 0xFFFFFFFFu;
			bi[j] = 0;
		}
		if(ok && f32ok) {
			// x.c on the FP32 pipe (exact, see above), then the integer criterion |c|^2 - 2 x.c
			// (|x|^2 is common to all centroids of a point): same first minimum as the exact
			// squared distance
			float pf[kKmPts][16];
			int ib[kKmPts];
#pragma unroll
			for(int j = 0; j < kKmPts; ++j) {
				ib[j] = INT_MAX;
#pragma unroll
				for(int q = 0; q < 16; ++q) pf[j][q] = static_cast<float>(static_cast<int32_t>(p[j][q]));
			}
			const float4* cf4 = reinterpret_cast<const float4*>(cf);
#pragma unroll 1
			for(int c = 0; c < k; ++c) {
				float cv[16];
#pragma unroll
				for(int v4 = 0; v4 < 4; ++v4) {
					const float4 t = cf4[c * 4 + v4];
					cv[4 * v4] = t.x;
					cv[4 * v4 + 1] = t.y;
					cv[4 * v4 + 2] = t.z;
					cv[4 * v4 + 3] = t.w;
				}
				const int cc = static_cast<int>(cn[c]);
#pragma unroll
				for(int j = 0; j < kKmPts; ++j) {
					float m0 = 0.f, m1 = 0.f; // two independent chains (both partial sums exact)
#pragma unroll
					for(int q = 0; q < 16; q += 2) {
						m0 = fmaf(pf[j][q], cv[q], m0);
						m1 = fmaf(pf[j][q + 1], cv[q + 1], m1);
					}
					const float m = m0 + m1;
					const int crit = cc - 2 * __float2int_rn(m);
					if(crit < ib[j]) {
						ib[j] = crit;
						bi[j] = c;
					}
				}
			}
		} else if(ok) {
#pragma unroll 1
			for(int c = 0; c < k; ++c) {
				const int4* crow = cs4 + c * 4;
				uint32_t cv[16];
#pragma unroll
				for(int v4 = 0; v4 < 4; ++v4) {
					const int4 t = crow[v4];
					cv[4 * v4] = static_cast<uint32_t>(t.x);
					cv[4 * v4 + 1] = static_cast<uint32_t>(t.y);
					cv[4 * v4 + 2] = static_cast<uint32_t>(t.z);
					cv[4 * v4 + 3] = static_cast<uint32_t>(t.w);
				}
				const uint32_t cc = cn[c];
#pragma unroll
				for(int j = 0; j < kKmPts; ++j) {
					uint32_t m2 = 0; // -2 x.c (mod 2^32)
#pragma unroll
					for(int q = 0; q < 16; ++q) m2 += p[j][q] * cv[q];
					const uint32_t dist = xx[j] + cc + m2;
					if(dist < best[j]) {
						best[j] = dist;
						bi[j] = c;
					}
				}
			}
		} else {
			// exact int64 path (reference arithmetic, kernels.cpp:283-292)
#pragma unroll 1
			for(int j = 0; j < kKmPts; ++j) {
				int64_t b64 = INT64_MAX;
				const int64_t i = base + j;
				for(int c = 0; c < k; ++c) {
					int64_t dist = 0;
					for(int q = 0; q < d; ++q) {
						const int64_t df = static_cast<int64_t>(i < n_local ? points[i * pld + q] : 0) - cents[static_cast<int64_t>(c) * cld + q];
						dist += df * df;
					}
					if(dist < b64) {
						b64 = dist;
						bi[j] = c;
					}
				}
			}
		}
#pragma unroll
		for(int j = 0; j < kKmPts; ++j)
			if(base + j < n_local) assign[base + j] = bi[j];
	}
}

// k-means update: a warp takes 32 points. Lane l counts point l (one shared atomic for 32
// points), then the warp walks the 32 points in pairs, a half-warp per point and lane q adding
// coordinate q, so one instruction covers two points x 16 dimensions with a coalesced 128-byte
// load. Each half-warp owns its own copy of the per-CTA sum table, laid out so copy 0 lives in
// banks 0-15 and copy 1 in banks 16-31 (row c of copy h at word 32c + 16h): the two points of
// an instruction never collide in a bank. Each sum is an exact wrapping int64 held as signed
// i32 words plus one shared wrap counter touched only when an i32 add overflows (detected from
// the atomics' old values, checked once per group of 8), so a coordinate costs one shared
// atomic. Points whose assignment lies outside the partial (the reference's bounds-checked view
// would throw) and lanes past d go to a dummy row k / add 0, so the atomics need no predicates.
// Flushed once per CTA with 64-bit global atomics.
template <bool kContig>
__global__ void __launch_bounds__(512, 2) kmeans_update_fast_kernel(const int32_t* __restrict__ points, int64_t pld, const int32_t* __restrict__ assign,
    int64_t n_local, int k, int d, unsigned long long* sums, int64_t sld, unsigned long long* counts) {
	extern __shared__ uint32_t sm[];
	const int rows = k + 1;
	uint32_t* lo = sm;                // rows x 32 words (two 16-word copies)
	uint32_t* hi = sm + rows * 32;    // rows x 16 wrap counters
	uint32_t* cnt = sm + rows * 48;   // rows counts
	for(int e = threadIdx.x; e < rows * 49; e += blockDim.x) sm[e] = 0;
	__syncthreads();
	const int lane = threadIdx.x & 31;
	const int q = lane & 15;
	const int h = lane >> 4;
	const int qc = q < d ? q : 0;
	const int64_t step = kContig ? 16 : pld;
	const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
	const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
	for(int64_t i0 = warp * 32; i0 < n_local; i0 += warps * 32) {
		int cl;
		int32_t v[16];
		if(i0 + 32 <= n_local) {
			cl = __ldcs(assign + i0 + lane);
			const int32_t* pp = points + (i0 + h) * step + qc;
#pragma unroll
			for(int u = 0; u < 16; ++u) v[u] = __ldcs(pp + 2 * u * step);
		} else {
			cl = i0 + lane < n_local ? assign[i0 + lane] : k;
#pragma unroll
			for(int u = 0; u < 16; ++u) v[u] = i0 + 2 * u + h < n_local ? points[(i0 + 2 * u + h) * step + qc] : 0;
		}
		if(static_cast<uint32_t>(cl) >= static_cast<uint32_t>(k)) cl = k;
		atomicAdd(&cnt[cl], 1u);
#pragma unroll
		for(int g = 0; g < 16; g += 8) {
			uint32_t old[8], uv[8];
			int c[8];
			uint32_t ovf = 0;
#pragma unroll
			for(int u = 0; u < 8; ++u) {
				c[u] = __shfl_sync(0xFFFFFFFFu, cl, 2 * (g + u) + h);
				uv[u] = q < d ? static_cast<uint32_t>(v[g + u]) : 0u;
				old[u] = atomicAdd(&lo[c[u] * 32 + h * 16 + q], uv[u]);
				const uint32_t nw = old[u] + uv[u];
				ovf |= (old[u] ^ nw) & (uv[u] ^ nw);
			}
			if(static_cast<int32_t>(ovf) < 0) {
#pragma unroll
				for(int u = 0; u < 8; ++u) {
					const uint32_t nw = old[u] + uv[u];
					if(static_cast<int32_t>((old[u] ^ nw) & (uv[u] ^ nw)) < 0)
						atomicAdd(&hi[c[u] * 16 + q], static_cast<int32_t>(uv[u]) < 0 ? 0xFFFFFFFFu : 1u);
				}
			}
		}
	}
	__syncthreads();
	for(int e = threadIdx.x; e < k * 16; e += blockDim.x) {
		const int c = e / 16, qq = e % 16;
		if(qq >= d) continue;
		const int64_t v = static_cast<int64_t>(static_cast<int32_t>(lo[c * 32 + qq])) + static_cast<int64_t>(static_cast<int32_t>(lo[c * 32 + 16 + qq]))
		                  + static_cast<int64_t>(static_cast<uint64_t>(hi[e]) << 32);
		if(v) atomicAdd(sums + static_cast<int64_t>(c) * sld + qq, static_cast<unsigned long long>(v));
	}
	for(int c = threadIdx.x; c < k; c += blockDim.x)
		if(cnt[c]) atomicAdd(counts + c, static_cast<unsigned long long>(cnt[c]));
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
	} else if(bins <= kHistQuadMaxBins && reinterpret_cast<uintptr_t>(x) % 16 == 0 && !(std::getenv("MTB_HIST_QUAD") && std::atoi(std::getenv("MTB_HIST_QUAD")) == 0)) {
		// u8 counters: two CTAs per SM up to 110K bins (65536 bins: 2.67 vs 2.85 ms for the u16
		// single-CTA kernel), one CTA per SM up to 220K bins
		const size_t smem = static_cast<size_t>((bins + 3) / 4) * sizeof(uint32_t);
		static const int unroll = [] {
			const char* e = std::getenv("MTB_HIST_U"); // A/B runs: 16-byte loads in flight per thread, 2 (default) or 4
			return e && std::atoi(e) == 4 ? 4 : 2;
		}();
		const auto kern = unroll == 4 ? histogram_quad_kernel<4> : histogram_quad_kernel<2>;
		ensure_smem(kern, static_cast<int>(((kHistQuadMaxBins + 3) / 4) * 4));
		const int per_sm = bins <= kHistPairMaxBins ? 2 : 1;
		int64_t blocks = (n_local / 4 + 1023) / 1024;
		blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, per_sm * 148));
		kern<<<static_cast<unsigned>(blocks), 1024, smem, s>>>(x, n_local, static_cast<int>(bins), hist);
	} else if(bins <= kHistPairMaxBins && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
		const size_t smem = static_cast<size_t>((bins + 1) / 2) * sizeof(uint32_t);
		ensure_smem(histogram_pair_kernel, static_cast<int>(((kHistPairMaxBins + 1) / 2) * 4));
		int64_t blocks = (n_local / 4 + 1023) / 1024;
		blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148));
		histogram_pair_kernel<<<static_cast<unsigned>(blocks), 1024, smem, s>>>(x, n_local, static_cast<int>(bins), hist);
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
	const mt_view& va = c->views[3];
	const mt_view& vp = c->views[4];
	const mt_view& vc = c->views[5];
	const size_t fast_smem = static_cast<size_t>(k) * 16 * 4 * 3 + static_cast<size_t>((k + 3) / 4) * 4 * 4 + static_cast<size_t>(k) * 4;
	const bool fast = d >= 1 && d <= 16 && fast_smem <= 200 * 1024 && vp.stride[1] == 1 && vc.stride[1] == 1 && va.stride[0] == 1 && vc.offset[0] == 0
	                  && vc.offset[1] == 0 && vp.offset[1] == 0 && vc.extent[0] >= k;
	if(fast) {
		const int32_t* pts = static_cast<const int32_t*>(vp.base) + (r.lo[0] - vp.offset[0]) * vp.stride[0];
		int32_t* asg = static_cast<int32_t*>(va.base) + (r.lo[0] - va.offset[0]);
		const auto run = [&](auto kern, int pts_per_thread, int per_sm) {
			ensure_smem(kern, 200 * 1024);
			const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(static_cast<unsigned>((r.total + 256 * pts_per_thread - 1) / (256 * pts_per_thread)), 148 * per_sm));
			kern<<<blocks, 256, fast_smem, s>>>(pts, vp.stride[0], r.total, static_cast<int>(k), static_cast<int>(d), static_cast<const int32_t*>(vc.base),
			    vc.stride[0], asg);
		};
		// uncentred FP32 tier (round 1): 4x2 47.4 ms, 8x1 48.2, 6x1 50.4, 2x3 56.7 for 2e8 points;
		// the IMAD-only kernel took 55.1
		static const int variant = [] {
			const char* e = std::getenv("MTB_KM_VARIANT");
			return e ? std::atoi(e) : 0;
		}();
		// measured on 2e8 points (centred tier): 8 points x 1 CTA per SM with the centroid loop
		// unrolled twice 36.5 ms; 4 x 2 CTAs 39.2 (unrolled) / 41-42 (not); 8 x 1 not unrolled 42.8;
		// 6 x 1 40.7. MTB_KM_VARIANT selects the others for A/B runs
		switch(variant) {
		case 1: run(kmeans_assign_fast_kernel<8, 1>, 8, 1); break;
		case 2: run(kmeans_assign_fast_kernel<4, 2, 2>, 4, 2); break;
		case 4: run(kmeans_assign_fast_kernel<6, 1>, 6, 1); break;
		case 5: run(kmeans_assign_fast_kernel<4, 2>, 4, 2); break;
		default: run(kmeans_assign_fast_kernel<8, 1, 2>, 8, 1); break;
		}
		return cudaGetLastError() == cudaSuccess ? 0 : 1;
	}
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
	{
		const mt_view& vp = c->views[2];
		const mt_view& va = c->views[3];
		const mt_view& vn = c->views[5];
		const size_t smem = static_cast<size_t>(k + 1) * 49 * 4;
		if(d >= 1 && d <= 16 && vs.offset[0] == 0 && vs.offset[1] == 0 && vs.extent[1] == d && vn.offset[0] == 0 && vn.extent[0] == k && smem <= 200 * 1024
		    && vp.stride[1] == 1 && vp.offset[1] == 0 && va.stride[0] == 1) {
			const int32_t* pts = static_cast<const int32_t*>(vp.base) + (r.lo[0] - vp.offset[0]) * vp.stride[0];
			const int32_t* asg = static_cast<const int32_t*>(va.base) + (r.lo[0] - va.offset[0]);
			const unsigned blocks = std::max<unsigned>(1, std::min<unsigned>(static_cast<unsigned>((r.total + 511) / 512), 148 * 2));
			const auto kern = vp.stride[0] == 16 ? kmeans_update_fast_kernel<true> : kmeans_update_fast_kernel<false>;
			ensure_smem(kern, 200 * 1024);
			kern<<<blocks, 512, smem, static_cast<cudaStream_t>(stream)>>>(pts, vp.stride[0], asg, r.total, static_cast<int>(k), static_cast<int>(d),
			    static_cast<unsigned long long*>(vs.base), vs.stride[0], static_cast<unsigned long long*>(vn.base));
			return cudaGetLastError() == cudaSuccess ? 0 : 1;
		}
	}
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
