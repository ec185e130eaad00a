// Device-side helpers shared by the sm_100a kernel launchers.
//
// A launcher receives one superblock (mt_launch_ctx): the global thread range it must cover
// and, per parameter, either a scalar or a chunk view. Views address elements with GLOBAL
// array coordinates exactly like the reference's array_view (kernels.hpp:18-42): element g
// lives at base[sum_k (g_k - offset_k) * stride_k]. The CUDA grid a launcher uses is its own
// choice; only the set of global threads executed (and, for order-sensitive float kernels,
// the per-output accumulation order) has to match the reference's CPU body.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "../../../include/manta_b200.h"

namespace mtb {
namespace kern {

struct dview {
	char* base;
	int64_t off[3];
	int64_t st[3];
};

inline dview make_view(const mt_view& v) {
	dview d{};
	d.base = static_cast<char*>(v.base);
	for(int k = 0; k < 3; ++k) {
		d.off[k] = v.offset[k];
		d.st[k] = v.stride[k];
	}
	return d;
}

template <typename T>
__device__ __forceinline__ T* at1(const dview& v, int64_t i) {
	return reinterpret_cast<T*>(v.base) + (i - v.off[0]) * v.st[0];
}
template <typename T>
__device__ __forceinline__ T* at2(const dview& v, int64_t i, int64_t j) {
	return reinterpret_cast<T*>(v.base) + (i - v.off[0]) * v.st[0] + (j - v.off[1]) * v.st[1];
}
template <typename T>
__device__ __forceinline__ T* at3(const dview& v, int64_t i, int64_t j, int64_t k) {
	return reinterpret_cast<T*>(v.base) + (i - v.off[0]) * v.st[0] + (j - v.off[1]) * v.st[1] + (k - v.off[2]) * v.st[2];
}

// thread range of a superblock clipped by per-axis limits [0, lim_k)
struct range {
	int rank;
	int64_t lo[3];
	int64_t ext[3];
	int64_t total;
};

inline range clip_range(const mt_launch_ctx* c, const int64_t* lim) {
	range r{};
	r.rank = c->rank;
	r.total = 1;
	for(int k = 0; k < 3; ++k) {
		r.lo[k] = 0;
		r.ext[k] = 1;
	}
	for(int k = 0; k < c->rank; ++k) {
		const int64_t hi = c->threads_hi[k] < lim[k] ? c->threads_hi[k] : lim[k];
		r.lo[k] = c->threads_lo[k];
		r.ext[k] = hi > r.lo[k] ? hi - r.lo[k] : 0;
		r.total *= r.ext[k];
	}
	return r;
}

// global coordinates of the linear index t (last axis fastest)
__device__ __forceinline__ void coords(const range& r, int64_t t, int64_t* g) {
	for(int k = r.rank - 1; k >= 0; --k) {
		const int64_t e = r.ext[k];
		g[k] = r.lo[k] + t % e;
		t /= e;
	}
}

inline unsigned grid_1d(int64_t n, int threads) {
	int64_t b = (n + threads - 1) / threads;
	const int64_t cap = 148ll * 64;
	if(b > cap) b = cap;
	if(b < 1) b = 1;
	return static_cast<unsigned>(b);
}

// cudaFuncSetAttribute is per device: remember which devices a kernel was configured on
template <typename F>
inline void ensure_smem(F* func, int bytes) {
	static std::mutex mu;
	static std::set<std::pair<const void*, int>> done;
	int dev = 0;
	cudaGetDevice(&dev);
	std::lock_guard<std::mutex> lock(mu);
	if(!done.insert({reinterpret_cast<const void*>(func), dev}).second) return;
	cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

__device__ __forceinline__ uint64_t mix64(uint64_t h) {
	h ^= h >> 33;
	h *= 0xff51afd7ed558ccdULL;
	h ^= h >> 33;
	h *= 0xc4ceb9fe1a85ec53ULL;
	h ^= h >> 33;
	return h;
}

} // namespace kern
} // namespace mtb
