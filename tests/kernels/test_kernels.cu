// Test-only kernels registered through the public plugin API (mt_kernel_register), the
// B200 counterpart of the kernels the reference's tests register on the fly
// (proj/tests/unit/test_runtime.cpp:130-142 row_reduce_i64, :167-178 partial_min).
// Loading this library registers them (constructor below).
#include <cuda_runtime.h>

#include <cstring>

#include "../../include/manta_b200.h"

namespace {

struct view1 {
	char* base;
	int64_t off0, st0, off1, st1;
};

view1 v(const mt_view& m) { return view1{static_cast<char*>(m.base), m.offset[0], m.stride[0], m.offset[1], m.stride[1]}; }

__global__ void row_reduce_i64_k(int64_t r0, int64_t r1, int64_t c0, int64_t c1, view1 a, view1 sum) {
	const int64_t i = r0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
	if(i >= r1) return;
	auto* s = reinterpret_cast<unsigned long long*>(sum.base) + (i - sum.off0) * sum.st0;
	unsigned long long acc = *s;
	for(int64_t j = c0; j < c1; ++j)
		acc += static_cast<unsigned long long>(*(reinterpret_cast<int64_t*>(a.base) + (i - a.off0) * a.st0 + (j - a.off1) * a.st1));
	*s = acc;
}

int launch_row_reduce_i64(const mt_launch_ctx* c, void* stream) {
	const int64_t rows = c->scalars_int[0], cols = c->scalars_int[1];
	const int64_t r0 = c->threads_lo[0], r1 = c->threads_hi[0] < rows ? c->threads_hi[0] : rows;
	const int64_t c0 = c->threads_lo[1], c1 = c->threads_hi[1] < cols ? c->threads_hi[1] : cols;
	if(r0 >= r1 || c0 >= c1) return 0;
	row_reduce_i64_k<<<static_cast<unsigned>((r1 - r0 + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(r0, r1, c0, c1, v(c->views[2]),
	    v(c->views[3]));
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

__global__ void partial_min_k(int64_t lo, int64_t hi, view1 src, view1 dst) {
	const int64_t i = lo + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
	if(i >= hi) return;
	auto* cell = reinterpret_cast<int64_t*>(dst.base) + (i - dst.off0) * dst.st0;
	const int64_t x = *(reinterpret_cast<int64_t*>(src.base) + (i - src.off0) * src.st0) + i;
	if(x < *cell) *cell = x;
}

int launch_partial_min(const mt_launch_ctx* c, void* stream) {
	const int64_t n = c->scalars_int[0];
	const int64_t lim = n < 4 ? n : 4; // only the first half contributes
	const int64_t lo = c->threads_lo[0], hi = c->threads_hi[0] < lim ? c->threads_hi[0] : lim;
	if(lo >= hi) return 0;
	partial_min_k<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(lo, hi, v(c->views[1]), v(c->views[2]));
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// bf16 partial sums: cell c of the partial accumulates src[i] for i = c mod 8 of this superblock,
// one f32 add rounded to bf16 (nearest-even) per element, in ascending i
__device__ float bf(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
__device__ uint16_t to_bf(float f) {
	uint32_t u = __float_as_uint(f);
	u += 0x7fffu + ((u >> 16) & 1u);
	return static_cast<uint16_t>(u >> 16);
}

__global__ void partial_sum_bf16_k(int64_t lo, int64_t hi, view1 src, view1 dst) {
	const int64_t c = threadIdx.x;
	auto* cell = reinterpret_cast<uint16_t*>(dst.base) + (c - dst.off0) * dst.st0;
	uint16_t acc = *cell;
	for(int64_t i = lo; i < hi; ++i)
		if(i % 8 == c) acc = to_bf(__fadd_rn(bf(acc), bf(*(reinterpret_cast<uint16_t*>(src.base) + (i - src.off0) * src.st0))));
	*cell = acc;
}

int launch_partial_sum_bf16(const mt_launch_ctx* c, void* stream) {
	const int64_t n = c->scalars_int[0];
	const int64_t lo = c->threads_lo[0], hi = c->threads_hi[0] < n ? c->threads_hi[0] : n;
	if(lo >= hi) return 0;
	partial_sum_bf16_k<<<1, 8, 0, static_cast<cudaStream_t>(stream)>>>(lo, hi, v(c->views[1]), v(c->views[2]));
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

mt_param_spec P(const char* n, int kind, int dtype, int rank, int w) {
	mt_param_spec p{};
	std::strncpy(p.name, n, sizeof(p.name) - 1);
	p.kind = kind;
	p.dtype = dtype;
	p.rank = rank;
	p.writable = w;
	return p;
}

__attribute__((constructor)) void register_test_kernels() {
	const mt_param_spec rr[] = {P("rows", MT_PARAM_SCALAR, MT_I64, 0, 0), P("cols", MT_PARAM_SCALAR, MT_I64, 0, 0), P("A", MT_PARAM_ARRAY, MT_I64, 2, 0),
	    P("sum", MT_PARAM_ARRAY, MT_I64, 1, 1)};
	mt_kernel_register("row_reduce_i64", rr, 4, launch_row_reduce_i64);
	const mt_param_spec pm[] = {P("n", MT_PARAM_SCALAR, MT_I64, 0, 0), P("src", MT_PARAM_ARRAY, MT_I64, 1, 0), P("dst", MT_PARAM_ARRAY, MT_I64, 1, 1)};
	mt_kernel_register("partial_min", pm, 3, launch_partial_min);
	const mt_param_spec ps[] = {P("n", MT_PARAM_SCALAR, MT_I64, 0, 0), P("src", MT_PARAM_ARRAY, MT_BF16, 1, 0), P("dst", MT_PARAM_ARRAY, MT_BF16, 1, 1)};
	mt_kernel_register("partial_sum_bf16", ps, 3, launch_partial_sum_bf16);
}

} // namespace
