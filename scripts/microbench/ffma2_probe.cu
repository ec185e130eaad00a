// FFMA2 vs FFMA dot-product throughput probe (k-means assign inner loop shape)
#include <cstdio>
template <int J>
__global__ void dots2(const float2* __restrict__ cv, float* out, int iters) {
	float2 p[J][16];
	for(int j = 0; j < J; ++j)
		for(int q = 0; q < 16; ++q) p[j][q] = make_float2((float)(threadIdx.x + j * 16 + q), (float)(threadIdx.x + j * 16 + q + 1));
	float2 acc[J];
	for(int j = 0; j < J; ++j) acc[j] = make_float2(0.f, 0.f);
	__shared__ float2 cs[256 * 16];
	for(int i = threadIdx.x; i < 256 * 16; i += blockDim.x) cs[i] = cv[i];
	__syncthreads();
	for(int it = 0; it < iters; ++it) {
#pragma unroll 1
		for(int c = 0; c < 256; ++c) {
			float2 c16[16];
#pragma unroll
			for(int q = 0; q < 16; ++q) c16[q] = cs[c * 16 + q];
#pragma unroll
			for(int j = 0; j < J; ++j) {
				float2 m = make_float2(0.f, 0.f);
#pragma unroll
				for(int q = 0; q < 16; ++q) m = __ffma2_rn(p[j][q], c16[q], m);
				acc[j] = __fadd2_rn(acc[j], m);
			}
		}
	}
	float s = 0;
	for(int j = 0; j < J; ++j) s += acc[j].x + acc[j].y;
	out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int J>
__global__ void dots1(const float* __restrict__ cv, float* out, int iters) {
	float p[J][16];
	for(int j = 0; j < J; ++j)
		for(int q = 0; q < 16; ++q) p[j][q] = (float)(threadIdx.x + j * 16 + q);
	float acc[J];
	for(int j = 0; j < J; ++j) acc[j] = 0;
	__shared__ float cs[256 * 16];
	for(int i = threadIdx.x; i < 256 * 16; i += blockDim.x) cs[i] = cv[i];
	__syncthreads();
	for(int it = 0; it < iters; ++it) {
#pragma unroll 1
		for(int c = 0; c < 256; ++c) {
			float c16[16];
#pragma unroll
			for(int q = 0; q < 16; ++q) c16[q] = cs[c * 16 + q];
#pragma unroll
			for(int j = 0; j < J; ++j) {
				float m = 0;
#pragma unroll
				for(int q = 0; q < 16; ++q) m = fmaf(p[j][q], c16[q], m);
				acc[j] += m;
			}
		}
	}
	float s = 0;
	for(int j = 0; j < J; ++j) s += acc[j];
	out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class T> double run(void (*kern)(const T*, float*, int), const void* cv, float* o, int blocks, int threads, int iters, double fma_per_iter_thread) {
	cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
	const T* c = static_cast<const T*>(cv);
	kern<<<blocks, threads>>>(c, o, 1);
	cudaEventRecord(a); kern<<<blocks, threads>>>(c, o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
	float ms; cudaEventElapsedTime(&ms, a, b);
	return double(blocks) * threads * iters * fma_per_iter_thread / ms / 1e9;
}
int main() {
	float* c; float* o; cudaMalloc(&c, 256 * 16 * 8); cudaMemset(c, 0, 256 * 16 * 8); cudaMalloc(&o, 148 * 4 * 256 * 4);
	for(int bpsm = 1; bpsm <= 2; ++bpsm) {
		printf("FFMA  J=4 %d CTA/SM: %.2f Tfma/s\n", bpsm, run(dots1<4>, c, o, 148 * bpsm, 256, 20, 256.0 * 4 * 16));
		printf("FFMA  J=8 %d CTA/SM: %.2f Tfma/s\n", bpsm, run(dots1<8>, c, o, 148 * bpsm, 256, 20, 256.0 * 8 * 16));
		printf("FFMA2 J=2 %d CTA/SM: %.2f Tfma/s\n", bpsm, run(dots2<2>, c, o, 148 * bpsm, 256, 20, 256.0 * 2 * 32));
		printf("FFMA2 J=4 %d CTA/SM: %.2f Tfma/s\n", bpsm, run(dots2<4>, c, o, 148 * bpsm, 256, 20, 256.0 * 4 * 32));
	}
	printf("nominal at 1.965 GHz: %.2f Tfma/s\n", 148 * 128 * 1.965e-3);
	return 0;
}
