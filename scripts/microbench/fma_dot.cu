#include <cstdio>
#include <cstdint>
// throughput of 16-term dot products (4 independent chains, operand c reused across chains)
template <typename T>
__global__ void dots(const T* __restrict__ cv, T* out, int iters) {
	T p[4][16];
	for(int j = 0; j < 4; ++j)
		for(int q = 0; q < 16; ++q) p[j][q] = (T)(threadIdx.x + j * 16 + q);
	T acc[4] = {0, 0, 0, 0};
	__shared__ T cs[256 * 16];
	for(int i = threadIdx.x; i < 256 * 16; i += blockDim.x) cs[i] = cv[i];
	__syncthreads();
	for(int it = 0; it < iters; ++it) {
#pragma unroll 1
		for(int c = 0; c < 256; ++c) {
			T c16[16];
#pragma unroll
			for(int q = 0; q < 16; ++q) c16[q] = cs[c * 16 + q];
#pragma unroll
			for(int j = 0; j < 4; ++j) {
				T m = 0;
#pragma unroll
				for(int q = 0; q < 16; ++q) m += p[j][q] * c16[q];
				acc[j] += m;
			}
		}
	}
	out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}
int main() {
	float* cf; int* ci; float* of; int* oi;
	cudaMalloc(&cf, 4096 * 4); cudaMalloc(&ci, 4096 * 4); cudaMemset(cf, 0, 4096*4); cudaMemset(ci, 0, 4096*4);
	const int blocks = 148 * 2, threads = 256, iters = 20;
	cudaMalloc(&of, blocks * threads * 4); cudaMalloc(&oi, blocks * threads * 4);
	cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
	for(int r = 0; r < 2; ++r) {
		float ms; cudaError_t e0 = cudaGetLastError(); if(e0) printf("err %s\n", cudaGetErrorString(e0));
		dots<int><<<blocks, threads>>>(ci, oi, 1);
		cudaEventRecord(a); dots<int><<<blocks, threads>>>(ci, oi, iters); cudaEventRecord(b); cudaEventSynchronize(b);
		cudaEventElapsedTime(&ms, a, b);
		double ops = double(blocks) * threads * iters * 256 * 4 * 16;
		{ cudaError_t e1 = cudaGetLastError(); if(e1) printf("err2 %s\n", cudaGetErrorString(e1)); }
		printf("IMAD: %.3f ms, %.2f Tmac/s\n", ms, ops / ms / 1e9);
		dots<float><<<blocks, threads>>>(cf, of, 1);
		cudaEventRecord(a); dots<float><<<blocks, threads>>>(cf, of, iters); cudaEventRecord(b); cudaEventSynchronize(b);
		cudaEventElapsedTime(&ms, a, b);
		printf("FFMA: %.3f ms, %.2f Tmac/s\n", ms, ops / ms / 1e9);
	}
	return 0;
}
