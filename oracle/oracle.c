/*
 * ORACLE / TEST INFRASTRUCTURE — plain-C restatement of the kernel formulas on the hot path.
 * Never linked into the product; loaded only by tests/ (and smoke()) as the checker.
 *
 * Each function restates one CPU kernel body of the reference (or of the reference-API
 * restatement in oracle/ref_shim.cpp for kernels the reference lacks), over whole row-major
 * arrays instead of per-chunk views, so GPU results can be checked at sizes where running the
 * reference executor would take minutes. Compiled with -ffp-contract=off: float expressions
 * round after every operation, in the order written, like the reference build.
 *
 *   stencil1d      proj/src/kernels.cpp:147-165
 *   matmul (f32)   proj/src/kernels.cpp:167-193
 *   kmeans_*       proj/src/kernels.cpp:267-346 (i32 storage variant: ref_shim.cpp)
 *   ipattern/ramp  proj/src/kernels.cpp:425-496, mix64 :103-110
 *   heat2d, histogram, hpattern1d, ramp2d_f32: oracle/ref_shim.cpp (plugin-API restatements)
 *
 * Pinned against the reference executor in tests/test_oracle.py and against the golden
 * vectors of tests/golden/ (oracle/make_golden.py).
 */
#include <stdint.h>
#include <string.h>

static uint64_t mix64(uint64_t h) {
	h ^= h >> 33;
	h *= 0xff51afd7ed558ccdULL;
	h ^= h >> 33;
	h *= 0xc4ceb9fe1a85ec53ULL;
	h ^= h >> 33;
	return h;
}

/* out rows [r0, r1) of a heat step; `in` holds rows [in_r0, in_r0 + in_rows) x [0, cols) */
void oracle_heat2d_rows(int64_t rows, int64_t cols, double alpha, const float* in, int64_t in_r0, int64_t in_rows, float* out, int64_t r0,
    int64_t r1) {
	const float a = (float)alpha;
	for(int64_t i = r0; i < r1; ++i) {
		const float* row = in + (i - in_r0) * cols;
		const float* up_row = (i > 0 && i - 1 >= in_r0) ? row - cols : 0;
		const float* dn_row = (i + 1 < rows && i + 1 < in_r0 + in_rows) ? row + cols : 0;
		float* o = out + (i - r0) * cols;
		for(int64_t j = 0; j < cols; ++j) {
			const float c = row[j];
			const float up = i > 0 ? up_row[j] : 0.0f;
			const float dn = i + 1 < rows ? dn_row[j] : 0.0f;
			const float lf = j > 0 ? row[j - 1] : 0.0f;
			const float rt = j + 1 < cols ? row[j + 1] : 0.0f;
			const float s = ((up + dn) + (lf + rt)) - 4.0f * c;
			o[j] = c + a * s;
		}
	}
}

void oracle_heat2d(int64_t rows, int64_t cols, double alpha, const float* in, float* out) {
	oracle_heat2d_rows(rows, cols, alpha, in, 0, rows, out, 0, rows);
}

void oracle_stencil1d(int64_t n, const float* in, float* out) {
	for(int64_t i = 0; i < n; ++i) {
		const float left = i - 1 >= 0 ? in[i - 1] : 0.0f;
		const float mid = in[i];
		const float right = i + 1 < n ? in[i + 1] : 0.0f;
		out[i] = (left + mid + right) / 3.0f;
	}
}

void oracle_ramp2d_f32(int64_t rows, int64_t cols, int64_t mod, double base, double scale, float* out) {
	for(int64_t i = 0; i < rows; ++i)
		for(int64_t j = 0; j < cols; ++j) out[i * cols + j] = (float)(base + scale * (double)((i * 31 + j * 17 + 7) % mod) / (double)mod);
}

void oracle_ipattern2d_i32(int64_t rows, int64_t cols, int64_t mod, int32_t* out) {
	for(int64_t i = 0; i < rows; ++i)
		for(int64_t j = 0; j < cols; ++j) out[i * cols + j] = (int32_t)((i * 31 + j * 17 + 7) % mod);
}

void oracle_hpattern1d(int64_t lo, int64_t hi, int64_t bins, int64_t seed, int32_t* out) {
	for(int64_t i = lo; i < hi; ++i) out[i - lo] = (int32_t)(mix64((uint64_t)i ^ (uint64_t)seed) % (uint64_t)bins);
}

/* counts of x[i] in [0, bins) (wrapping u64, like every integer reduce of the reference) */
void oracle_histogram(const int32_t* x, int64_t n, int64_t bins, int64_t* hist) {
	memset(hist, 0, (size_t)bins * sizeof(int64_t));
	for(int64_t i = 0; i < n; ++i) {
		const int64_t b = x[i];
		if(b >= 0 && b < bins) hist[b] = (int64_t)((uint64_t)hist[b] + 1u);
	}
}

/* histogram of hpattern1d(i) for i in [lo, hi) without materialising x */
void oracle_histogram_hashed(int64_t lo, int64_t hi, int64_t bins, int64_t seed, int64_t* hist) {
	memset(hist, 0, (size_t)bins * sizeof(int64_t));
	for(int64_t i = lo; i < hi; ++i) hist[mix64((uint64_t)i ^ (uint64_t)seed) % (uint64_t)bins] += 1;
}

void oracle_kmeans_assign_i32(int64_t n, int64_t k, int64_t d, const int32_t* points, const int32_t* cents, int32_t* assign) {
	for(int64_t i = 0; i < n; ++i) {
		int64_t best = 0, best_dist = INT64_MAX;
		for(int64_t c = 0; c < k; ++c) {
			int64_t dist = 0;
			for(int64_t t = 0; t < d; ++t) {
				const int64_t diff = (int64_t)points[i * d + t] - cents[c * d + t];
				dist += diff * diff;
			}
			if(dist < best_dist) {
				best_dist = dist;
				best = c;
			}
		}
		assign[i] = (int32_t)best;
	}
}

void oracle_kmeans_update_i32(int64_t n, int64_t k, int64_t d, const int32_t* points, const int32_t* assign, int64_t* sums, int64_t* counts) {
	memset(sums, 0, (size_t)(k * d) * sizeof(int64_t));
	memset(counts, 0, (size_t)k * sizeof(int64_t));
	for(int64_t i = 0; i < n; ++i) {
		const int64_t c = assign[i];
		for(int64_t t = 0; t < d; ++t) sums[c * d + t] = (int64_t)((uint64_t)sums[c * d + t] + (uint64_t)(int64_t)points[i * d + t]);
		counts[c] += 1;
	}
}

void oracle_kmeans_finalize_i32(int64_t k, int64_t d, const int64_t* sums, const int64_t* counts, int32_t* cents) {
	for(int64_t c = 0; c < k; ++c)
		if(counts[c] > 0)
			for(int64_t t = 0; t < d; ++t) cents[c * d + t] = (int32_t)(sums[c * d + t] / counts[c]);
}

/* C[i,j] = sum_l A[i,l] * B[l,j], f32, l ascending, each op rounded (no FMA) */
void oracle_matmul_f32(int64_t m, int64_t n, int64_t k, const float* a, const float* b, float* c) {
	for(int64_t i = 0; i < m; ++i)
		for(int64_t j = 0; j < n; ++j) {
			float acc = 0.0f;
			for(int64_t l = 0; l < k; ++l) acc += a[i * k + l] * b[l * n + j];
			c[i * n + j] = acc;
		}
}

/* fp64-accumulated reference product for the tensor-core GEMM tolerance check; a/b given as
 * f32 (exact images of bf16 inputs) */
void oracle_matmul_f64acc(int64_t m, int64_t n, int64_t k, const float* a, const float* b, double* c) {
	for(int64_t i = 0; i < m; ++i) {
		for(int64_t j = 0; j < n; ++j) c[i * n + j] = 0.0;
		for(int64_t l = 0; l < k; ++l) {
			const double av = a[i * k + l];
			for(int64_t j = 0; j < n; ++j) c[i * n + j] += av * (double)b[l * n + j];
		}
	}
}
