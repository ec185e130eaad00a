// Synthesized `gather` kernels (the reference's make_gather_kernel, proj/src/scenario.cpp:276-364)
// as one data-driven sm_100a interpreter kernel.
//
// The reference gives any annotation a body: every thread folds (wrapping u64 sum, seeded by a
// hash of its index) the elements of its declared read regions, then writes that digest to, or
// reduce-combines it into, every element of its declared write/reduce regions. The fuzz
// campaign (scenario.cpp:814-849) and the correlator_like scenario run on it. Here the parsed
// annotation is flattened into a POD descriptor passed by value; one GPU thread interprets it
// for one global thread index. Reduce combines use 64-bit atomics (wrapping add, signed
// min/max, CAS for *), which commute, so results are bit-exact against the sequential CPU body.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>

#include "../annotation.hpp"
#include "../executor.hpp"
#include "../registry.hpp"
#include "common.cuh"

namespace mtb {
namespace gather {

constexpr int kMaxAcc = 8;

struct lin {
	int64_t c;
	int nt;
	int slot[3];
	int64_t coeff[3];
};

struct ixd {
	int is_slice, has_lo, has_hi;
	lin single, lo, hi;
};

struct accd {
	int mode; // 0 read, 1 write, 2 readwrite, 3 reduce
	int op;   // reduce_op
	int dtype;
	int rank;
	int64_t dom_lo[3], dom_hi[3];
	ixd ix[3];
};

struct desc {
	int nvars;
	int space[3];
	int axis[3];
	int nacc;
	accd acc[kMaxAcc];
};

struct views {
	kern::dview v[kMaxAcc];
};

__device__ __forceinline__ int64_t eval(const lin& e, const int64_t* env) {
	int64_t r = e.c;
	for(int t = 0; t < e.nt; ++t) r += e.coeff[t] * env[e.slot[t]];
	return r;
}

__device__ __forceinline__ uint64_t mix64(uint64_t h) { return kern::mix64(h); }

__device__ __forceinline__ uint64_t hash_point(const int64_t* g, int rank) {
	uint64_t h = 0x243f6a8885a308d3ULL;
	for(int k = 0; k < rank; ++k) h = mix64(h ^ (static_cast<uint64_t>(g[k]) * 0x100000001b3ULL + static_cast<uint64_t>(k)));
	return h;
}

__device__ __forceinline__ char* cell(const kern::dview& v, const accd& a, const int64_t* p) {
	int64_t off = 0;
	for(int k = 0; k < a.rank; ++k) off += (p[k] - v.off[k]) * v.st[k];
	return v.base + off * (a.dtype == 1 || a.dtype == 3 ? 8 : 4);
}

__device__ __forceinline__ int64_t load_int(const accd& a, const char* c) {
	switch(a.dtype) {
	case 0: return *reinterpret_cast<const int32_t*>(c);
	case 1: return *reinterpret_cast<const int64_t*>(c);
	case 2: return static_cast<int64_t>(*reinterpret_cast<const float*>(c));
	default: return static_cast<int64_t>(*reinterpret_cast<const double*>(c));
	}
}

__device__ __forceinline__ void store_int(const accd& a, char* c, int64_t v) {
	switch(a.dtype) {
	case 0: *reinterpret_cast<int32_t*>(c) = static_cast<int32_t>(v); break;
	case 1: *reinterpret_cast<int64_t*>(c) = v; break;
	case 2: *reinterpret_cast<float*>(c) = static_cast<float>(v); break;
	default: *reinterpret_cast<double*>(c) = static_cast<double>(v); break;
	}
}

// thread_region of scenario.cpp:301-319: inclusive per-thread bounds, clipped; false if empty
__device__ __forceinline__ bool region(const accd& a, const int64_t* env, int64_t* lo, int64_t* hi) {
	for(int k = 0; k < a.rank; ++k) {
		const ixd& x = a.ix[k];
		int64_t s, e;
		if(!x.is_slice) {
			s = e = eval(x.single, env);
		} else {
			s = x.has_lo ? eval(x.lo, env) : a.dom_lo[k];
			e = x.has_hi ? eval(x.hi, env) : a.dom_hi[k] - 1;
		}
		if(s > e) return false;
		lo[k] = s > a.dom_lo[k] ? s : a.dom_lo[k];
		hi[k] = e + 1 < a.dom_hi[k] ? e + 1 : a.dom_hi[k];
		if(hi[k] <= lo[k]) return false;
	}
	return true;
}

__device__ void combine(const accd& a, char* c, int64_t out) {
	if(a.dtype == 1) {
		auto* p = reinterpret_cast<unsigned long long*>(c);
		switch(a.op) {
		case 0: atomicAdd(p, static_cast<unsigned long long>(out)); return;
		case 2: atomicMin(reinterpret_cast<long long*>(c), static_cast<long long>(out)); return;
		case 3: atomicMax(reinterpret_cast<long long*>(c), static_cast<long long>(out)); return;
		default: {
			unsigned long long old = *p, assumed;
			do {
				assumed = old;
				old = atomicCAS(p, assumed, assumed * static_cast<unsigned long long>(out));
			} while(old != assumed);
			return;
		}
		}
	}
	// non-i64 reduce targets: CAS on the containing word (fuzz arrays are i64; kept exact)
	if(a.dtype == 0) {
		auto* p = reinterpret_cast<int*>(c);
		int old = *p, assumed;
		do {
			assumed = old;
			int64_t cur = assumed, r = cur;
			switch(a.op) {
			case 0: r = static_cast<int64_t>(static_cast<uint64_t>(cur) + static_cast<uint64_t>(out)); break;
			case 1: r = static_cast<int64_t>(static_cast<uint64_t>(cur) * static_cast<uint64_t>(out)); break;
			case 2: r = cur < out ? cur : out; break;
			default: r = cur < out ? out : cur; break;
			}
			old = atomicCAS(p, assumed, static_cast<int>(static_cast<int32_t>(r)));
		} while(old != assumed);
	}
}

__global__ void gather_kernel(desc d, views vw, kern::range r, int64_t bs0, int64_t bs1, int64_t bs2) {
	const int64_t bs[3] = {bs0, bs1, bs2};
	for(int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < r.total; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		int64_t g[3] = {0, 0, 0};
		kern::coords(r, t, g);
		int64_t env[3];
		for(int v = 0; v < d.nvars; ++v) {
			const int ax = d.axis[v];
			env[v] = d.space[v] == 0 ? g[ax] : (d.space[v] == 1 ? g[ax] / bs[ax] : g[ax] % bs[ax]);
		}
		uint64_t val = hash_point(g, r.rank);
		int64_t lo[3], hi[3], p[3];
		for(int i = 0; i < d.nacc; ++i) {
			const accd& a = d.acc[i];
			if(!(a.mode == 0 || a.mode == 2)) continue;
			if(!region(a, env, lo, hi)) continue;
			for(p[0] = lo[0]; p[0] < hi[0]; ++p[0])
				for(p[1] = a.rank > 1 ? lo[1] : 0; p[1] < (a.rank > 1 ? hi[1] : 1); ++p[1])
					for(p[2] = a.rank > 2 ? lo[2] : 0; p[2] < (a.rank > 2 ? hi[2] : 1); ++p[2]) val += static_cast<uint64_t>(load_int(a, cell(vw.v[i], a, p)));
		}
		const int64_t out = static_cast<int64_t>(val);
		for(int i = 0; i < d.nacc; ++i) {
			const accd& a = d.acc[i];
			if(a.mode == 0) continue;
			if(!region(a, env, lo, hi)) continue;
			for(p[0] = lo[0]; p[0] < hi[0]; ++p[0])
				for(p[1] = a.rank > 1 ? lo[1] : 0; p[1] < (a.rank > 1 ? hi[1] : 1); ++p[1])
					for(p[2] = a.rank > 2 ? lo[2] : 0; p[2] < (a.rank > 2 ? hi[2] : 1); ++p[2]) {
						char* c = cell(vw.v[i], a, p);
						if(a.mode == 3)
							combine(a, c, out);
						else
							store_int(a, c, out);
					}
		}
	}
}

int launcher(const mt_launch_ctx* c, void* stream) {
	const desc& d = *static_cast<const desc*>(c->user);
	views vw{};
	for(int i = 0; i < d.nacc && i < c->nparams; ++i) vw.v[i] = kern::make_view(c->views[i]);
	// every lane of the superblock runs (the CPU context's grid is [0, threads.hi))
	kern::range r{};
	r.rank = c->rank;
	r.total = 1;
	for(int k = 0; k < 3; ++k) {
		r.lo[k] = 0;
		r.ext[k] = 1;
	}
	for(int k = 0; k < c->rank; ++k) {
		r.lo[k] = c->threads_lo[k];
		r.ext[k] = c->threads_hi[k] - c->threads_lo[k];
		r.total *= r.ext[k];
	}
	if(r.total <= 0) return 0;
	gather_kernel<<<kern::grid_1d(r.total, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(d, vw, r, c->block_size[0], c->rank > 1 ? c->block_size[1] : 1,
	    c->rank > 2 ? c->block_size[2] : 1);
	return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

lin flatten(const lin_expr& e) {
	lin l{};
	l.c = e.constant;
	l.nt = static_cast<int>(e.terms.size());
	if(l.nt > 3) throw validation_error("gather: expression has more than 3 variables");
	for(int t = 0; t < l.nt; ++t) {
		l.slot[t] = e.terms[static_cast<size_t>(t)].slot;
		l.coeff[t] = e.terms[static_cast<size_t>(t)].coeff;
	}
	return l;
}

} // namespace gather

// Builds the synthesized kernel for `annotation` over arrays of the given element types and
// domains (one per access, in access order), as a descriptor owned by the caller.
std::shared_ptr<void> make_gather_kernel(const std::string& annotation_text, const std::vector<dtype>& types, const std::vector<box>& domains,
    kernel_entry& out) {
	using namespace gather;
	const annotation ann = parse_annotation(annotation_text);
	if(ann.accesses.size() > static_cast<size_t>(kMaxAcc)) throw validation_error("gather: too many accesses");
	if(types.size() != ann.accesses.size() || domains.size() != ann.accesses.size()) throw validation_error("gather: one type and domain per access");
	auto d = std::make_shared<desc>();
	std::memset(d.get(), 0, sizeof(desc));
	d->nvars = static_cast<int>(ann.vars.size());
	for(size_t v = 0; v < ann.vars.size(); ++v) {
		d->space[v] = static_cast<int>(ann.vars[v].space);
		d->axis[v] = ann.vars[v].axis;
	}
	d->nacc = static_cast<int>(ann.accesses.size());
	out.params.clear();
	for(size_t i = 0; i < ann.accesses.size(); ++i) {
		const auto& a = ann.accesses[i];
		auto& x = d->acc[i];
		x.mode = static_cast<int>(a.mode.kind);
		x.op = static_cast<int>(a.mode.op);
		x.dtype = static_cast<int>(types[i]);
		if(types[i] == dtype::bf16) throw validation_error("gather: bf16 arrays are not supported");
		x.rank = domains[i].rank();
		if(static_cast<int>(a.indices.size()) != x.rank) throw validation_error("gather: index count differs from the array rank");
		for(int k = 0; k < x.rank; ++k) {
			x.dom_lo[k] = domains[i].lo[k];
			x.dom_hi[k] = domains[i].hi[k];
			const auto& ix = a.indices[static_cast<size_t>(k)];
			x.ix[k].is_slice = ix.is_slice;
			x.ix[k].has_lo = ix.has_lower;
			x.ix[k].has_hi = ix.has_upper;
			x.ix[k].single = flatten(ix.single);
			x.ix[k].lo = flatten(ix.lower);
			x.ix[k].hi = flatten(ix.upper);
		}
		const bool writable = a.mode.writes() || a.mode.reduces();
		out.params.push_back(param_sig{a.argument, true, types[i], x.rank, writable});
	}
	out.launcher = gather::launcher;
	out.user = d.get();
	return d;
}

} // namespace mtb
