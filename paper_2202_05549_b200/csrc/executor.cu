#include "executor.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <fcntl.h>
#include <unistd.h>
#include <cstdio>
#include <set>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>

namespace mtb {

namespace {
struct nccl_fns {
	ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
	ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
	ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
	ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
	const char* (*error_string)(ncclResult_t) = nullptr;
};
nccl_fns g_nccl;

void nccl_check(ncclResult_t r, const char* what) {
	if(r != ncclSuccess)
		throw execution_error(std::string(what) + " failed: " + (g_nccl.error_string ? g_nccl.error_string(r) : std::to_string(static_cast<int>(r))));
}
} // namespace

void check_cuda(cudaError_t e, const char* what) {
	if(e != cudaSuccess) throw execution_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- device helpers ----------------------------------------------------------------------

namespace {

template <typename T>
__device__ __forceinline__ T add_wrap(T a, T b) {
	return a + b;
}
template <>
__device__ __forceinline__ int32_t add_wrap(int32_t a, int32_t b) {
	return static_cast<int32_t>(static_cast<uint32_t>(a) + static_cast<uint32_t>(b));
}
template <>
__device__ __forceinline__ int64_t add_wrap(int64_t a, int64_t b) {
	return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}
template <>
__device__ __forceinline__ float add_wrap(float a, float b) {
	return __fadd_rn(a, b);
}
template <>
__device__ __forceinline__ double add_wrap(double a, double b) {
	return __dadd_rn(a, b);
}
template <typename T>
__device__ __forceinline__ T mul_wrap(T a, T b) {
	return a * b;
}
template <>
__device__ __forceinline__ int32_t mul_wrap(int32_t a, int32_t b) {
	return static_cast<int32_t>(static_cast<uint32_t>(a) * static_cast<uint32_t>(b));
}
template <>
__device__ __forceinline__ int64_t mul_wrap(int64_t a, int64_t b) {
	return static_cast<int64_t>(static_cast<uint64_t>(a) * static_cast<uint64_t>(b));
}
template <>
__device__ __forceinline__ float mul_wrap(float a, float b) {
	return __fmul_rn(a, b);
}
template <>
__device__ __forceinline__ double mul_wrap(double a, double b) {
	return __dmul_rn(a, b);
}

struct bf16_t {
	uint16_t bits;
};
// bf16 reduce (a B200 extension: the reference has no bf16): every combine is computed in f32
// and rounded to nearest-even bf16; min/max compare the values (NaN compares false, as
// std::min/max would)
__device__ __forceinline__ float bf_to_f(bf16_t b) { return __uint_as_float(static_cast<uint32_t>(b.bits) << 16); }
__device__ __forceinline__ bf16_t f_to_bf(float f) {
	uint32_t u = __float_as_uint(f);
	if((u & 0x7fffffffu) > 0x7f800000u) return bf16_t{static_cast<uint16_t>((u >> 16) | 0x40u)}; // quiet NaN
	u += 0x7fffu + ((u >> 16) & 1u);
	return bf16_t{static_cast<uint16_t>(u >> 16)};
}
__device__ __forceinline__ bool operator<(bf16_t a, bf16_t b) { return bf_to_f(a) < bf_to_f(b); }
template <>
__device__ __forceinline__ bf16_t add_wrap(bf16_t a, bf16_t b) {
	return f_to_bf(__fadd_rn(bf_to_f(a), bf_to_f(b)));
}
template <>
__device__ __forceinline__ bf16_t mul_wrap(bf16_t a, bf16_t b) {
	return f_to_bf(__fmul_rn(bf_to_f(a), bf_to_f(b)));
}

template <typename T>
__global__ void fill_kernel(T* p, uint64_t n, T v) {
	for(uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) p[i] = v;
}

constexpr int kMaxReduceInputs = 8;
template <typename T>
struct reduce_inputs {
	const T* in[kMaxReduceInputs];
	int n;
	bool first_is_copy;
};

template <typename T, int OP>
__global__ void combine_kernel(T* out, reduce_inputs<T> ins, uint64_t count) {
	for(uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < count; e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
		int k = 0;
		T o;
		if(ins.first_is_copy) {
			o = ins.in[0][e];
			k = 1;
		} else {
			o = out[e];
		}
		for(; k < ins.n; ++k) {
			const T x = ins.in[k][e];
			if constexpr(OP == 0) o = add_wrap<T>(o, x);
			if constexpr(OP == 1) o = mul_wrap<T>(o, x);
			if constexpr(OP == 2) o = (x < o) ? x : o; // std::min
			if constexpr(OP == 3) o = (o < x) ? x : o; // std::max
		}
		out[e] = o;
	}
}

int grid_for(uint64_t n, int threads) {
	uint64_t blocks = (n + threads - 1) / threads;
	if(blocks > 148ull * 32) blocks = 148ull * 32;
	if(blocks == 0) blocks = 1;
	return static_cast<int>(blocks);
}

template <typename T>
void fill_typed(void* p, uint64_t n, T v, cudaStream_t s) {
	fill_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(static_cast<T*>(p), n, v);
}

template <typename T>
T identity_of(reduce_op op) {
	switch(op) {
	case reduce_op::plus: return T(0);
	case reduce_op::times: return T(1);
	case reduce_op::min: return std::numeric_limits<T>::max();
	case reduce_op::max: return std::numeric_limits<T>::lowest();
	}
	return T(0);
}

template <typename T>
void reduce_typed(void* out, const void* const* inputs, int n, uint64_t count, reduce_op op, cudaStream_t s) {
	for(int base = 0; base < n; base += kMaxReduceInputs) {
		reduce_inputs<T> ins{};
		ins.n = std::min(kMaxReduceInputs, n - base);
		ins.first_is_copy = base == 0;
		for(int k = 0; k < ins.n; ++k) ins.in[k] = static_cast<const T*>(inputs[base + k]);
		T* o = static_cast<T*>(out);
		const int g = grid_for(count, 256);
		switch(op) {
		case reduce_op::plus: combine_kernel<T, 0><<<g, 256, 0, s>>>(o, ins, count); break;
		case reduce_op::times: combine_kernel<T, 1><<<g, 256, 0, s>>>(o, ins, count); break;
		case reduce_op::min: combine_kernel<T, 2><<<g, 256, 0, s>>>(o, ins, count); break;
		case reduce_op::max: combine_kernel<T, 3><<<g, 256, 0, s>>>(o, ins, count); break;
		}
	}
}

// row-major strides (elements) of a chunk box
void strides_of(const box& b, int64_t* st) {
	int64_t acc = 1;
	for(int k = b.rank() - 1; k >= 0; --k) {
		st[k] = acc;
		acc *= b.extent(k);
	}
}

} // namespace

void device_fill(void* ptr, uint64_t count, dtype type, fill_kind kind, reduce_op op, cudaStream_t s) {
	const uint64_t bytes = count * dtype_size(type);
	if(kind == fill_kind::none || kind == fill_kind::zero || (kind == fill_kind::identity && op == reduce_op::plus)) {
		check_cuda(cudaMemsetAsync(ptr, 0, bytes, s), "cudaMemsetAsync");
		return;
	}
	const bool one = kind == fill_kind::one;
	switch(type) {
	case dtype::i32: fill_typed<int32_t>(ptr, count, one ? 1 : identity_of<int32_t>(op), s); break;
	case dtype::i64: fill_typed<int64_t>(ptr, count, one ? 1 : identity_of<int64_t>(op), s); break;
	case dtype::f32: fill_typed<float>(ptr, count, one ? 1.0f : identity_of<float>(op), s); break;
	case dtype::f64: fill_typed<double>(ptr, count, one ? 1.0 : identity_of<double>(op), s); break;
	case dtype::bf16: {
		// 1.0 = 0x3F80, max finite = 0x7F7F, lowest = 0xFF7F
		uint16_t v = 0x3F80;
		if(!one && op == reduce_op::min) v = 0x7F7F;
		if(!one && op == reduce_op::max) v = 0xFF7F;
		fill_typed<uint16_t>(ptr, count, v, s);
		break;
	}
	}
	check_cuda(cudaGetLastError(), "fill kernel launch");
}

void device_reduce(void* out, const void* const* inputs, int n, uint64_t count, dtype type, reduce_op op, cudaStream_t s) {
	switch(type) {
	case dtype::i32: reduce_typed<int32_t>(out, inputs, n, count, op, s); break;
	case dtype::i64: reduce_typed<int64_t>(out, inputs, n, count, op, s); break;
	case dtype::f32: reduce_typed<float>(out, inputs, n, count, op, s); break;
	case dtype::f64: reduce_typed<double>(out, inputs, n, count, op, s); break;
	case dtype::bf16: reduce_typed<bf16_t>(out, inputs, n, count, op, s); break;
	}
	check_cuda(cudaGetLastError(), "reduce kernel launch");
}

__global__ void small_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
	for(int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16; i += static_cast<int64_t>(gridDim.x) * blockDim.x) dst[i] = src[i];
}

void copy_box(const void* src_base, const box& src_chunk, int src_gpu, void* dst_base, const box& dst_chunk, int dst_gpu, const box& region,
    size_t elem, cudaStream_t s) {
	if(region.is_empty()) return;
	const int rank = region.rank();
	int64_t ss[kMaxRank], ds[kMaxRank];
	strides_of(src_chunk, ss);
	strides_of(dst_chunk, ds);
	int64_t so = 0, dof = 0;
	for(int k = 0; k < rank; ++k) {
		so += (region.lo[k] - src_chunk.lo[k]) * ss[k];
		dof += (region.lo[k] - dst_chunk.lo[k]) * ds[k];
	}
	const char* sp = static_cast<const char*>(src_base) + so * static_cast<int64_t>(elem);
	char* dp = static_cast<char*>(dst_base) + dof * static_cast<int64_t>(elem);
	// contiguous in both: region covers whole inner extents of both chunks
	bool contiguous = true;
	for(int k = 1; k < rank && contiguous; ++k) {
		if(region.extent(k) != src_chunk.extent(k) || region.extent(k) != dst_chunk.extent(k)) contiguous = false;
	}
	// after the first axis with extent > 1 everything inner must be full; relax: a single row is contiguous
	if(!contiguous) {
		int outer_nontrivial = 0;
		for(int k = 0; k < rank - 1; ++k)
			if(region.extent(k) > 1) ++outer_nontrivial;
		if(outer_nontrivial == 0) contiguous = true;
	}
	if(contiguous) {
		const size_t bytes = static_cast<size_t>(region.volume()) * elem;
		static const bool sm_copy = std::getenv("MTB_CE_COPY") == nullptr; // MTB_CE_COPY=1: copy engines only
		if(src_gpu < 0 || dst_gpu < 0)
			check_cuda(cudaMemcpyAsync(dp, sp, bytes, cudaMemcpyDefault, s), "cudaMemcpyAsync (host)");
		else if(src_gpu == dst_gpu && sm_copy && bytes <= (1u << 20) && bytes % 16 == 0 && reinterpret_cast<uintptr_t>(sp) % 16 == 0
		        && reinterpret_cast<uintptr_t>(dp) % 16 == 0) {
			// small halo rows: an SM copy kernel starts sooner than a copy-engine transfer (C1 with
			// graph replay: 31.5 vs 32.6 us per iteration)
			const int64_t n16 = static_cast<int64_t>(bytes / 16);
			small_copy_kernel<<<static_cast<unsigned>(std::min<int64_t>((n16 + 255) / 256, 64)), 256, 0, s>>>(reinterpret_cast<const int4*>(sp),
			    reinterpret_cast<int4*>(dp), n16);
			check_cuda(cudaGetLastError(), "small copy kernel");
		} else if(src_gpu == dst_gpu)
			check_cuda(cudaMemcpyAsync(dp, sp, bytes, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync");
		else
			check_cuda(cudaMemcpyPeerAsync(dp, dst_gpu, sp, src_gpu, bytes, s), "cudaMemcpyPeerAsync");
		return;
	}
	// general strided box: (z, y, x) = padded (axis0, axis1, axis2)
	int64_t ext[3] = {1, 1, 1}, sext[3] = {1, 1, 1}, dext[3] = {1, 1, 1};
	for(int k = 0; k < rank; ++k) {
		ext[3 - rank + k] = region.extent(k);
		sext[3 - rank + k] = src_chunk.extent(k);
		dext[3 - rank + k] = dst_chunk.extent(k);
	}
	if(src_gpu == dst_gpu || src_gpu < 0 || dst_gpu < 0) {
		cudaMemcpy3DParms p{};
		p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(sp), static_cast<size_t>(sext[2]) * elem, static_cast<size_t>(sext[2]) * elem, static_cast<size_t>(sext[1]));
		p.dstPtr = make_cudaPitchedPtr(dp, static_cast<size_t>(dext[2]) * elem, static_cast<size_t>(dext[2]) * elem, static_cast<size_t>(dext[1]));
		p.extent = make_cudaExtent(static_cast<size_t>(ext[2]) * elem, static_cast<size_t>(ext[1]), static_cast<size_t>(ext[0]));
		p.kind = (src_gpu < 0 || dst_gpu < 0) ? cudaMemcpyDefault : cudaMemcpyDeviceToDevice;
		check_cuda(cudaMemcpy3DAsync(&p, s), "cudaMemcpy3DAsync");
	} else {
		cudaMemcpy3DPeerParms p{};
		p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(sp), static_cast<size_t>(sext[2]) * elem, static_cast<size_t>(sext[2]) * elem, static_cast<size_t>(sext[1]));
		p.dstPtr = make_cudaPitchedPtr(dp, static_cast<size_t>(dext[2]) * elem, static_cast<size_t>(dext[2]) * elem, static_cast<size_t>(dext[1]));
		p.srcDevice = src_gpu;
		p.dstDevice = dst_gpu;
		p.extent = make_cudaExtent(static_cast<size_t>(ext[2]) * elem, static_cast<size_t>(ext[1]), static_cast<size_t>(ext[0]));
		check_cuda(cudaMemcpy3DPeerAsync(&p, s), "cudaMemcpy3DPeerAsync");
	}
}

// ---- executor ------------------------------------------------------------------------------

executor::executor(const executor_config& cfg) : cfg_(cfg), rng_state_(cfg.schedule_seed) {
	int n = 0;
	const cudaError_t e = cudaGetDeviceCount(&n);
	if(e != cudaSuccess || n == 0) throw execution_error("no CUDA device available for the B200 executor (" + std::string(cudaGetErrorString(e)) + ")");
	const int ng = cfg.num_gpus > 0 ? std::min(cfg.num_gpus, n) : n;
	gpus_.resize(static_cast<size_t>(ng));
	for(int g = 0; g < ng; ++g) {
		auto& G = gpus_[static_cast<size_t>(g)];
		G.ordinal = cfg.gpu_base + g;
		check_cuda(cudaSetDevice(G.ordinal), "cudaSetDevice");
		cudaMemPoolProps props{};
		props.allocType = cudaMemAllocationTypePinned;
		props.location.type = cudaMemLocationTypeDevice;
		props.location.id = G.ordinal;
		check_cuda(cudaMemPoolCreate(&G.pool, &props), "cudaMemPoolCreate");
		uint64_t threshold = std::numeric_limits<uint64_t>::max();
		check_cuda(cudaMemPoolSetAttribute(G.pool, cudaMemPoolAttrReleaseThreshold, &threshold), "cudaMemPoolSetAttribute");
		size_t free_b = 0, total_b = 0;
		check_cuda(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
		G.capacity = cfg.device_capacity ? cfg.device_capacity : static_cast<uint64_t>(static_cast<double>(free_b) * 0.9);
		check_cuda(cudaStreamCreateWithFlags(&G.service, cudaStreamNonBlocking), "cudaStreamCreate");
		check_cuda(cudaStreamCreateWithFlags(&G.timing, cudaStreamNonBlocking), "cudaStreamCreate");
		check_cuda(cudaStreamCreateWithFlags(&G.graph, cudaStreamNonBlocking), "cudaStreamCreate");
		check_cuda(cudaStreamCreateWithFlags(&G.h2d, cudaStreamNonBlocking), "cudaStreamCreate");
		check_cuda(cudaStreamCreateWithFlags(&G.d2h, cudaStreamNonBlocking), "cudaStreamCreate");
		for(auto& m : G.marks) check_cuda(cudaEventCreate(&m), "cudaEventCreate");
	}
	spill_ = cfg.host_capacity > 0;
	free_events_.resize(static_cast<size_t>(ng));
	peer_ok_.assign(static_cast<size_t>(ng * ng), 0);
	for(int a = 0; a < ng; ++a) {
		peer_ok_[static_cast<size_t>(a * ng + a)] = 1;
		for(int b = 0; b < ng; ++b) {
			if(a == b) continue;
			int can = 0;
			cudaDeviceCanAccessPeer(&can, ord(a), ord(b));
			if(!can) continue;
			peer_ok_[static_cast<size_t>(a * ng + b)] = 1; // kernels on a may store into b's pool
			cudaSetDevice(ord(a));
			const cudaError_t pe = cudaDeviceEnablePeerAccess(ord(b), 0);
			if(pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) check_cuda(pe, "cudaDeviceEnablePeerAccess");
			cudaGetLastError();
			// let kernels on `a` dereference chunks allocated from b's pool
			cudaMemAccessDesc d{};
			d.location.type = cudaMemLocationTypeDevice;
			d.location.id = ord(a);
			d.flags = cudaMemAccessFlagsProtReadWrite;
			check_cuda(cudaMemPoolSetAccess(gpus_[static_cast<size_t>(b)].pool, &d, 1), "cudaMemPoolSetAccess");
		}
	}
	const int nw = cfg.workers, nd = cfg.devices_per_worker;
	const int k = cfg.streams_per_device > 0 ? cfg.streams_per_device : 4;
	ldevs_.resize(static_cast<size_t>(nw * nd));
	wctr_.assign(static_cast<size_t>(nw), worker_counters{});
	dev_used_.assign(static_cast<size_t>(nw * nd), 0);
	dev_peak_.assign(static_cast<size_t>(nw * nd), 0);
	pins_.assign(static_cast<size_t>(nw * nd), {});
	pinned_bytes_.assign(static_cast<size_t>(nw * nd), 0);
	for(int w = 0; w < nw; ++w) {
		const bool local = cfg.local_workers < 0 || (w >= cfg.first_worker && w < cfg.first_worker + cfg.local_workers);
		for(int d = 0; d < nd; ++d) {
			auto& L = ldevs_[static_cast<size_t>(w * nd + d)];
			const int global_index = local && cfg.local_workers >= 0 ? (w - cfg.first_worker) * nd + d : w * nd + d;
			L.gpu = global_index % ng;
			if(!local) continue;
			check_cuda(cudaSetDevice(ord(L.gpu)), "cudaSetDevice");
			L.compute.resize(static_cast<size_t>(k));
			for(auto& s : L.compute) check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
			check_cuda(cudaStreamCreateWithFlags(&L.copy, cudaStreamNonBlocking), "cudaStreamCreate");
			check_cuda(cudaStreamCreateWithFlags(&L.recv, cudaStreamNonBlocking), "cudaStreamCreate");
			check_cuda(cudaStreamCreateWithFlags(&L.host_in, cudaStreamNonBlocking), "cudaStreamCreate");
			check_cuda(cudaStreamCreateWithFlags(&L.host_out, cudaStreamNonBlocking), "cudaStreamCreate");
		}
	}
}

executor::~executor() {
	for(auto& G : gpus_) {
		cudaSetDevice(G.ordinal);
		cudaDeviceSynchronize();
	}
	if(nccl_comm_ && g_nccl.comm_destroy) g_nccl.comm_destroy(static_cast<ncclComm_t>(nccl_comm_));
	// peers must have stopped writing into our mailbox (callers barrier before teardown)
	for(void* p : opened_) cudaIpcCloseMemHandle(p);
	if(mbox_) cudaFree(mbox_);
	if(link_ctr_) cudaFree(link_ctr_);
	for(auto& l : links_) {
		if(l.tx) cudaStreamDestroy(l.tx);
		if(l.rx) cudaStreamDestroy(l.rx);
	}
	for(auto& [id, b] : bufs_) {
		cudaSetDevice(ord(b.gpu));
		if(b.ptr) cudaFree(b.ptr); // pool memory: cudaFree is legal on stream-ordered allocations
		if(b.host) cudaFreeHost(b.host);
	}
	for(auto& [sz, blk] : host_free_) cudaFreeHost(blk.first);
	if(spill_fd_ >= 0) {
		::close(spill_fd_);
		::unlink(spill_path_.c_str());
	}
	std::set<cudaEvent_t> live; // replayed submissions share one completion event
	for(auto& [id, d] : done_) live.insert(d.ev);
	for(auto e : live) cudaEventDestroy(e);
	for(auto& [sig, g] : graphs_)
		if(g.exec) cudaGraphExecDestroy(g.exec);
	for(auto& r : trace_recs_) {
		if(r.t0) cudaEventDestroy(r.t0);
		if(r.t1) cudaEventDestroy(r.t1);
	}
	for(auto e : trace_base_)
		if(e) cudaEventDestroy(e);
	for(auto& pool : free_events_)
		for(auto ev : pool) cudaEventDestroy(ev);
	for(auto& L : ldevs_) {
		for(auto s : L.compute) cudaStreamDestroy(s);
		if(L.copy) cudaStreamDestroy(L.copy);
		if(L.recv) cudaStreamDestroy(L.recv);
		if(L.host_in) cudaStreamDestroy(L.host_in);
		if(L.host_out) cudaStreamDestroy(L.host_out);
	}
	for(auto& G : gpus_) {
		cudaSetDevice(G.ordinal);
		cudaDeviceSynchronize();
		if(G.service) cudaStreamDestroy(G.service);
		if(G.timing) cudaStreamDestroy(G.timing);
		if(G.graph) cudaStreamDestroy(G.graph);
		if(G.h2d) cudaStreamDestroy(G.h2d);
		if(G.d2h) cudaStreamDestroy(G.d2h);
		for(auto m : G.marks)
			if(m) cudaEventDestroy(m);
		if(G.pool) cudaMemPoolDestroy(G.pool);
	}
}

int executor::gpu_of(device_id d) const { return ldevs_.at(static_cast<size_t>(d.worker * cfg_.devices_per_worker + d.device)).gpu; }

executor::ldev& executor::dev(device_id d) {
	if(d.worker < 0 || d.worker >= cfg_.workers || d.device < 0 || d.device >= cfg_.devices_per_worker)
		throw validation_error("task routed to unknown device " + to_string(d));
	auto& L = ldevs_[static_cast<size_t>(d.worker * cfg_.devices_per_worker + d.device)];
	if(L.compute.empty()) throw validation_error("device " + to_string(d) + " is not executed by this process");
	check_cuda(cudaSetDevice(ord(L.gpu)), "cudaSetDevice");
	return L;
}

executor::buffer& executor::buf(int64_t chunk) {
	const auto it = bufs_.find(chunk);
	if(it == bufs_.end()) throw execution_error("no buffer for chunk " + std::to_string(chunk));
	return it->second;
}

cudaEvent_t executor::take_event(int gpu) {
	auto& pool = free_events_[static_cast<size_t>(gpu)];
	if(!pool.empty()) {
		cudaEvent_t ev = pool.back();
		pool.pop_back();
		return ev;
	}
	cudaEvent_t ev = nullptr;
	check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
	return ev;
}

void executor::wait_deps(const task& t, cudaStream_t s) {
	for(const auto d : t.deps) {
		if(capturing_ && d < capture_first_) continue; // satisfied before the graph launch (replay)
		const auto it = done_.find(d);
		if(it == done_.end() || it->second.stream == s) continue;
		check_cuda(cudaStreamWaitEvent(s, it->second.ev, 0), "cudaStreamWaitEvent");
	}
	for(auto ev : stage_waits_) check_cuda(cudaStreamWaitEvent(s, ev, 0), "cudaStreamWaitEvent");
	stage_waits_.clear();
	if(trace_) {
		int cur = 0;
		cudaGetDevice(&cur);
		trace_rec r{t.id, t.worker, t.kind, cur - cfg_.gpu_base};
		check_cuda(cudaEventCreate(&r.t0), "cudaEventCreate");
		check_cuda(cudaEventRecord(r.t0, s), "cudaEventRecord");
		trace_open_[t.id] = trace_recs_.size();
		trace_recs_.push_back(r);
	}
}

void executor::set_trace(bool on) {
	if(on && !trace_) {
		trace_base_.assign(gpus_.size(), nullptr);
		for(size_t g = 0; g < gpus_.size(); ++g) {
			check_cuda(cudaSetDevice(gpus_[g].ordinal), "cudaSetDevice");
			check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
			check_cuda(cudaEventCreate(&trace_base_[g]), "cudaEventCreate");
			check_cuda(cudaEventRecord(trace_base_[g], gpus_[g].timing), "cudaEventRecord");
			check_cuda(cudaEventSynchronize(trace_base_[g]), "cudaEventSynchronize");
		}
	}
	trace_ = on;
}

namespace {
__global__ void delay_kernel(uint32_t ns) {
	const uint64_t until = [] {
		uint64_t t;
		asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
		return t;
	}() + ns;
	for(;;) {
		uint64_t now;
		asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
		if(now >= until) break;
		__nanosleep(256);
	}
}
} // namespace

uint64_t executor::next_random() { // splitmix64
	uint64_t z = (rng_state_ += 0x9e3779b97f4a7c15ull);
	z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
	z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
	return z ^ (z >> 31);
}

// Seeded schedule perturbation: half of the tasks wait 0-40 us on the device before they
// start, so ready work on different streams and devices completes in a different order per
// seed (the reference picks a random ready task per step, runtime.cpp:313-319).
void executor::perturb(cudaStream_t s) {
	if(!cfg_.schedule_seed) return;
	const uint64_t r = next_random();
	if(r & 1) return;
	delay_kernel<<<1, 1, 0, s>>>(static_cast<uint32_t>((r >> 8) % 40000));
	check_cuda(cudaGetLastError(), "delay kernel");
}

cudaStream_t executor::pick_compute(const task& t, ldev& L) {
	if(cfg_.schedule_seed) {
		cudaStream_t s = L.compute[next_random() % L.compute.size()];
		perturb(s);
		return s;
	}
	int64_t best = -1;
	cudaStream_t chosen = nullptr;
	for(const auto d : t.deps) {
		const auto it = done_.find(d);
		if(it == done_.end() || d < best) continue;
		for(auto s : L.compute) {
			if(s == it->second.stream && tail_[s] == d) {
				best = d;
				chosen = s;
			}
		}
	}
	if(chosen) return chosen;
	return L.compute[L.rr++ % L.compute.size()];
}

void executor::finish(const task& t, cudaStream_t s) {
	int cur = 0;
	cudaGetDevice(&cur);
	cur -= cfg_.gpu_base; // ordinal -> executor GPU index
	cudaEvent_t ev = take_event(cur);
	check_cuda(cudaEventRecord(ev, s), "cudaEventRecord");
	done_[t.id] = {ev, s, cur};
	tail_[s] = t.id;
	++ctr_.tasks;
	if(trace_) {
		const auto it = trace_open_.find(t.id);
		if(it != trace_open_.end()) {
			auto& r = trace_recs_[it->second];
			check_cuda(cudaEventCreate(&r.t1), "cudaEventCreate");
			check_cuda(cudaEventRecord(r.t1, s), "cudaEventRecord");
			trace_open_.erase(it);
		}
	}
	if(done_.size() > 16384 && !capturing_) retire_completed();
}

void executor::retire_completed() {
	for(auto it = done_.begin(); it != done_.end();) {
		if(cudaEventQuery(it->second.ev) == cudaSuccess) {
			release_done_event(it->second.ev, it->second.gpu);
			it = done_.erase(it);
		} else {
			++it;
		}
	}
	cudaGetLastError();
}

void executor::submit(const std::vector<task>& tasks) {
	for(const auto& t : tasks) submit_one(t);
	end_submit();
}

void executor::submit_one(const task& t) {
	if(t.id <= last_id_) throw validation_error("tasks must be submitted in ascending id order");
	last_id_ = t.id;
	if(cfg_.local_workers >= 0 && (t.worker < cfg_.first_worker || t.worker >= cfg_.first_worker + cfg_.local_workers)) return;
	if(spill_)
		queue_.push_back(t);
	else if(graphs_on_ && !trace_ && !profile_)
		gbatch_.push_back(t);
	else
		issue(t);
}

void executor::end_submit() {
	if(spill_) drain(false);
	issue_batch();
}

void executor::plan_mirrors(const std::vector<task>& b) {
	mirror_plan_.clear();
	if(!fusion_on_ || spill_ || trace_ || cfg_.staging_threshold || cfg_.schedule_seed) return;
	std::unordered_map<int64_t, const task*> execs;
	for(const auto& t : b)
		if(t.kind == task_kind::execute && t.kern && t.kern->mirror_param >= 0) execs[t.id] = &t;
	if(execs.empty()) return;
	const int ng = static_cast<int>(gpus_.size());
	for(const auto& c : b) {
		if(c.kind != task_kind::copy) continue;
		const task* e = nullptr;
		for(const auto d : c.deps) {
			const auto it = execs.find(d);
			if(it == execs.end()) continue;
			const auto& arg = it->second->args[static_cast<size_t>(it->second->kern->mirror_param)];
			if(arg.kind == arg_kind::chunk && arg.chunk == c.src && (arg.access & 2)) e = it->second;
		}
		if(!e) continue;
		bool aliased = false; // the kernel must not store into a chunk it also reads or writes
		for(const auto& arg : e->args)
			if(arg.kind == arg_kind::chunk && arg.chunk == c.dst) aliased = true;
		if(aliased) continue;
		bool older = true; // E may wait for C's other dependencies without reordering anything
		for(const auto d : c.deps)
			if(d != e->id && d >= e->id) older = false;
		const auto s = bufs_.find(c.src), d = bufs_.find(c.dst);
		if(!older || s == bufs_.end() || d == bufs_.end() || !s->second.ptr || !d->second.ptr || s->second.type != d->second.type) continue;
		if(d->second.gpu < 0 || d->second.gpu >= ng || !peer_ok_[static_cast<size_t>(s->second.gpu * ng + d->second.gpu)]) continue;
		auto& v = mirror_plan_[e->id];
		if(v.size() < 4) v.push_back(&c);
	}
}

void executor::issue_batch() {
	if(gbatch_.empty()) return;
	std::vector<task> b;
	b.swap(gbatch_);
	plan_mirrors(b);
	struct clear_plan {
		executor* x;
		~clear_plan() { x->mirror_plan_.clear(); }
	} clear{this};
	int gpu = -1;
	if(graph_eligible(b, &gpu)) {
		const std::string sig = signature(b);
		auto it = graphs_.find(sig);
		if(it == graphs_.end() && ++sig_seen_[sig] >= 2 && graphs_.size() < 256) {
			graph_entry g;
			if(capture(b, gpu, g)) it = graphs_.emplace(sig, g).first;
			else sig_seen_[sig] = -1000000; // not capturable: never try again
		}
		if(it != graphs_.end()) {
			replay(it->second, b);
			return;
		}
		if(sig_seen_.size() > 4096) sig_seen_.clear();
	}
	for(const auto& t : b) issue(t);
}

bool executor::graph_eligible(const std::vector<task>& b, int* gpu) const {
	if(spill_ || trace_ || profile_ || cfg_.schedule_seed || cfg_.staging_threshold) return false;
	// Only submissions whose GPU work is short enough that issuing them costs as much as running
	// them: consecutive replays run back to back on one stream, which gives up the overlap
	// between submissions that the multi-stream path keeps for large superblocks.
	static const double max_threads = [] {
		const char* e = std::getenv("MTB_GRAPH_MAX_THREADS");
		return e ? std::atof(e) : 268435456.0; // 2^28: e.g. ten 4096^2 launches in one flush
	}();
	double threads = 0;
	for(const auto& t : b)
		if(t.kind == task_kind::execute) threads += static_cast<double>(t.sb_threads.volume());
	if(threads > max_threads) return false;
	int g = -1;
	for(const auto& t : b) {
		if(t.kind != task_kind::execute && t.kind != task_kind::copy) return false;
		const auto chunk_gpu = [&](int64_t c) {
			const auto it = bufs_.find(c);
			return it == bufs_.end() || !it->second.ptr ? -1 : it->second.gpu;
		};
		int tg;
		if(t.kind == task_kind::execute) {
			if(t.device.worker < 0 || t.device.worker >= cfg_.workers || t.device.device < 0 || t.device.device >= cfg_.devices_per_worker) return false;
			const auto& L = ldevs_[static_cast<size_t>(t.device.worker * cfg_.devices_per_worker + t.device.device)];
			if(L.compute.empty() || !t.kern) return false;
			tg = L.gpu;
			for(const auto& a : t.args)
				if(a.kind == arg_kind::chunk && chunk_gpu(a.chunk) != tg) return false;
		} else {
			tg = chunk_gpu(t.dst);
			if(tg < 0 || chunk_gpu(t.src) != tg) return false;
		}
		if(g >= 0 && tg != g) return false;
		g = tg;
	}
	*gpu = g;
	return g >= 0;
}

std::string executor::signature(const std::vector<task>& b) const {
	std::string s;
	s.reserve(b.size() * 192);
	const auto put = [&](const void* p, size_t n) { s.append(static_cast<const char*>(p), n); };
	const auto put_box = [&](const box& r) {
		const int k = r.rank();
		put(&k, sizeof k);
		for(int d = 0; d < k; ++d) {
			const int64_t lo = r.lo[d], hi = r.hi[d];
			put(&lo, 8);
			put(&hi, 8);
		}
	};
	const int64_t first = b.front().id;
	for(const auto& t : b) {
		const int64_t rel = t.id - first;
		put(&rel, 8);
		put(&t.kind, sizeof t.kind);
		put(&t.resource, sizeof t.resource);
		for(const auto d : t.deps)
			if(d >= first) {
				const int64_t r = d - first;
				put(&r, 8);
			}
		const int64_t sep = -1;
		put(&sep, 8);
		if(t.kind == task_kind::execute) {
			put(&t.kern, sizeof t.kern);
			put(&t.device, sizeof t.device);
			put_box(t.sb_blocks);
			put_box(t.sb_threads);
			put_box(box(t.block_size, t.block_size));
			for(const auto& a : t.args) {
				put(&a.kind, sizeof a.kind);
				put(&a.i, 8);
				put(&a.f, 8);
				put(&a.chunk, 8);
			}
		} else {
			put(&t.src, 8);
			put(&t.dst, 8);
			put_box(t.src_region);
			put_box(t.dst_region);
		}
	}
	return s;
}

bool executor::capture(const std::vector<task>& b, int gpu, graph_entry& out) {
	auto& G = gpus_[static_cast<size_t>(gpu)];
	check_cuda(cudaSetDevice(G.ordinal), "cudaSetDevice");
	std::vector<cudaStream_t> streams;
	for(const auto& L : ldevs_)
		if(L.gpu == gpu && !L.compute.empty()) {
			streams.insert(streams.end(), L.compute.begin(), L.compute.end());
			streams.push_back(L.copy);
		}
	const exec_counters before = ctr_;
	const auto tail_before = tail_;
	cudaGraph_t graph = nullptr;
	std::vector<cudaEvent_t> used; // events recorded inside the capture go back to the pool
	bool ok = cudaStreamBeginCapture(G.graph, cudaStreamCaptureModeRelaxed) == cudaSuccess;
	if(ok) {
		capturing_ = true;
		capture_first_ = b.front().id;
		try {
			cudaEvent_t fork = take_event(gpu);
			used.push_back(fork);
			check_cuda(cudaEventRecord(fork, G.graph), "cudaEventRecord (fork)");
			for(auto st : streams) check_cuda(cudaStreamWaitEvent(st, fork, 0), "cudaStreamWaitEvent (fork)");
			for(const auto& t : b) issue(t);
			for(auto st : streams) {
				cudaEvent_t j = take_event(gpu);
				used.push_back(j);
				check_cuda(cudaEventRecord(j, st), "cudaEventRecord (join)");
				check_cuda(cudaStreamWaitEvent(G.graph, j, 0), "cudaStreamWaitEvent (join)");
			}
		} catch(const std::exception&) {
			ok = false;
		}
		capturing_ = false;
		const cudaError_t e = cudaStreamEndCapture(G.graph, &graph);
		ok = ok && e == cudaSuccess && graph;
	}
	cudaGetLastError();
	if(ok) ok = cudaGraphInstantiate(&out.exec, graph, 0) == cudaSuccess;
	cudaGetLastError();
	if(graph) cudaGraphDestroy(graph);
	// nothing of the submission ran: forget the capture-time completion records
	for(const auto& t : b) {
		const auto it = done_.find(t.id);
		if(it == done_.end()) continue;
		used.push_back(it->second.ev);
		done_.erase(it);
	}
	for(auto e : used) free_events_[static_cast<size_t>(gpu)].push_back(e);
	tail_ = tail_before;
	out.gpu = gpu;
	out.tasks = static_cast<int64_t>(ctr_.tasks - before.tasks);
	out.kernels = static_cast<int64_t>(ctr_.kernels - before.kernels);
	out.copies = static_cast<int64_t>(ctr_.copies - before.copies);
	out.bytes_copied = ctr_.bytes_copied - before.bytes_copied;
	out.fused_copies = static_cast<int64_t>(ctr_.fused_copies - before.fused_copies);
	out.bytes_fused = ctr_.bytes_fused - before.bytes_fused;
	ctr_ = before;
	if(ok) ++ctr_.graph_captures;
	return ok;
}

void executor::replay(const graph_entry& g, const std::vector<task>& b) {
	auto& G = gpus_[static_cast<size_t>(g.gpu)];
	check_cuda(cudaSetDevice(G.ordinal), "cudaSetDevice");
	const int64_t first = b.front().id;
	for(const auto& t : b)
		for(const auto d : t.deps) {
			if(d >= first) continue;
			const auto it = done_.find(d);
			if(it == done_.end() || it->second.stream == G.graph) continue;
			check_cuda(cudaStreamWaitEvent(G.graph, it->second.ev, 0), "cudaStreamWaitEvent");
		}
	nvtx3::scoped_range_in<nvtx_domain> range{"graph replay"};
	check_cuda(cudaGraphLaunch(g.exec, G.graph), "cudaGraphLaunch");
	cudaEvent_t ev = take_event(g.gpu);
	check_cuda(cudaEventRecord(ev, G.graph), "cudaEventRecord");
	shared_ev_[ev] = static_cast<int>(b.size());
	for(const auto& t : b) {
		const auto old = done_.find(t.id);
		if(old != done_.end()) release_done_event(old->second.ev, old->second.gpu);
		done_[t.id] = {ev, G.graph, g.gpu};
		tail_[G.graph] = t.id;
	}
	last_exec_stream_ = G.graph;
	ctr_.tasks += static_cast<uint64_t>(g.tasks);
	ctr_.kernels += static_cast<uint64_t>(g.kernels);
	ctr_.copies += static_cast<uint64_t>(g.copies);
	ctr_.bytes_copied += g.bytes_copied;
	ctr_.fused_copies += static_cast<uint64_t>(g.fused_copies);
	ctr_.bytes_fused += g.bytes_fused;
	++ctr_.graph_replays;
	if(done_.size() > 16384) retire_completed();
}

void executor::release_done_event(cudaEvent_t ev, int gpu) {
	const auto it = shared_ev_.find(ev);
	if(it != shared_ev_.end()) {
		if(--it->second > 0) return;
		shared_ev_.erase(it);
	}
	free_events_[static_cast<size_t>(gpu)].push_back(ev);
}

void executor::drain(bool all) {
	while(!queue_.empty() && (all || static_cast<int>(queue_.size()) > cfg_.lookahead)) {
		task t = std::move(queue_.front());
		queue_.pop_front();
		issue(t);
	}
}

void executor::charge(const buffer& b, uint64_t bytes, bool add) {
	auto& G = gpus_[static_cast<size_t>(b.gpu)];
	const size_t d = static_cast<size_t>(b.home.worker * cfg_.devices_per_worker + b.home.device);
	if(add) {
		G.used += bytes;
		ctr_.peak_device_bytes = std::max(ctr_.peak_device_bytes, G.used);
		dev_used_[d] += bytes;
		dev_peak_[d] = std::max(dev_peak_[d], dev_used_[d]);
	} else {
		G.used -= bytes;
		dev_used_[d] -= bytes;
	}
}

// Staging throttle (memory.cpp:290-295) and its safety monitor (memory.cpp:371-374). The
// reference stages a task only if the union of chunks pinned by staged-but-unfinished tasks on
// its resource stays within the threshold; here "staged" is "issued to a stream and not yet
// complete", and a task that would exceed it waits on the host for the oldest in-flight tasks.
// A single task whose chunks alone exceed the threshold is the reference's fatal error
// (memory.cpp:278-281). The monitor counts one check per admitted task and a violation for
// every device over the threshold at that moment (by construction none).
void executor::throttle(const task& t) {
	const uint64_t thr = cfg_.staging_threshold;
	std::vector<std::pair<int64_t, bool>> uses;
	used_chunks(t, uses);
	staged_task st{t.id, static_cast<size_t>(t.resource.worker * cfg_.devices_per_worker + t.resource.device), {}};
	const auto add = [&](int64_t c, uint64_t bytes) {
		for(const auto& x : st.chunks)
			if(x.first == c) return;
		st.chunks.emplace_back(c, bytes);
	};
	if(t.kind == task_kind::create) add(t.chunk, static_cast<uint64_t>(t.region.volume()) * dtype_size(t.type));
	for(const auto& [c, w] : uses) {
		const auto it = bufs_.find(c);
		if(it != bufs_.end()) add(c, it->second.bytes);
	}
	uint64_t footprint = 0;
	for(const auto& x : st.chunks) footprint += x.second;
	if(footprint > thr)
		throw execution_error("task " + std::to_string(t.id) + " footprint " + std::to_string(footprint) + " exceeds the staging threshold " + std::to_string(thr));
	auto& pins = pins_[st.dev];
	const auto fresh = [&] {
		uint64_t n = 0;
		for(const auto& [c, b] : st.chunks)
			if(!pins.count(c)) n += b;
		return n;
	};
	const auto complete = [&](int64_t id) {
		const auto it = done_.find(id);
		return it == done_.end() || cudaEventQuery(it->second.ev) == cudaSuccess;
	};
	while(!staged_.empty() && complete(staged_.front().id)) {
		unpin(staged_.front());
		staged_.pop_front();
	}
	while(pinned_bytes_[st.dev] + fresh() > thr && !staged_.empty()) {
		const auto it = done_.find(staged_.front().id);
		if(it != done_.end()) check_cuda(cudaEventSynchronize(it->second.ev), "cudaEventSynchronize (staging throttle)");
		unpin(staged_.front());
		staged_.pop_front();
		while(!staged_.empty() && complete(staged_.front().id)) {
			unpin(staged_.front());
			staged_.pop_front();
		}
	}
	cudaGetLastError();
	for(const auto& [c, b] : st.chunks)
		if(pins[c]++ == 0) pinned_bytes_[st.dev] += b;
	auto& w = wc(t.resource.worker);
	++w.staging_checks;
	for(const auto bytes : pinned_bytes_)
		if(bytes > thr) ++w.staging_violations;
	staged_.push_back(std::move(st));
}

void executor::unpin(const staged_task& st) {
	auto& pins = pins_[st.dev];
	for(const auto& [c, b] : st.chunks) {
		const auto it = pins.find(c);
		if(it == pins.end()) continue;
		if(--it->second == 0) {
			pins.erase(it);
			pinned_bytes_[st.dev] -= b;
		}
	}
}

void executor::issue(const task& t) {
	if(t.kind == task_kind::copy) {
		const auto it = mirrored_.find(t.id);
		if(it != mirrored_.end()) { // stored by its producing kernel, completion already recorded
			mirrored_.erase(it);
			return;
		}
	}
	nvtx3::scoped_range_in<nvtx_domain> range{task_kind_name(t.kind)};
	if(cfg_.staging_threshold && !remote_worker(t.resource.worker)) throttle(t);
	if(spill_) stage(t);
	switch(t.kind) {
	case task_kind::create: run_create(t); break;
	case task_kind::del: run_delete(t); break;
	case task_kind::execute: run_execute(t); break;
	case task_kind::copy: run_copy(t); break;
	case task_kind::send: run_send(t); break;
	case task_kind::recv: run_recv(t); break;
	case task_kind::reduce: run_reduce(t); break;
	case task_kind::allreduce: run_allreduce(t); break;
	case task_kind::host_write:
	case task_kind::host_read: run_host_io(t); break;
	}
	if(spill_) note_use(t);
}

// ---- spill tier -------------------------------------------------------------------------------
//
// The reference stages every task through an LRU memory manager with unconditional write-back
// (memory.cpp:161-186, 245-377), which on a cyclic stencil sweep evicts exactly the chunk the
// next iteration needs first and moves 2.0-2.4x the minimum bytes. Here every
// decision is taken when a task is issued, with `lookahead` later tasks already known:
//   * victims are resident chunks the current task does not use, furthest next use first
//     (Belady/MIN over the lookahead window), clean ones (valid host copy) before dirty ones,
//     least recently used last;
//   * eviction = D2H on the GPU's d2h stream after every task that touched the chunk (only when
//     the host copy is stale: dirty tracking) + cudaFreeAsync; restoration = allocation on the
//     h2d stream after the latest eviction's free + H2D, and the using task waits on it;
//   * all of it is stream-ordered, so H2D, D2H and kernels overlap (full-duplex PCIe).

void executor::used_chunks(const task& t, std::vector<std::pair<int64_t, bool>>& out) const {
	out.clear();
	switch(t.kind) {
	case task_kind::create: break;
	case task_kind::del: out.emplace_back(t.chunk, true); break;
	case task_kind::execute:
		for(size_t i = 0; i < t.args.size(); ++i) {
			if(t.args[i].kind != arg_kind::chunk) continue;
			const bool w = t.kern && i < t.kern->params.size() && t.kern->params[i].writable;
			out.emplace_back(t.args[i].chunk, w);
		}
		break;
	case task_kind::copy:
		out.emplace_back(t.src, false);
		out.emplace_back(t.dst, true);
		break;
	case task_kind::send: out.emplace_back(t.chunk, false); break;
	case task_kind::recv: out.emplace_back(t.chunk, true); break;
	case task_kind::reduce:
		for(const auto c : t.inputs) out.emplace_back(c, false);
		out.emplace_back(t.output, true);
		break;
	case task_kind::host_write: out.emplace_back(t.chunk, true); break;
	case task_kind::host_read: out.emplace_back(t.chunk, false); break;
	case task_kind::allreduce: {
		// the last local member combines every member: keep them all resident
		for(const auto c : t.inputs)
			if(bufs_.count(c)) out.emplace_back(c, false);
		const auto g = groups_.find(t.tag);
		if(g != groups_.end())
			for(const auto c : g->second.outputs) out.emplace_back(c, true);
		out.emplace_back(t.output, true);
		break;
	}
	}
}

void executor::accesses_of(const task& t, std::vector<access_t>& out) const {
	out.clear();
	const auto full = [&](int64_t c) {
		const auto it = bufs_.find(c);
		return it == bufs_.end() ? box() : it->second.region;
	};
	switch(t.kind) {
	case task_kind::create: out.push_back({t.chunk, t.region, false, true, false}); break;
	case task_kind::del: out.push_back({t.chunk, full(t.chunk), false, false, true}); break;
	case task_kind::execute:
		for(size_t i = 0; i < t.args.size(); ++i) {
			const auto& a = t.args[i];
			if(a.kind != arg_kind::chunk) continue;
			const box whole = full(a.chunk);
			const bool known = a.access != 0 && whole.rank() == a.region.rank();
			const box r = known ? intersect(a.region, whole) : whole;
			// a trailing partial block's threads outside the grid write nothing (the kernels
			// guard on their extents), so such a superblock's region is not fully overwritten
			const bool dense = t.kern && t.kern->dense_writes && t.sb_inside_grid;
			const bool overwrite = known && (a.access & 2) && !(a.access & 1) && dense;
			out.push_back({a.chunk, r, !overwrite, overwrite, false});
		}
		break;
	case task_kind::copy:
		out.push_back({t.src, t.src_region, true, false, false});
		out.push_back({t.dst, t.dst_region, false, true, false});
		break;
	case task_kind::send: out.push_back({t.chunk, t.region, true, false, false}); break;
	case task_kind::recv: out.push_back({t.chunk, t.region, false, true, false}); break;
	case task_kind::reduce:
		for(const auto c : t.inputs) out.push_back({c, full(c), true, false, false});
		out.push_back({t.output, full(t.output), false, true, false});
		break;
	case task_kind::host_write: out.push_back({t.chunk, t.region, false, true, false}); break;
	case task_kind::host_read: out.push_back({t.chunk, t.region, true, false, false}); break;
	case task_kind::allreduce:
		for(const auto c : t.inputs)
			if(c != t.output && bufs_.count(c)) out.push_back({c, full(c), true, false, false});
		out.push_back({t.output, full(t.output), true, false, false}); // in place: read and written
		break;
	}
}

bool executor::dead_ahead(int64_t chunk, const task* first) const {
	const auto it = bufs_.find(chunk);
	if(it == bufs_.end()) return false;
	std::vector<box> live{it->second.region};
	std::vector<access_t> accs;
	const auto step = [&](const task& t) -> int {
		accesses_of(t, accs);
		for(const auto& a : accs)
			if(a.chunk == chunk && a.kill) return 1;
		for(const auto& a : accs) {
			if(a.chunk != chunk || !a.read || a.region.is_empty()) continue;
			for(const auto& l : live)
				if(overlaps(l, a.region)) return -1;
		}
		for(const auto& a : accs) {
			if(a.chunk != chunk || !a.overwrite || a.region.is_empty()) continue;
			std::vector<box> next;
			for(const auto& l : live) {
				if(!overlaps(l, a.region)) {
					next.push_back(l);
					continue;
				}
				box rest = l; // l minus a.region, slab by slab
				for(int k = 0; k < rest.rank(); ++k) {
					if(rest.lo[k] < a.region.lo[k]) {
						box piece = rest;
						piece.hi[k] = a.region.lo[k];
						next.push_back(piece);
						rest.lo[k] = a.region.lo[k];
					}
					if(a.region.hi[k] < rest.hi[k]) {
						box piece = rest;
						piece.lo[k] = a.region.hi[k];
						next.push_back(piece);
						rest.hi[k] = a.region.hi[k];
					}
				}
			}
			live.swap(next);
		}
		return live.empty() ? 1 : 0;
	};
	if(first) {
		const int r = step(*first);
		if(r != 0) return r > 0;
	}
	for(const auto& t : queue_) {
		const int r = step(t);
		if(r != 0) return r > 0;
	}
	return false; // unknown beyond the window: keep the data
}

// An allocation under memory pressure reuses memory freed by an eviction kFreeLag evictions
// back rather than the one just issued, so the H2D of a restore overlaps the D2H of the
// eviction that made room for it (full-duplex PCIe); the device keeps kFreeLag chunks of
// physical headroom above the logical capacity.
constexpr size_t kFreeLag = 2;

cudaEvent_t executor::alloc_event(int gpu) const {
	const auto& G = gpus_[static_cast<size_t>(gpu)];
	if(G.frees.size() <= kFreeLag) return nullptr;
	return G.frees[G.frees.size() - 1 - kFreeLag];
}

void executor::alloc_wait(int gpu, cudaStream_t s) {
	if(cudaEvent_t e = alloc_event(gpu)) check_cuda(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent");
}

void* executor::host_alloc(uint64_t bytes, int gpu, int64_t exclude) {
	auto it = host_free_.find(bytes);
	if(it != host_free_.end()) {
		auto [p, ev] = it->second;
		host_free_.erase(it);
		// the block's previous owner may still be read by an in-flight H2D: D2H waits for it
		if(ev) {
			check_cuda(cudaStreamWaitEvent(gpus_[static_cast<size_t>(gpu)].d2h, ev, 0), "cudaStreamWaitEvent");
			cudaEventDestroy(ev);
		}
		return p;
	}
	// over capacity: take back host copies of chunks that are resident again — stale ones
	// (written since) first, then clean ones (their next eviction writes back again)
	while(host_used_ + bytes > cfg_.host_capacity) {
		buffer* pick = nullptr;
		for(auto& [id, b] : bufs_) {
			// resident chunks' copies, and blocks of evicted chunks whose data was dropped as dead
			if(id == exclude || !b.host || (!b.ptr && b.host_valid)) continue;
			const bool better = !pick || (pick->host_valid && !b.host_valid) || (pick->host_valid == b.host_valid && (pick->bytes != bytes && b.bytes == bytes));
			if(better) pick = &b;
		}
		if(!pick && cfg_.disk_capacity > 0) {
			if(void* blk = spill_host_to_disk(bytes, exclude)) return blk;
			continue; // a block of another size went to disk and was freed
		}
		if(!pick)
			throw execution_error("host tier exhausted: " + std::to_string(host_used_ + bytes) + " bytes needed, capacity " + std::to_string(cfg_.host_capacity));
		void* blk = pick->host;
		const uint64_t sz = pick->bytes;
		pick->host = nullptr;
		pick->host_valid = false;
		// an H2D restore may still be reading the block
		auto& H = gpus_[static_cast<size_t>(pick->gpu)];
		cudaEvent_t after = nullptr;
		check_cuda(cudaEventCreateWithFlags(&after, cudaEventDisableTiming), "cudaEventCreate");
		check_cuda(cudaEventRecord(after, H.h2d), "cudaEventRecord");
		if(sz == bytes) {
			check_cuda(cudaStreamWaitEvent(gpus_[static_cast<size_t>(gpu)].d2h, after, 0), "cudaStreamWaitEvent");
			cudaEventDestroy(after);
			++ctr_.host_reclaims;
			return blk;
		}
		check_cuda(cudaEventSynchronize(after), "cudaEventSynchronize");
		cudaEventDestroy(after);
		check_cuda(cudaFreeHost(blk), "cudaFreeHost");
		host_used_ -= sz;
		++ctr_.host_reclaims;
	}
	void* p = nullptr;
	check_cuda(cudaHostAlloc(&p, bytes, cudaHostAllocPortable), "cudaHostAlloc");
	host_used_ += bytes;
	return p;
}

void executor::host_release(void* p, uint64_t bytes, cudaEvent_t after) { host_free_.emplace(bytes, std::make_pair(p, after)); }

uint64_t executor::disk_alloc(uint64_t bytes) {
	if(spill_fd_ < 0) {
		const char* dir = cfg_.spill_dir.empty() ? (std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") : cfg_.spill_dir.c_str();
		std::string tmpl = std::string(dir) + "/manta-b200-spill-XXXXXX";
		std::vector<char> path(tmpl.begin(), tmpl.end());
		path.push_back('\0');
		spill_fd_ = ::mkstemp(path.data());
		if(spill_fd_ < 0) throw execution_error("cannot create spill file in " + std::string(dir));
		spill_path_ = path.data();
	}
	auto it = disk_free_.find(bytes);
	if(it == disk_free_.end() && disk_end_ + bytes > cfg_.disk_capacity) it = disk_free_.lower_bound(bytes);
	if(it != disk_free_.end()) {
		const uint64_t off = it->second;
		disk_free_.erase(it);
		return off;
	}
	if(disk_end_ + bytes > cfg_.disk_capacity)
		throw execution_error("disk tier exhausted: " + std::to_string(bytes) + " more bytes, capacity " + std::to_string(cfg_.disk_capacity));
	const uint64_t off = disk_end_;
	disk_end_ += bytes;
	return off;
}

void executor::disk_release(buffer& b) {
	if(b.disk_off >= 0) disk_free_.emplace(b.bytes, static_cast<uint64_t>(b.disk_off));
	b.disk_off = -1;
	b.disk_valid = false;
}

void executor::disk_read(const buffer& b, void* dst) {
	uint64_t done = 0;
	while(done < b.bytes) {
		const ssize_t r = ::pread(spill_fd_, static_cast<char*>(dst) + done, b.bytes - done, static_cast<off_t>(b.disk_off + done));
		if(r <= 0) throw execution_error("spill read failed");
		done += static_cast<uint64_t>(r);
	}
	ctr_.bytes_disk_to_host += b.bytes;
	wc(b.home.worker).bytes_disk_to_host += b.bytes;
}

// The host tier is full and holds only copies of evicted chunks: write the least recently used
// one (same size as the request when possible) to the spill file and reuse or free its block.
void* executor::spill_host_to_disk(uint64_t bytes, int64_t exclude) {
	buffer* pick = nullptr;
	for(auto& [id, b] : bufs_) {
		if(id == exclude || b.ptr || !b.host || !b.host_valid) continue;
		const bool better = !pick || (pick->bytes != bytes && b.bytes == bytes) || ((pick->bytes == bytes) == (b.bytes == bytes) && b.last_use < pick->last_use);
		if(better) pick = &b;
	}
	if(!pick) throw execution_error("host tier exhausted and nothing left to spill to disk");
	buffer& b = *pick;
	if(b.evicted) check_cuda(cudaEventSynchronize(b.evicted), "cudaEventSynchronize"); // its D2H has landed
	if(!b.disk_valid) {
		if(b.disk_off < 0) b.disk_off = static_cast<int64_t>(disk_alloc(b.bytes));
		uint64_t done = 0;
		while(done < b.bytes) {
			const ssize_t w = ::pwrite(spill_fd_, static_cast<const char*>(b.host) + done, b.bytes - done, static_cast<off_t>(b.disk_off + done));
			if(w <= 0) throw execution_error("spill write failed");
			done += static_cast<uint64_t>(w);
		}
		b.disk_valid = true;
		ctr_.bytes_host_to_disk += b.bytes;
		wc(b.home.worker).bytes_host_to_disk += b.bytes;
	}
	void* blk = b.host;
	b.host = nullptr;
	b.host_valid = false;
	if(b.bytes == bytes) return blk;
	check_cuda(cudaFreeHost(blk), "cudaFreeHost");
	host_used_ -= b.bytes;
	return nullptr;
}

void executor::evict(int64_t chunk) {
	buffer& b = buf(chunk);
	auto& G = gpus_[static_cast<size_t>(b.gpu)];
	check_cuda(cudaSetDevice(ord(b.gpu)), "cudaSetDevice");
	for(const auto u : b.users) {
		const auto it = done_.find(u);
		if(it != done_.end()) check_cuda(cudaStreamWaitEvent(G.d2h, it->second.ev, 0), "cudaStreamWaitEvent");
	}
	if(b.restored) check_cuda(cudaStreamWaitEvent(G.d2h, b.restored, 0), "cudaStreamWaitEvent");
	if(!b.host_valid && !b.disk_valid && dead_ahead(chunk, nullptr)) {
		++ctr_.dead_drops; // overwritten before it is read again: no write-back
	} else if(!b.host_valid && !b.disk_valid) {
		if(!b.host) b.host = host_alloc(b.bytes, b.gpu, chunk);
		check_cuda(cudaMemcpyAsync(b.host, b.ptr, b.bytes, cudaMemcpyDeviceToHost, G.d2h), "cudaMemcpyAsync D2H (evict)");
		b.host_valid = true;
		ctr_.bytes_device_to_host += b.bytes;
		wc(b.home.worker).bytes_device_to_host += b.bytes;
	}
	check_cuda(cudaFreeAsync(b.ptr, G.d2h), "cudaFreeAsync");
	if(!b.evicted) check_cuda(cudaEventCreateWithFlags(&b.evicted, cudaEventDisableTiming), "cudaEventCreate");
	check_cuda(cudaEventRecord(b.evicted, G.d2h), "cudaEventRecord");
	cudaEvent_t fe = take_event(b.gpu);
	check_cuda(cudaEventRecord(fe, G.d2h), "cudaEventRecord");
	G.frees.push_back(fe);
	while(G.frees.size() > 4 * kFreeLag) {
		free_events_[static_cast<size_t>(b.gpu)].push_back(G.frees.front());
		G.frees.pop_front();
	}
	b.ptr = nullptr;
	b.users.clear();
	charge(b, b.bytes, false);
	++ctr_.evictions;
	++wc(b.home.worker).evictions;
}

void executor::ensure_room(int gpu, uint64_t bytes, const std::vector<int64_t>& pinned) {
	auto& G = gpus_[static_cast<size_t>(gpu)];
	if(bytes > G.capacity)
		throw execution_error("a chunk of " + std::to_string(bytes) + " bytes can never fit the device capacity " + std::to_string(G.capacity));
	if(G.used + bytes <= G.capacity) return;
	// next use of every chunk within the lookahead window (queue_ holds the future tasks) that
	// needs its data on the device: a read, or a write of part of it (a halo row: the rest must
	// be there). A chunk that is only overwritten ahead does not need its data kept (Belady on
	// data uses; the dead-data check below catches piecewise overwrites)
	std::unordered_map<int64_t, size_t> next;
	std::vector<access_t> accs;
	for(size_t i = 0; i < queue_.size(); ++i) {
		accesses_of(queue_[i], accs);
		for(const auto& a : accs) {
			if(next.count(a.chunk)) continue;
			if(a.read || a.kill) {
				if(!a.kill) next.emplace(a.chunk, i);
				continue;
			}
			const auto b = bufs_.find(a.chunk);
			if(!a.overwrite || b == bufs_.end()) continue;
			// a partial write needs the data; a whole-chunk overwrite ends its life
			next.emplace(a.chunk, intersect(a.region, b->second.region) == b->second.region ? SIZE_MAX : i);
		}
	}
	while(G.used + bytes > G.capacity) {
		int64_t victim = -1;
		size_t v_next = 0;
		bool v_clean = false;
		uint64_t v_last = 0;
		for(auto& [id, b] : bufs_) {
			if(b.gpu != gpu || !b.ptr || std::find(pinned.begin(), pinned.end(), id) != pinned.end()) continue;
			// data that is overwritten before it is read again is worth nothing: never-needed,
			// and free to drop (no write-back)
			const bool dead = !b.host_valid && dead_ahead(id, nullptr);
			const auto it = next.find(id);
			const size_t nu = dead || it == next.end() ? SIZE_MAX : it->second;
			const bool free_drop = dead || b.host_valid;
			const bool better = victim < 0 || nu > v_next || (nu == v_next && free_drop && !v_clean)
			                    || (nu == v_next && free_drop == v_clean && b.last_use < v_last);
			if(better) {
				victim = id;
				v_next = nu;
				v_clean = free_drop;
				v_last = b.last_use;
			}
		}
		if(victim < 0)
			throw execution_error("device " + std::to_string(gpu) + ": task footprint exceeds capacity " + std::to_string(G.capacity)
			                      + " with every resident chunk in use");
		if(std::getenv("MTB_SPILL_TRACE"))
			std::fprintf(stderr, "[spill] evict chunk %ld next_read %ld clean %d queue %zu used %lu cap %lu\n", static_cast<long>(victim),
			    v_next == SIZE_MAX ? -1L : static_cast<long>(v_next), v_clean ? 1 : 0, queue_.size(), static_cast<unsigned long>(G.used),
			    static_cast<unsigned long>(G.capacity));
		evict(victim);
	}
}

void executor::restore(int64_t chunk, const std::vector<int64_t>& pinned, const task& current) {
	buffer& b = buf(chunk);
	ensure_room(b.gpu, b.bytes, pinned);
	auto& G = gpus_[static_cast<size_t>(b.gpu)];
	check_cuda(cudaSetDevice(ord(b.gpu)), "cudaSetDevice");
	alloc_wait(b.gpu, G.h2d);
	check_cuda(cudaMallocFromPoolAsync(&b.ptr, b.bytes, G.pool, G.h2d), "cudaMallocFromPoolAsync (restore)");
	const bool needed = (b.host_valid || b.disk_valid) && !dead_ahead(chunk, &current);
	if(std::getenv("MTB_SPILL_TRACE"))
		std::fprintf(stderr, "[spill] restore chunk %ld for task %ld (%s) copy %d\n", static_cast<long>(chunk), static_cast<long>(current.id),
		    task_kind_name(current.kind), needed ? 1 : 0);
	if(!needed) {
		// contents are overwritten before they are read: allocate only
		charge(b, b.bytes, true);
		if(!b.restored) check_cuda(cudaEventCreateWithFlags(&b.restored, cudaEventDisableTiming), "cudaEventCreate");
		check_cuda(cudaEventRecord(b.restored, G.h2d), "cudaEventRecord");
		++ctr_.dead_skips;
		return;
	}
	if(b.evicted) check_cuda(cudaStreamWaitEvent(G.h2d, b.evicted, 0), "cudaStreamWaitEvent"); // its own write-back first
	if(!b.host_valid) {
		// the copy is on disk: bring it into a pinned block first (synchronous file read)
		if(!b.host) b.host = host_alloc(b.bytes, b.gpu, chunk);
		check_cuda(cudaStreamSynchronize(G.h2d), "cudaStreamSynchronize"); // the block's previous users
		check_cuda(cudaStreamSynchronize(G.d2h), "cudaStreamSynchronize");
		disk_read(b, b.host);
		b.host_valid = true;
	}
	check_cuda(cudaMemcpyAsync(b.ptr, b.host, b.bytes, cudaMemcpyHostToDevice, G.h2d), "cudaMemcpyAsync H2D (restore)");
	if(!b.restored) check_cuda(cudaEventCreateWithFlags(&b.restored, cudaEventDisableTiming), "cudaEventCreate");
	check_cuda(cudaEventRecord(b.restored, G.h2d), "cudaEventRecord");
	charge(b, b.bytes, true);
	ctr_.bytes_host_to_device += b.bytes;
	wc(b.home.worker).bytes_host_to_device += b.bytes;
}

void executor::stage(const task& t) {
	std::vector<std::pair<int64_t, bool>> uses;
	used_chunks(t, uses);
	std::vector<int64_t> pinned;
	for(const auto& [c, w] : uses) pinned.push_back(c);
	for(const auto& [c, w] : uses) {
		buffer& b = buf(c);
		if(!b.ptr) restore(c, pinned, t);
		if(b.restored) stage_waits_.push_back(b.restored);
	}
	if(t.kind == task_kind::create) {
		const uint64_t bytes = static_cast<uint64_t>(t.region.volume()) * dtype_size(t.type);
		ensure_room(gpu_of(t.home), bytes, pinned);
		if(cudaEvent_t e = alloc_event(gpu_of(t.home))) stage_waits_.push_back(e);
	}
}

void executor::note_use(const task& t) {
	std::vector<std::pair<int64_t, bool>> uses;
	used_chunks(t, uses);
	if(t.kind == task_kind::create) uses.emplace_back(t.chunk, true);
	++clock_;
	for(const auto& [c, w] : uses) {
		const auto it = bufs_.find(c);
		if(it == bufs_.end()) continue; // deleted by this task
		buffer& b = it->second;
		b.users.push_back(t.id);
		b.last_use = clock_;
		if(w) {
			b.host_valid = false;
			disk_release(b);
		}
		if(b.users.size() > 64) {
			std::vector<int64_t> keep;
			for(const auto u : b.users) {
				const auto d = done_.find(u);
				if(d != done_.end() && cudaEventQuery(d->second.ev) != cudaSuccess) keep.push_back(u);
			}
			cudaGetLastError();
			b.users.swap(keep);
		}
	}
}

void executor::run_create(const task& t) {
	ldev& L = dev(t.home);
	cudaStream_t s = pick_compute(t, L);
	wait_deps(t, s);
	auto& G = gpus_[static_cast<size_t>(L.gpu)];
	const uint64_t count = static_cast<uint64_t>(t.region.volume());
	const uint64_t bytes = count * dtype_size(t.type);
	if(bufs_.count(t.chunk)) throw execution_error("chunk " + std::to_string(t.chunk) + " created twice");
	if(G.used + bytes > G.capacity)
		throw execution_error("task " + std::to_string(t.id) + " needs " + std::to_string(bytes) + " bytes on GPU " + std::to_string(L.gpu) + " beyond its capacity "
		                      + std::to_string(G.capacity));
	void* p = nullptr;
	check_cuda(cudaMallocFromPoolAsync(&p, bytes, G.pool, s), "cudaMallocFromPoolAsync");
	device_fill(p, count, t.type, t.fill, t.fill_op, s);
	++ctr_.kernels;
	bufs_[t.chunk] = buffer{p, bytes, t.region, t.type, t.home, L.gpu};
	charge(bufs_[t.chunk], bytes, true);
	finish(t, s);
}

void executor::run_delete(const task& t) {
	buffer b = buf(t.chunk);
	ldev& L = dev(b.home);
	cudaStream_t s = pick_compute(t, L);
	wait_deps(t, s);
	if(b.ptr) {
		check_cuda(cudaFreeAsync(b.ptr, s), "cudaFreeAsync");
		charge(b, b.bytes, false);
	}
	if(b.host) {
		// the pinned block is reusable once every earlier use of the chunk is done
		cudaEvent_t after = nullptr;
		check_cuda(cudaEventCreateWithFlags(&after, cudaEventDisableTiming), "cudaEventCreate");
		check_cuda(cudaEventRecord(after, s), "cudaEventRecord");
		host_release(b.host, b.bytes, after);
	}
	if(b.restored) cudaEventDestroy(b.restored);
	if(b.evicted) cudaEventDestroy(b.evicted);
	disk_release(buf(t.chunk));
	bufs_.erase(t.chunk);
	finish(t, s);
}

void executor::run_execute(const task& t) {
	if(!t.kern) throw execution_error("execute task without a kernel");
	const kernel_entry& k = *t.kern;
	if(!k.launcher) throw execution_error("kernel \"" + k.id + "\" has no device launcher");
	ldev& L = dev(t.device);
	cudaStream_t s = pick_compute(t, L);
	wait_deps(t, s);
	// fused halo copies planned for this task: the kernel runs after their other dependencies too
	const auto mp = mirror_plan_.find(t.id);
	const std::vector<const task*>* fused = mp == mirror_plan_.end() ? nullptr : &mp->second;
	if(fused)
		for(const task* c : *fused)
			for(const auto d : c->deps) {
				if(d == t.id || (capturing_ && d < capture_first_)) continue;
				const auto it = done_.find(d);
				if(it == done_.end() || it->second.stream == s) continue;
				check_cuda(cudaStreamWaitEvent(s, it->second.ev, 0), "cudaStreamWaitEvent");
			}
	const size_t np = t.args.size();
	std::vector<int64_t> si(np, 0);
	std::vector<double> sf(np, 0.0);
	std::vector<mt_view> views(np);
	std::memset(views.data(), 0, np * sizeof(mt_view));
	for(size_t i = 0; i < np; ++i) {
		const auto& a = t.args[i];
		si[i] = a.i;
		sf[i] = a.f;
		if(a.kind != arg_kind::chunk) continue;
		const buffer& b = buf(a.chunk);
		if(b.gpu != L.gpu) throw execution_error("kernel argument chunk " + std::to_string(a.chunk) + " lives on another GPU");
		auto& v = views[i];
		v.base = b.ptr;
		v.dtype = static_cast<int32_t>(b.type);
		v.rank = b.region.rank();
		int64_t st[kMaxRank];
		strides_of(b.region, st);
		for(int d = 0; d < v.rank; ++d) {
			v.offset[d] = b.region.lo[d];
			v.stride[d] = st[d];
			v.extent[d] = b.region.extent(d);
		}
	}
	mt_launch_ctx c{};
	c.rank = t.sb_blocks.rank();
	c.nparams = static_cast<int32_t>(np);
	for(int d = 0; d < c.rank; ++d) {
		c.block_offset[d] = t.sb_blocks.lo[d];
		c.block_count[d] = t.sb_blocks.extent(d);
		c.block_size[d] = t.block_size[d];
		c.threads_lo[d] = t.sb_threads.lo[d];
		c.threads_hi[d] = t.sb_threads.hi[d];
	}
	c.scalars_int = si.data();
	c.scalars_float = sf.data();
	c.views = views.data();
	c.user = k.user;
	std::vector<mt_mirror> mirrors;
	std::vector<int32_t> applied;
	if(fused) {
		for(const task* cp : *fused) {
			const buffer& d = buf(cp->dst);
			mt_mirror m{};
			m.param = k.mirror_param;
			const int r = cp->dst_region.rank();
			for(int q = 0; q < r; ++q) {
				m.lo[q] = cp->dst_region.lo[q];
				m.hi[q] = cp->dst_region.hi[q];
			}
			m.dst.base = d.ptr;
			m.dst.dtype = static_cast<int32_t>(d.type);
			m.dst.rank = d.region.rank();
			int64_t st[kMaxRank];
			strides_of(d.region, st);
			for(int q = 0; q < m.dst.rank; ++q) {
				m.dst.offset[q] = d.region.lo[q];
				m.dst.stride[q] = st[q];
				m.dst.extent[q] = d.region.extent(q);
			}
			mirrors.push_back(m);
		}
		applied.assign(mirrors.size(), 0);
		c.nmirrors = static_cast<int32_t>(mirrors.size());
		c.mirrors = mirrors.data();
		c.mirror_applied = applied.data();
	}
	cudaEvent_t kt0 = nullptr, kt1 = nullptr;
	if(profile_) {
		check_cuda(cudaEventCreate(&kt0), "cudaEventCreate");
		check_cuda(cudaEventCreate(&kt1), "cudaEventCreate");
		check_cuda(cudaEventRecord(kt0, s), "cudaEventRecord");
	}
	const int rc = k.launcher(&c, s);
	if(profile_) {
		check_cuda(cudaEventRecord(kt1, s), "cudaEventRecord");
		ktimes_[k.id].pending.emplace_back(kt0, kt1);
	}
	if(rc != 0) throw execution_error("kernel \"" + k.id + "\" launcher failed with code " + std::to_string(rc));
	check_cuda(cudaGetLastError(), ("kernel \"" + k.id + "\" launch").c_str());
	++ctr_.kernels;
	last_exec_stream_ = s;
	finish(t, s);
	for(size_t i = 0; i < applied.size(); ++i) {
		if(!applied[i]) continue; // issued as an ordinary copy when its turn comes
		const task& cp = *(*fused)[i];
		finish(cp, s);
		mirrored_[cp.id] = 1;
		++ctr_.fused_copies;
		ctr_.bytes_fused += static_cast<uint64_t>(cp.dst_region.volume()) * dtype_size(buf(cp.dst).type);
	}
}

void executor::run_copy(const task& t) {
	const buffer& src = buf(t.src);
	const buffer& dst = buf(t.dst);
	if(src.type != dst.type) throw execution_error("copy between chunks of different element types");
	ldev& L = dev(t.resource);
	cudaStream_t s = L.copy;
	perturb(s);
	wait_deps(t, s);
	copy_box(src.ptr, src.region, ord(src.gpu), dst.ptr, dst.region, ord(dst.gpu), t.dst_region, dtype_size(src.type), s);
	++ctr_.copies;
	ctr_.bytes_copied += static_cast<uint64_t>(t.dst_region.volume()) * dtype_size(src.type);
	finish(t, s);
}

void executor::run_send(const task& t) {
	if(remote_worker(t.peer)) return remote_send(t);
	const buffer& src = buf(t.chunk);
	ldev& L = dev(t.resource);
	cudaStream_t s = L.copy;
	wait_deps(t, s);
	auto& G = gpus_[static_cast<size_t>(L.gpu)];
	message m;
	m.bytes = static_cast<uint64_t>(t.region.volume()) * dtype_size(src.type);
	m.gpu = L.gpu;
	check_cuda(cudaMallocFromPoolAsync(&m.ptr, m.bytes, G.pool, s), "cudaMallocFromPoolAsync");
	copy_box(src.ptr, src.region, ord(src.gpu), m.ptr, t.region, ord(L.gpu), t.region, dtype_size(src.type), s);
	m.ready = take_event(L.gpu);
	check_cuda(cudaEventRecord(m.ready, s), "cudaEventRecord");
	const auto key = std::make_tuple(t.worker, t.peer, t.tag);
	if(mailbox_.count(key)) throw execution_error("duplicate message tag");
	mailbox_[key] = m;
	ctr_.bytes_sent += m.bytes;
	wc(t.worker).bytes_sent += m.bytes;
	finish(t, s);
}

void executor::run_recv(const task& t) {
	if(remote_worker(t.peer)) return remote_recv(t);
	const auto key = std::make_tuple(t.peer, t.worker, t.tag);
	const auto it = mailbox_.find(key);
	if(it == mailbox_.end())
		throw execution_error("receive (w" + std::to_string(t.peer) + " -> w" + std::to_string(t.worker) + ", tag " + std::to_string(t.tag)
		                      + ") has no matching send (protocol violation)");
	const message m = it->second;
	mailbox_.erase(it);
	const buffer& dst = buf(t.chunk);
	ldev& L = dev(t.resource);
	cudaStream_t s = L.copy;
	wait_deps(t, s);
	check_cuda(cudaStreamWaitEvent(s, m.ready, 0), "cudaStreamWaitEvent");
	if(m.bytes != static_cast<uint64_t>(t.region.volume()) * dtype_size(dst.type))
		throw execution_error("received payload size does not match the destination region");
	copy_box(m.ptr, t.region, ord(m.gpu), dst.ptr, dst.region, ord(dst.gpu), t.region, dtype_size(dst.type), s);
	// release the message buffer on its own device once the unpack is done
	cudaEvent_t unpacked = take_event(L.gpu);
	check_cuda(cudaEventRecord(unpacked, s), "cudaEventRecord");
	auto& G = gpus_[static_cast<size_t>(m.gpu)];
	check_cuda(cudaSetDevice(ord(m.gpu)), "cudaSetDevice");
	check_cuda(cudaStreamWaitEvent(G.service, unpacked, 0), "cudaStreamWaitEvent");
	check_cuda(cudaFreeAsync(m.ptr, G.service), "cudaFreeAsync");
	check_cuda(cudaSetDevice(ord(L.gpu)), "cudaSetDevice");
	free_events_[static_cast<size_t>(m.gpu)].push_back(m.ready);
	free_events_[static_cast<size_t>(L.gpu)].push_back(unpacked);
	ctr_.bytes_received += m.bytes;
	wc(t.worker).bytes_received += m.bytes;
	finish(t, s);
}

void executor::run_reduce(const task& t) {
	const buffer& out = buf(t.output);
	ldev& L = dev(t.resource);
	cudaStream_t s = pick_compute(t, L);
	wait_deps(t, s);
	std::vector<const void*> ins;
	for(const auto c : t.inputs) {
		const buffer& b = buf(c);
		if(b.region != out.region) throw execution_error("reduce task combines chunks of different regions");
		ins.push_back(b.ptr);
	}
	if(!ins.empty()) device_reduce(out.ptr, ins.data(), static_cast<int>(ins.size()), static_cast<uint64_t>(out.region.volume()), out.type, t.op, s);
	++ctr_.kernels;
	finish(t, s);
}

// ---- allreduce (collective reduce trees) ------------------------------------------------------
//
// The reference reduces every worker's partial at the root w0d0 and sends the total back
// (planner.cpp:389-517). With cfg.collective_reduce the planner emits one allreduce task per
// worker instead. Between processes it is one ncclAllReduce in place on the member buffer
// (NVLink / NVLS inside NCCL; float sums in NCCL's order, within the reductions tolerance). In
// one process the members are issued in worker order and the last one combines them with the
// reduce kernel in the reference's root order, so the result is bit-identical to the tree.

void executor::finish_id(int64_t id, cudaStream_t s, int gpu) {
	cudaEvent_t ev = take_event(gpu);
	check_cuda(cudaEventRecord(ev, s), "cudaEventRecord");
	done_[id] = {ev, s, gpu};
	tail_[s] = id;
	++ctr_.tasks;
}


void executor::nccl_load(const char* lib) {
	if(nccl_dl_) return;
	void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD); // e.g. torch.distributed's copy
	if(!h && lib && *lib) h = dlopen(lib, RTLD_NOW);
	if(!h) h = dlopen("libnccl.so.2", RTLD_NOW);
	if(!h) throw execution_error(std::string("cannot load libnccl.so.2: ") + dlerror());
	const auto sym = [&](const char* name) {
		void* f = dlsym(h, name);
		if(!f) throw execution_error(std::string("libnccl lacks ") + name);
		return f;
	};
	g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(sym("ncclGetUniqueId"));
	g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(sym("ncclCommInitRank"));
	g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(sym("ncclAllReduce"));
	g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(sym("ncclCommDestroy"));
	g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(sym("ncclGetErrorString"));
	nccl_dl_ = h;
}

void executor::nccl_unique_id(const char* lib, void* id128) {
	nccl_load(lib);
	ncclUniqueId id;
	nccl_check(g_nccl.get_unique_id(&id), "ncclGetUniqueId");
	static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
	std::memcpy(id128, &id, sizeof(id));
}

void executor::nccl_init(const char* lib, const void* id128, int nranks, int rank) {
	nccl_load(lib);
	if(nccl_comm_) throw validation_error("the NCCL communicator is already initialised");
	ncclUniqueId id;
	std::memcpy(&id, id128, sizeof(id));
	check_cuda(cudaSetDevice(gpus_.at(0).ordinal), "cudaSetDevice");
	ncclComm_t comm = nullptr;
	nccl_check(g_nccl.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
	nccl_comm_ = comm;
}

void executor::run_allreduce(const task& t) {
	ldev& L = dev(t.resource);
	cudaStream_t s = pick_compute(t, L);
	wait_deps(t, s);
	const buffer& out = buf(t.output);
	const uint64_t count = static_cast<uint64_t>(out.region.volume());
	if(cfg_.local_workers >= 0 && cfg_.local_workers < cfg_.workers) {
		if(cfg_.local_workers != 1) throw execution_error("an allreduce across processes needs one worker per process");
		if(!nccl_comm_) throw execution_error("allreduce task but no NCCL communicator (mt_ctx_nccl_init / Context.connect_peers)");
		ncclDataType_t dt = ncclFloat32;
		switch(out.type) {
		case dtype::i32: dt = ncclInt32; break;
		case dtype::i64: dt = ncclInt64; break;
		case dtype::f32: dt = ncclFloat32; break;
		case dtype::f64: dt = ncclFloat64; break;
		case dtype::bf16: dt = ncclBfloat16; break;
		}
		ncclRedOp_t op = ncclSum;
		switch(t.op) {
		case reduce_op::plus: op = ncclSum; break;
		case reduce_op::times: op = ncclProd; break;
		case reduce_op::min: op = ncclMin; break;
		case reduce_op::max: op = ncclMax; break;
		}
		nccl_check(g_nccl.all_reduce(out.ptr, out.ptr, count, dt, op, static_cast<ncclComm_t>(nccl_comm_), s), "ncclAllReduce");
		ctr_.bytes_sent += count * dtype_size(out.type);
		wc(t.worker).bytes_sent += count * dtype_size(out.type);
		finish(t, s);
		return;
	}
	auto& g = groups_[t.tag];
	g.tasks.push_back(t.id);
	g.outputs.push_back(t.output);
	if(static_cast<int>(g.tasks.size()) < cfg_.workers) {
		cudaEvent_t ev = take_event(L.gpu);
		check_cuda(cudaEventRecord(ev, s), "cudaEventRecord");
		g.ready.emplace_back(ev, L.gpu);
		return; // completes when the last member has combined the group
	}
	for(const auto& [ev, gi] : g.ready) check_cuda(cudaStreamWaitEvent(s, ev, 0), "cudaStreamWaitEvent");
	const uint64_t bytes = count * dtype_size(out.type);
	std::vector<const void*> ins;
	for(const auto c : t.inputs) {
		const buffer& b = buf(c);
		if(b.region != out.region) throw execution_error("allreduce members cover different regions");
		ins.push_back(b.ptr);
	}
	if(!ins.empty() && bytes > 0) {
		void* total = nullptr;
		check_cuda(cudaMallocFromPoolAsync(&total, bytes, gpus_[static_cast<size_t>(L.gpu)].pool, s), "cudaMallocFromPoolAsync");
		device_reduce(total, ins.data(), static_cast<int>(ins.size()), count, out.type, t.op, s);
		++ctr_.kernels;
		for(const auto o : g.outputs) {
			const buffer& b = buf(o);
			if(b.gpu == L.gpu)
				check_cuda(cudaMemcpyAsync(b.ptr, total, bytes, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync");
			else
				check_cuda(cudaMemcpyPeerAsync(b.ptr, ord(b.gpu), total, ord(L.gpu), bytes, s), "cudaMemcpyPeerAsync");
		}
		check_cuda(cudaFreeAsync(total, s), "cudaFreeAsync");
	}
	for(const auto& [ev, gi] : g.ready) free_events_[static_cast<size_t>(gi)].push_back(ev);
	for(const auto id : g.tasks) finish_id(id, s, L.gpu);
	groups_.erase(t.tag);
}

// host_write / host_read: one region copy between the chunk and the host array, on the
// device's host-in / host-out stream so uploads, downloads and kernels all overlap
void executor::run_host_io(const task& t) {
	buffer& b = buf(t.chunk);
	ldev& L = dev(t.resource);
	const bool in = t.kind == task_kind::host_write;
	cudaStream_t s = in ? L.host_in : L.host_out;
	wait_deps(t, s);
	if(!encloses(b.region, t.region) || !encloses(t.src_region, t.region)) throw execution_error("host transfer region outside the chunk or the host array");
	void* host = reinterpret_cast<void*>(static_cast<uintptr_t>(t.tag));
	const size_t elem = dtype_size(b.type);
	if(!b.ptr) throw execution_error("host transfer on a non-resident chunk");
	if(in)
		copy_box(host, t.src_region, -1, b.ptr, b.region, ord(b.gpu), t.region, elem, s);
	else
		copy_box(b.ptr, b.region, ord(b.gpu), host, t.src_region, -1, t.region, elem, s);
	const uint64_t bytes = static_cast<uint64_t>(t.region.volume()) * elem;
	if(in)
		ctr_.bytes_host_in += bytes;
	else
		ctr_.bytes_host_out += bytes;
	finish(t, s);
}

void executor::mark(int slot) {
	if(slot < 0 || slot > 1) throw validation_error("mark slot must be 0 or 1");
	drain(true);
	issue_batch();
	for(size_t g = 0; g < gpus_.size(); ++g) {
		auto& G = gpus_[g];
		check_cuda(cudaSetDevice(G.ordinal), "cudaSetDevice");
		for(const auto& [s, tail] : tail_) {
			const auto it = done_.find(tail);
			if(it == done_.end() || it->second.gpu != static_cast<int>(g)) continue; // done_ev.gpu is the executor GPU index
			check_cuda(cudaStreamWaitEvent(G.timing, it->second.ev, 0), "cudaStreamWaitEvent");
		}
		// spill-tier transfers are not tasks: join their streams explicitly
		for(cudaStream_t s : {G.h2d, G.d2h}) {
			cudaEvent_t e = take_event(static_cast<int>(g));
			check_cuda(cudaEventRecord(e, s), "cudaEventRecord");
			check_cuda(cudaStreamWaitEvent(G.timing, e, 0), "cudaStreamWaitEvent");
			free_events_[g].push_back(e);
		}
		check_cuda(cudaEventRecord(G.marks[slot], G.timing), "cudaEventRecord");
	}
}

double executor::elapsed_ms() {
	double worst = 0.0;
	for(auto& G : gpus_) {
		check_cuda(cudaSetDevice(G.ordinal), "cudaSetDevice");
		check_cuda(cudaEventSynchronize(G.marks[1]), "cudaEventSynchronize");
		float ms = 0.f;
		check_cuda(cudaEventElapsedTime(&ms, G.marks[0], G.marks[1]), "cudaEventElapsedTime");
		worst = std::max(worst, static_cast<double>(ms));
	}
	return worst;
}

void executor::kernel_time(const std::string& kernel, int64_t* count, double* total_ms) {
	auto& kt = ktimes_[kernel];
	for(auto& [a, b] : kt.pending) {
		check_cuda(cudaEventSynchronize(b), "cudaEventSynchronize");
		float ms = 0.f;
		check_cuda(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
		kt.total_ms += ms;
		kt.count += 1;
		cudaEventDestroy(a);
		cudaEventDestroy(b);
	}
	kt.pending.clear();
	*count = kt.count;
	*total_ms = kt.total_ms;
}

void executor::sync() {
	drain(true);
	issue_batch();
	std::string err;
	for(auto& G : gpus_) {
		cudaSetDevice(G.ordinal);
		const cudaError_t e = cudaDeviceSynchronize();
		if(e != cudaSuccess && err.empty()) err = std::string("device execution failed: ") + cudaGetErrorString(e);
	}
	for(auto& [id, d] : done_) release_done_event(d.ev, d.gpu);
	done_.clear();
	tail_.clear();
	for(const auto& st : staged_) unpin(st);
	staged_.clear();
	if(!err.empty()) throw execution_error(err);
	if(!mailbox_.empty()) throw execution_error(std::to_string(mailbox_.size()) + " transport messages were never received (protocol violation)");
}

void executor::download(int64_t chunk, void* host, const box& host_box, const box& region) {
	drain(true);
	const buffer& b = buf(chunk);
	if(!encloses(b.region, region) || !encloses(host_box, region)) throw validation_error("download region outside the chunk or the host box");
	check_cuda(cudaSetDevice(ord(b.gpu)), "cudaSetDevice");
	cudaStream_t s = gpus_[static_cast<size_t>(b.gpu)].service;
	check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
	std::vector<char> from_disk;
	if(b.ptr)
		copy_box(b.ptr, b.region, ord(b.gpu), host, host_box, -1, region, dtype_size(b.type), s);
	else if(b.host && b.host_valid)
		copy_box(b.host, b.region, -1, host, host_box, -1, region, dtype_size(b.type), s); // evicted: host copy is current
	else if(b.disk_valid) {
		from_disk.resize(b.bytes);
		disk_read(b, from_disk.data());
		copy_box(from_disk.data(), b.region, -1, host, host_box, -1, region, dtype_size(b.type), s);
	} else if(b.host)
		copy_box(b.host, b.region, -1, host, host_box, -1, region, dtype_size(b.type), s);
	check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

void executor::upload(int64_t chunk, const void* host, const box& host_box) {
	drain(true);
	buffer& b = buf(chunk);
	if(!encloses(host_box, b.region)) throw validation_error("upload: chunk outside the host box");
	check_cuda(cudaSetDevice(ord(b.gpu)), "cudaSetDevice");
	cudaStream_t s = gpus_[static_cast<size_t>(b.gpu)].service;
	check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
	if(b.ptr) {
		copy_box(host, host_box, -1, b.ptr, b.region, ord(b.gpu), b.region, dtype_size(b.type), s);
		b.host_valid = false;
	} else {
		if(!b.host) b.host = host_alloc(b.bytes, b.gpu, chunk);
		copy_box(host, host_box, -1, b.host, b.region, -1, b.region, dtype_size(b.type), s);
		b.host_valid = true;
		disk_release(b);
	}
	check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

// ---- inter-process send/recv (one process per worker) -------------------------------------
//
// A message of the planner's send/recv pair (planner.cpp:96-119) moves as segments of at most
// kSlotBytes through a per-(src, dst) ring of kSlots slots that lives in the RECEIVER's
// IPC-mapped mailbox. Per segment q (slot q % kSlots), entirely GPU-driven and stream-ordered:
//   sender   (copy stream): wait consumed >= q+1-kSlots  ->  peer copy into the slot over
//                           NVLink  ->  release-store ready[slot] = q+1 (system scope)
//   receiver (recv stream): acquire-wait ready[slot] >= q+1  ->  copy slot into the chunk  ->
//                           release-store the sender's consumed counter = q+1
// Both sides derive the same segment sequence from the replicated plan (same regions, tags in
// issue order), so no host round trip is needed. Sends and receives use different streams so a
// sender spinning on a full ring never blocks the receive that would drain the peer's ring.

namespace {

// A peer that never sends (a crashed rank, a protocol bug) must not hang the GPU: after
// `timeout_ns` of waiting the kernel traps, the context reports a launch failure and the next
// mt_sync raises execution_error (the reference's stall detection, runtime.cpp:662-691).
__global__ void spin_until_geq(const uint64_t* flag, uint64_t value, uint64_t timeout_ns) {
	uint64_t v = 0, t0 = 0, now = 0;
	asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
	for(;;) {
		asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
		if(v >= value) break;
		__nanosleep(64);
		asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
		if(now - t0 > timeout_ns) {
			printf("manta-b200: peer message wait timed out (flag %p: %llu < %llu)\n", flag, static_cast<unsigned long long>(v),
			    static_cast<unsigned long long>(value));
			__trap();
		}
	}
}

// MTB_PEER_TIMEOUT_S (default 120 s) bounds every inter-process wait
uint64_t peer_timeout_ns() {
	static const uint64_t ns = [] {
		const char* e = std::getenv("MTB_PEER_TIMEOUT_S");
		const double s = e ? std::atof(e) : 120.0;
		return static_cast<uint64_t>((s > 0 ? s : 120.0) * 1e9);
	}();
	return ns;
}

__global__ void release_store(uint64_t* flag, uint64_t value) {
	asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

struct mbox_blob {
	uint64_t magic;
	int32_t rank, world, slots, pad;
	uint64_t slot_bytes;
	cudaIpcMemHandle_t handle;
};
constexpr uint64_t kMboxMagic = 0x6d616e7461623230ull; // "mantab20"

uint64_t ring_off(int src) { return static_cast<uint64_t>(src) * executor::kSlots * executor::kSlotBytes; }
uint64_t flag_off(int world, int src) { return static_cast<uint64_t>(world) * executor::kSlots * executor::kSlotBytes + static_cast<uint64_t>(src) * executor::kSlots * 8; }
uint64_t cons_off(int world, int dst) { return flag_off(world, world) + static_cast<uint64_t>(dst) * 128; }
uint64_t mbox_bytes(int world) { return cons_off(world, world); }

} // namespace

std::vector<uint8_t> executor::peer_export() {
	if(cfg_.local_workers != 1 || cfg_.devices_per_worker != 1) throw validation_error("inter-process messaging needs one worker with one device per process");
	if(mbox_) throw validation_error("mailbox already exported");
	world_ = cfg_.workers;
	my_rank_ = cfg_.first_worker;
	check_cuda(cudaSetDevice(ord(0)), "cudaSetDevice");
	const uint64_t bytes = mbox_bytes(world_);
	check_cuda(cudaMalloc(&mbox_, bytes), "cudaMalloc (mailbox)");
	check_cuda(cudaMemset(mbox_ + flag_off(world_, 0), 0, bytes - flag_off(world_, 0)), "cudaMemset (mailbox flags)");
	check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
	mbox_blob b{};
	b.magic = kMboxMagic;
	b.rank = my_rank_;
	b.world = world_;
	b.slots = kSlots;
	b.slot_bytes = kSlotBytes;
	check_cuda(cudaIpcGetMemHandle(&b.handle, mbox_), "cudaIpcGetMemHandle");
	std::vector<uint8_t> out(sizeof(b));
	std::memcpy(out.data(), &b, sizeof(b));
	return out;
}

void executor::peer_import(const std::vector<std::vector<uint8_t>>& blobs) {
	if(!mbox_) throw validation_error("export the local mailbox first");
	if(static_cast<int>(blobs.size()) != world_) throw validation_error("one mailbox blob per worker expected");
	check_cuda(cudaSetDevice(ord(0)), "cudaSetDevice");
	links_.assign(static_cast<size_t>(world_), peer_link{});
	check_cuda(cudaMalloc(&link_ctr_, sizeof(unsigned) * 2 * static_cast<size_t>(world_)), "cudaMalloc (link counters)");
	check_cuda(cudaMemset(link_ctr_, 0, sizeof(unsigned) * 2 * static_cast<size_t>(world_)), "cudaMemset");
	for(int p = 0; p < world_; ++p) {
		mbox_blob b{};
		if(blobs[static_cast<size_t>(p)].size() != sizeof(b)) throw validation_error("bad mailbox blob");
		std::memcpy(&b, blobs[static_cast<size_t>(p)].data(), sizeof(b));
		if(b.magic != kMboxMagic || b.rank != p || b.world != world_ || b.slots != kSlots || b.slot_bytes != kSlotBytes)
			throw validation_error("mailbox blob " + std::to_string(p) + " does not match this configuration");
		if(p == my_rank_) continue;
		void* base = nullptr;
		check_cuda(cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
		opened_.push_back(base);
		char* peer = static_cast<char*>(base);
		auto& l = links_[static_cast<size_t>(p)];
		l.tx_ring = peer + ring_off(my_rank_);
		l.tx_ready = reinterpret_cast<uint64_t*>(peer + flag_off(world_, my_rank_));
		l.tx_consumed = reinterpret_cast<uint64_t*>(mbox_ + cons_off(world_, p));
		l.rx_ring = mbox_ + ring_off(p);
		l.rx_ready = reinterpret_cast<uint64_t*>(mbox_ + flag_off(world_, p));
		l.rx_consumed = reinterpret_cast<uint64_t*>(peer + cons_off(world_, my_rank_));
		l.tx_done = link_ctr_ + 2 * p;
		l.rx_done = link_ctr_ + 2 * p + 1;
		check_cuda(cudaStreamCreateWithFlags(&l.tx, cudaStreamNonBlocking), "cudaStreamCreate");
		check_cuda(cudaStreamCreateWithFlags(&l.rx, cudaStreamNonBlocking), "cudaStreamCreate");
	}
	check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

// ---- fused single-segment path --------------------------------------------------------------
//
// A message that fits one ring slot (every halo row: 256 KiB at C2) moves with one copy kernel
// per side, no staging copies or allocations:
//   send (peer tx stream): from the kSlots-th message on, a one-thread kernel waits for the slot
//        to be free; the copy kernel's CTAs copy their rows of the region straight from the
//        chunk into the peer's slot over NVLink (st.global to the IPC-mapped peer memory) and
//        fence at system scope; the last CTA to finish release-stores the slot's ready flag in
//        the peer's memory.
//   recv (peer rx stream): a one-thread kernel acquire-waits on the ready flag; the copy
//        kernel's CTAs copy their rows from the slot (ld.global.cg: the peer's stores landed in
//        this GPU's L2) into the chunk; the last CTA release-stores the consumption counter back
//        into the sender's memory.
// Larger messages keep the segmented ring below (stage, per-segment wait / copy / flag).
struct box_rows {
	char* base;          // region start inside the chunk
	int64_t rows;        // e0 * e1 (rank 3: planes x rows; rank 2: rows; rank 1: 1)
	int64_t per_plane;   // e1
	int64_t pitch_plane; // bytes between planes
	int64_t pitch_row;   // bytes between rows
	int64_t row_bytes;   // contiguous bytes per row
};

box_rows rows_of(void* chunk_ptr, const box& chunk, const box& region, size_t elem) {
	const int r = region.rank();
	int64_t ext[3] = {1, 1, 1}, cext[3] = {1, 1, 1}, off[3] = {0, 0, 0};
	for(int k = 0; k < r; ++k) {
		ext[3 - r + k] = region.extent(k);
		cext[3 - r + k] = chunk.extent(k);
		off[3 - r + k] = region.lo[k] - chunk.lo[k];
	}
	box_rows b{};
	const int64_t e = static_cast<int64_t>(elem);
	b.pitch_row = cext[2] * e;
	b.pitch_plane = cext[1] * cext[2] * e;
	b.base = static_cast<char*>(chunk_ptr) + off[0] * b.pitch_plane + off[1] * b.pitch_row + off[2] * e;
	b.rows = ext[0] * ext[1];
	b.per_plane = ext[1];
	b.row_bytes = ext[2] * e;
	return b;
}

// packed message (row-major region) <-> rows of a chunk; `to_packed` chooses the direction
template <typename V, bool CG>
__device__ void move_rows(const box_rows& b, char* packed, bool to_packed) {
	const int64_t per = b.row_bytes / static_cast<int64_t>(sizeof(V));
	const int64_t total = per * b.rows;
	for(int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
		const int64_t r = i / per, c = i - r * per;
		V* chunk = reinterpret_cast<V*>(b.base + (r / b.per_plane) * b.pitch_plane + (r % b.per_plane) * b.pitch_row) + c;
		V* msg = reinterpret_cast<V*>(packed + r * b.row_bytes) + c;
		if(to_packed)
			*msg = *chunk;
		else if constexpr(CG)
			*chunk = __ldcg(msg);
		else
			*chunk = *msg;
	}
}

template <bool CG>
__device__ void move_any(const box_rows& b, char* packed, bool to_packed) {
	const uintptr_t a = reinterpret_cast<uintptr_t>(b.base) | reinterpret_cast<uintptr_t>(packed) | static_cast<uintptr_t>(b.row_bytes)
	                    | static_cast<uintptr_t>(b.pitch_row) | static_cast<uintptr_t>(b.pitch_plane);
	if(a % 16 == 0)
		move_rows<uint4, CG>(b, packed, to_packed);
	else if(a % 4 == 0)
		move_rows<unsigned, CG>(b, packed, to_packed);
	else
		move_rows<unsigned char, false>(b, packed, to_packed);
}

// the last CTA through `done` (after a system-scope fence) release-stores `value` to `flag`
__device__ void last_cta_release(unsigned* done, uint64_t* flag, uint64_t value) {
	__syncthreads();
	if(threadIdx.x == 0) {
		__threadfence_system();
		if(atomicAdd(done, 1u) == gridDim.x - 1) {
			*done = 0; // the next message on this stream starts after this kernel
			__threadfence_system();
			asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
		}
	}
}

// The waits themselves run in a one-thread spin_until_geq kernel ahead of these on the same
// stream: a copy kernel whose CTAs all spun would hold tens of CTAs per pending message
// resident, and ranks sharing a GPU (MPS) or a GPU busy with a large kernel could fill every
// SM with waiters while the kernels they wait for queue behind them (4 ranks under MPS
// deadlocked that way). One waiting thread per message cannot exhaust the SMs.
__global__ void fused_send_k(box_rows src, char* slot, uint64_t* ready, uint64_t value, unsigned* done) {
	move_any<false>(src, slot, true);
	last_cta_release(done, ready, value);
}

__global__ void fused_recv_k(box_rows dst, char* slot, uint64_t* consumed, uint64_t value, unsigned* done) {
	move_any<true>(dst, slot, false);
	last_cta_release(done, consumed, value);
}

unsigned fused_grid(uint64_t bytes) {
	return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(132, (bytes + 4095) / 4096)));
}

void executor::remote_send(const task& t) {
	if(links_.empty()) throw execution_error("send to worker " + std::to_string(t.peer) + " in another process before peer_import");
	const buffer& src = buf(t.chunk);
	ldev& L = dev(t.resource);
	auto& link = links_.at(static_cast<size_t>(t.peer));
	cudaStream_t s = link.tx;
	wait_deps(t, s);
	auto& G = gpus_[static_cast<size_t>(L.gpu)];
	const size_t elem = dtype_size(src.type);
	const uint64_t bytes = static_cast<uint64_t>(t.region.volume()) * elem;
	++ctr_.messages;
	if(bytes <= kSlotBytes) {
		const uint64_t q = link.tx_seq++;
		const uint64_t slot = q % kSlots;
		const uint64_t need = q >= static_cast<uint64_t>(kSlots) ? q + 1 - kSlots : 0;
		if(need) {
			spin_until_geq<<<1, 1, 0, s>>>(link.tx_consumed, need, peer_timeout_ns());
			++ctr_.message_ops;
		}
		fused_send_k<<<fused_grid(bytes), 256, 0, s>>>(rows_of(src.ptr, src.region, t.region, elem), link.tx_ring + slot * kSlotBytes, link.tx_ready + slot,
		    q + 1, link.tx_done);
		++ctr_.message_ops;
	} else {
		// contiguous staging of the region, then one ring segment at a time
		void* stage = nullptr;
		check_cuda(cudaMallocFromPoolAsync(&stage, bytes, G.pool, s), "cudaMallocFromPoolAsync");
		copy_box(src.ptr, src.region, ord(src.gpu), stage, t.region, ord(L.gpu), t.region, elem, s);
		ctr_.message_ops += 3;
		for(uint64_t off = 0; off < bytes; off += kSlotBytes) {
			const uint64_t seg = std::min<uint64_t>(kSlotBytes, bytes - off);
			const uint64_t q = link.tx_seq++;
			const uint64_t slot = q % kSlots;
			if(q >= static_cast<uint64_t>(kSlots)) spin_until_geq<<<1, 1, 0, s>>>(link.tx_consumed, q + 1 - kSlots, peer_timeout_ns());
			check_cuda(cudaMemcpyAsync(link.tx_ring + slot * kSlotBytes, static_cast<char*>(stage) + off, seg, cudaMemcpyDefault, s), "cudaMemcpyAsync (send)");
			release_store<<<1, 1, 0, s>>>(link.tx_ready + slot, q + 1);
			ctr_.message_ops += q >= static_cast<uint64_t>(kSlots) ? 3 : 2;
		}
		check_cuda(cudaFreeAsync(stage, s), "cudaFreeAsync");
	}
	check_cuda(cudaGetLastError(), "send kernels");
	ctr_.bytes_sent += bytes;
	wc(t.worker).bytes_sent += bytes;
	finish(t, s);
}

void executor::remote_recv(const task& t) {
	if(links_.empty()) throw execution_error("receive from worker " + std::to_string(t.peer) + " in another process before peer_import");
	const buffer& dst = buf(t.chunk);
	ldev& L = dev(t.resource);
	auto& link = links_.at(static_cast<size_t>(t.peer));
	cudaStream_t s = link.rx;
	wait_deps(t, s);
	auto& G = gpus_[static_cast<size_t>(L.gpu)];
	const size_t elem = dtype_size(dst.type);
	const uint64_t bytes = static_cast<uint64_t>(t.region.volume()) * elem;
	++ctr_.messages;
	if(bytes <= kSlotBytes) {
		const uint64_t q = link.rx_seq++;
		const uint64_t slot = q % kSlots;
		spin_until_geq<<<1, 1, 0, s>>>(link.rx_ready + slot, q + 1, peer_timeout_ns());
		fused_recv_k<<<fused_grid(bytes), 256, 0, s>>>(rows_of(dst.ptr, dst.region, t.region, elem), link.rx_ring + slot * kSlotBytes, link.rx_consumed,
		    q + 1, link.rx_done);
		ctr_.message_ops += 2;
	} else {
		void* stage = nullptr;
		check_cuda(cudaMallocFromPoolAsync(&stage, bytes, G.pool, s), "cudaMallocFromPoolAsync");
		ctr_.message_ops += 1;
		for(uint64_t off = 0; off < bytes; off += kSlotBytes) {
			const uint64_t seg = std::min<uint64_t>(kSlotBytes, bytes - off);
			const uint64_t q = link.rx_seq++;
			const uint64_t slot = q % kSlots;
			spin_until_geq<<<1, 1, 0, s>>>(link.rx_ready + slot, q + 1, peer_timeout_ns());
			check_cuda(cudaMemcpyAsync(static_cast<char*>(stage) + off, link.rx_ring + slot * kSlotBytes, seg, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync (recv)");
			release_store<<<1, 1, 0, s>>>(link.rx_consumed, q + 1);
			ctr_.message_ops += 3;
		}
		copy_box(stage, t.region, ord(L.gpu), dst.ptr, dst.region, ord(dst.gpu), t.region, elem, s);
		check_cuda(cudaFreeAsync(stage, s), "cudaFreeAsync");
		ctr_.message_ops += 2;
	}
	check_cuda(cudaGetLastError(), "recv kernels");
	ctr_.bytes_received += bytes;
	wc(t.worker).bytes_received += bytes;
	finish(t, s);
}

std::string executor::report_json() {
	// traced tasks per worker: {"id", "kind", "start_ns", "end_ns"} (runtime.cpp:626-629)
	std::vector<std::string> tasks(static_cast<size_t>(cfg_.workers));
	for(const auto& r : trace_recs_) {
		if(!r.t1 || r.worker < 0 || r.worker >= cfg_.workers) continue;
		check_cuda(cudaEventSynchronize(r.t1), "cudaEventSynchronize");
		float a = 0.f, b = 0.f;
		check_cuda(cudaEventElapsedTime(&a, trace_base_[static_cast<size_t>(r.gpu)], r.t0), "cudaEventElapsedTime");
		check_cuda(cudaEventElapsedTime(&b, trace_base_[static_cast<size_t>(r.gpu)], r.t1), "cudaEventElapsedTime");
		std::string& o = tasks[static_cast<size_t>(r.worker)];
		o += std::string(o.empty() ? "" : ", ") + "{\"id\": " + std::to_string(r.id) + ", \"kind\": \"" + task_kind_name(r.kind) + "\", \"start_ns\": "
		     + std::to_string(static_cast<int64_t>(static_cast<double>(a) * 1e6)) + ", \"end_ns\": " + std::to_string(static_cast<int64_t>(static_cast<double>(b) * 1e6)) + "}";
	}
	std::ostringstream os;
	os << "{\"workers\": [";
	for(int w = 0; w < cfg_.workers; ++w) {
		const auto& c = wctr_[static_cast<size_t>(w)];
		os << (w ? ", " : "") << "{\"worker\": " << w << ", \"evictions\": " << c.evictions << ", \"bytes_device_to_host\": " << c.bytes_device_to_host
		   << ", \"bytes_host_to_disk\": " << c.bytes_host_to_disk << ", \"bytes_host_to_device\": " << c.bytes_host_to_device
		   << ", \"bytes_disk_to_device\": " << c.bytes_disk_to_host << ", \"bytes_sent\": " << c.bytes_sent << ", \"bytes_received\": " << c.bytes_received
		   << ", \"staging_checks\": " << c.staging_checks << ", \"staging_violations\": " << c.staging_violations << ", \"peak_device_bytes\": [";
		for(int d = 0; d < cfg_.devices_per_worker; ++d) os << (d ? ", " : "") << dev_peak_[static_cast<size_t>(w * cfg_.devices_per_worker + d)];
		os << "], \"tasks\": [" << tasks[static_cast<size_t>(w)] << "]}";
	}
	os << "], \"tasks\": " << ctr_.tasks << ", \"kernel_launches\": " << ctr_.kernels << ", \"copies\": " << ctr_.copies << ", \"bytes_copied\": " << ctr_.bytes_copied
	   << "}";
	return os.str();
}

} // namespace mtb
