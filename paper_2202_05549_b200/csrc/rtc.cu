// Runtime kernel compilation with NVRTC (see rtc.hpp).
#include "rtc.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

#include "geometry.hpp"

namespace mtb {
namespace {

// device-side prelude: fixed-width integers (NVRTC has no libc headers) and the view types.
// A view holds the chunk pointer already shifted by the chunk offset, so global indices
// address it directly ("subtract this offset once on construction").
const char* kPrelude = R"(
typedef signed char int8_t; typedef short int16_t; typedef int int32_t; typedef long long int64_t;
typedef unsigned char uint8_t; typedef unsigned short uint16_t; typedef unsigned int uint32_t; typedef unsigned long long uint64_t;
namespace manta {
template <typename T, int R> struct Array;
template <typename T> struct Array<T, 0> {
	T* p;
	__device__ Array(T* q, const uint64_t (&)[1]) : p(q) {}
	__device__ T& operator*() const { return *p; }
	__device__ operator T&() const { return *p; }
};
template <typename T> struct Array<T, 1> {
	T* p; uint64_t s0;
	__device__ Array(T* q, const uint64_t (&s)[1]) : p(q), s0(s[0]) {}
	__device__ T& operator[](int64_t i) const { return p[i * (int64_t)s0]; }
	__device__ T& operator()(int64_t i) const { return p[i * (int64_t)s0]; }
};
template <typename T> struct Row { T* p; uint64_t s; __device__ T& operator[](int64_t j) const { return p[j * (int64_t)s]; } };
template <typename T> struct Array<T, 2> {
	T* p; uint64_t s0, s1;
	__device__ Array(T* q, const uint64_t (&s)[2]) : p(q), s0(s[0]), s1(s[1]) {}
	__device__ T& operator()(int64_t i, int64_t j) const { return p[i * (int64_t)s0 + j * (int64_t)s1]; }
	__device__ Row<T> operator[](int64_t i) const { return Row<T>{p + i * (int64_t)s0, s1}; }
};
template <typename T> struct Plane { T* p; uint64_t s1, s2; __device__ Row<T> operator[](int64_t j) const { return Row<T>{p + j * (int64_t)s1, s2}; } };
template <typename T> struct Array<T, 3> {
	T* p; uint64_t s0, s1, s2;
	__device__ Array(T* q, const uint64_t (&s)[3]) : p(q), s0(s[0]), s1(s[1]), s2(s[2]) {}
	__device__ T& operator()(int64_t i, int64_t j, int64_t k) const { return p[i * (int64_t)s0 + j * (int64_t)s1 + k * (int64_t)s2]; }
	__device__ Plane<T> operator[](int64_t i) const { return Plane<T>{p + i * (int64_t)s0, s1, s2}; }
};
template <typename T> using Scalar = Array<T, 0>;
template <typename T> using Vector = Array<T, 1>;
template <typename T> using Matrix = Array<T, 2>;
template <typename T> using Tensor = Array<T, 3>;
} // namespace manta
)";

const char* ctype(dtype t) {
	switch(t) {
	case dtype::i32: return "int32_t";
	case dtype::i64: return "int64_t";
	case dtype::f32: return "float";
	case dtype::f64: return "double";
	case dtype::bf16: return "uint16_t";
	}
	return "?";
}

// ---- NVRTC (run-time loaded: the library is optional until a kernel is compiled) -------------
struct nvrtc_api {
	decltype(&nvrtcCreateProgram) create = nullptr;
	decltype(&nvrtcCompileProgram) compile = nullptr;
	decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
	decltype(&nvrtcGetProgramLog) log = nullptr;
	decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
	decltype(&nvrtcGetCUBIN) cubin = nullptr;
	decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

const nvrtc_api& nvrtc() {
	static nvrtc_api api;
	static std::once_flag once;
	static std::string err;
	std::call_once(once, [] {
		void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
		if(!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
		if(!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
		if(!h) {
			err = dlerror() ? dlerror() : "libnvrtc.so.12 not found";
			return;
		}
		api.create = reinterpret_cast<decltype(api.create)>(dlsym(h, "nvrtcCreateProgram"));
		api.compile = reinterpret_cast<decltype(api.compile)>(dlsym(h, "nvrtcCompileProgram"));
		api.log_size = reinterpret_cast<decltype(api.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
		api.log = reinterpret_cast<decltype(api.log)>(dlsym(h, "nvrtcGetProgramLog"));
		api.cubin_size = reinterpret_cast<decltype(api.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
		api.cubin = reinterpret_cast<decltype(api.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
		api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
	});
	if(!api.create || !api.compile || !api.cubin) throw validation_error("runtime kernel compilation needs libnvrtc: " + err);
	return api;
}

// compiles `src` for sm_100a; returns the cubin or throws with the compiler log
std::vector<char> compile_cubin(const std::string& src, const std::string& name) {
	const auto& api = nvrtc();
	nvrtcProgram prog = nullptr;
	if(api.create(&prog, src.c_str(), name.c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS) throw validation_error("nvrtcCreateProgram failed");
	// IEEE operations as written (no FMA contraction), like the AOT kernels and the oracle
	const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-default-device"};
	const nvrtcResult r = api.compile(prog, 4, opts);
	size_t n = 0;
	api.log_size(prog, &n);
	std::string log(n, '\0');
	if(n > 1) api.log(prog, &log[0]);
	if(r != NVRTC_SUCCESS) {
		api.destroy(&prog);
		throw validation_error("kernel \"" + name + "\" does not compile:\n" + log);
	}
	size_t bytes = 0;
	api.cubin_size(prog, &bytes);
	std::vector<char> cubin(bytes);
	api.cubin(prog, cubin.data());
	api.destroy(&prog);
	return cubin;
}

// ---- driver API through the runtime's entry-point query (no link-time libcuda dependency) ----
struct drv_api {
	CUresult (*load)(CUmodule*, const void*) = nullptr;
	CUresult (*get_fn)(CUfunction*, CUmodule, const char*) = nullptr;
	CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream, void**, void**) = nullptr;
};

const drv_api& drv() {
	static drv_api api;
	static std::once_flag once;
	std::call_once(once, [] {
		const auto get = [](const char* sym) -> void* {
			void* p = nullptr;
			cudaDriverEntryPointQueryResult q{};
			if(cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) return nullptr;
			return p;
		};
		api.load = reinterpret_cast<decltype(api.load)>(get("cuModuleLoadData"));
		api.get_fn = reinterpret_cast<decltype(api.get_fn)>(get("cuModuleGetFunction"));
		api.launch = reinterpret_cast<decltype(api.launch)>(get("cuLaunchKernel"));
	});
	if(!api.load || !api.get_fn || !api.launch) throw execution_error("CUDA driver entry points for runtime kernels are unavailable");
	return api;
}

} // namespace

struct rtc_kernel {
	std::string id;
	std::vector<param_sig> params;
	std::string source;
	std::mutex mu;
	std::map<std::string, CUfunction> cache; // (device, instance constants) -> function
};

std::string wrapper_source(const std::string& id, const std::vector<param_sig>& params, const std::vector<int64_t>& block_offset,
    const std::vector<std::vector<int64_t>>& offsets, const std::vector<std::vector<int64_t>>& strides) {
	std::ostringstream os;
	os << "extern \"C\" __global__ void " << id << "_wrapper(\n";
	for(size_t i = 0; i < params.size(); ++i) {
		const auto& p = params[i];
		os << "  ";
		if(!p.is_array)
			os << ctype(p.type) << " " << p.name;
		else
			os << (p.writable ? "" : "const ") << ctype(p.type) << " *const " << p.name << "_ptr";
		os << (i + 1 < params.size() ? ",\n" : "\n");
	}
	os << ") {\n  // Worker-specific constants\n";
	const auto bo = [&](size_t k) { return k < block_offset.size() ? block_offset[k] : 0; };
	os << "  const uint32_t block_offset_x = " << bo(0) << ", block_offset_y = " << bo(1) << ", block_offset_z = " << bo(2) << ";\n";
	size_t v = 0;
	for(const auto& p : params) {
		if(!p.is_array) continue;
		const auto& off = offsets.at(v);
		const auto& st = strides.at(v);
		++v;
		if(p.rank == 0) continue;
		os << "  const uint64_t ";
		for(int k = 0; k < p.rank; ++k)
			os << (k ? ", " : "") << p.name << "_offset_" << k << " = " << off.at(static_cast<size_t>(k)) << ", " << p.name << "_strides_" << k << " = "
			   << st.at(static_cast<size_t>(k));
		os << ";\n";
	}
	os << "\n  // Prepare arguments\n";
	os << "  dim3 virtual_block_index(block_offset_x + blockIdx.x,\n    block_offset_y + blockIdx.y, block_offset_z + blockIdx.z);\n";
	for(const auto& p : params) {
		if(!p.is_array) continue;
		os << "  " << (p.writable ? "" : "const ") << "::manta::Array<" << ctype(p.type) << ", " << p.rank << "> " << p.name << "(\n    const_cast<"
		   << ctype(p.type) << "*>(" << p.name << "_ptr)";
		for(int k = 0; k < p.rank; ++k) os << " - " << p.name << "_offset_" << k << " * " << p.name << "_strides_" << k;
		os << ", {";
		if(p.rank == 0) os << "0";
		for(int k = 0; k < p.rank; ++k) os << (k ? ", " : "") << p.name << "_strides_" << k;
		os << "});\n";
	}
	os << "\n  // Call user kernel\n  " << id << "(virtual_block_index";
	for(const auto& p : params) os << ", " << p.name;
	os << ");\n}\n";
	return os.str();
}

namespace {

int rtc_launch(const mt_launch_ctx* c, void* stream) {
	auto* k = static_cast<rtc_kernel*>(const_cast<void*>(c->user));
	if(!k) return 9;
	std::vector<int64_t> bo(c->block_offset, c->block_offset + c->rank);
	std::vector<std::vector<int64_t>> offs, sts;
	std::vector<uint64_t> store(k->params.size());
	std::vector<void*> args(k->params.size());
	for(size_t i = 0; i < k->params.size(); ++i) {
		const auto& p = k->params[i];
		if(p.is_array) {
			const mt_view& v = c->views[i];
			offs.emplace_back(v.offset, v.offset + p.rank);
			sts.emplace_back(v.stride, v.stride + p.rank);
			store[i] = reinterpret_cast<uint64_t>(v.base);
		} else if(p.type == dtype::i32) {
			const int32_t x = static_cast<int32_t>(c->scalars_int[i]);
			std::memcpy(&store[i], &x, sizeof(x));
		} else if(p.type == dtype::i64) {
			std::memcpy(&store[i], &c->scalars_int[i], sizeof(int64_t));
		} else if(p.type == dtype::f32) {
			const float x = static_cast<float>(c->scalars_float[i]);
			std::memcpy(&store[i], &x, sizeof(x));
		} else {
			std::memcpy(&store[i], &c->scalars_float[i], sizeof(double));
		}
		args[i] = &store[i];
	}
	int dev = 0;
	cudaGetDevice(&dev);
	std::ostringstream key;
	key << dev;
	for(const auto b : bo) key << ',' << b;
	for(size_t i = 0; i < offs.size(); ++i) {
		key << '|';
		for(const auto o : offs[i]) key << o << ':';
		for(const auto s : sts[i]) key << s << ';';
	}
	CUfunction fn = nullptr;
	{
		std::lock_guard<std::mutex> lock(k->mu);
		const auto it = k->cache.find(key.str());
		if(it != k->cache.end()) {
			fn = it->second;
		} else {
			const std::string src = std::string(kPrelude) + "\n" + k->source + "\n" + wrapper_source(k->id, k->params, bo, offs, sts);
			const auto cubin = compile_cubin(src, k->id);
			CUmodule mod = nullptr;
			if(drv().load(&mod, cubin.data()) != CUDA_SUCCESS) return 10;
			if(drv().get_fn(&fn, mod, (k->id + "_wrapper").c_str()) != CUDA_SUCCESS) return 11;
			k->cache.emplace(key.str(), fn); // modules live as long as the process's contexts
		}
	}
	unsigned g[3] = {1, 1, 1}, b[3] = {1, 1, 1};
	for(int d = 0; d < c->rank && d < 3; ++d) {
		g[d] = static_cast<unsigned>(c->block_count[d]);
		b[d] = static_cast<unsigned>(c->block_size[d]);
	}
	if(g[0] * static_cast<uint64_t>(g[1]) * g[2] == 0) return 0;
	const CUresult r = drv().launch(fn, g[0], g[1], g[2], b[0], b[1], b[2], 0, static_cast<CUstream>(stream), args.data(), nullptr);
	return r == CUDA_SUCCESS ? 0 : 12;
}

} // namespace

std::shared_ptr<void> make_rtc_kernel(const std::string& id, const std::vector<param_sig>& params, const std::string& source, kernel_entry& e) {
	auto k = std::make_shared<rtc_kernel>();
	k->id = id;
	k->params = params;
	k->source = source;
	// probe instance: zero offsets, unit inner strides; compiles the user code now so errors
	// surface at registration, not at the first launch
	std::vector<std::vector<int64_t>> offs, sts;
	for(const auto& p : params) {
		if(!p.is_array) continue;
		offs.emplace_back(static_cast<size_t>(p.rank), 0);
		std::vector<int64_t> s(static_cast<size_t>(p.rank), 1);
		sts.push_back(s);
	}
	compile_cubin(std::string(kPrelude) + "\n" + source + "\n" + wrapper_source(id, params, {0, 0, 0}, offs, sts), id);
	e.id = id;
	e.params = params;
	e.launcher = &rtc_launch;
	e.user = k.get();
	return k;
}

} // namespace mtb
