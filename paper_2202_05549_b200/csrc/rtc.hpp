// Runtime kernel compilation (the paper's user-facing model; the reference
// generates the wrapper text, kernels.cpp:522-596, but has no GPU to compile it for).
//
// A user kernel is CUDA source defining
//     __device__ void <id>(dim3 virtBlockIdx, <scalar params...>, manta::Vector<T> out, const manta::Matrix<T> in, ...)
// Per superblock instance the generated wrapper bakes the block offset and every view's
// offsets/strides as compile-time constants (the paper's per-worker constants, so indexing
// costs nothing at run time), NVRTC compiles it for sm_100a on first use, and the module is
// cached per (device, instance). Repeated launches over the same decomposition (every
// iteration of a stencil) hit the cache.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/manta_b200.h"
#include "registry.hpp"

namespace mtb {

struct rtc_kernel;

// wrapper text for one instance (reference generate_wrapper_source, kernels.cpp:540-596):
// `offsets`/`strides` hold one vector per array parameter, in signature order
std::string wrapper_source(const std::string& id, const std::vector<param_sig>& params, const std::vector<int64_t>& block_offset,
    const std::vector<std::vector<int64_t>>& offsets, const std::vector<std::vector<int64_t>>& strides);

// validates the source by compiling a probe instance (throws validation_error with the NVRTC
// log) and returns the kernel; the entry's launcher/user are filled in
std::shared_ptr<void> make_rtc_kernel(const std::string& id, const std::vector<param_sig>& params, const std::string& source, kernel_entry& e);

} // namespace mtb
