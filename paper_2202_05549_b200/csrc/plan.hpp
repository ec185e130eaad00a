// Task IR shared by the planner and the GPU executor (the reference's task.hpp:19-112).
#pragma once

#include <string>
#include <vector>

#include "annotation.hpp"
#include "distribution.hpp"

namespace mtb {
struct kernel_entry;
}

namespace mtb {

enum class task_kind : int32_t { create = 0, del = 1, execute = 2, copy = 3, send = 4, recv = 5, reduce = 6, allreduce = 7, host_write = 8, host_read = 9 };
enum class fill_kind : int32_t { none = 0, zero = 1, one = 2, identity = 3 };
enum class arg_kind : int32_t { scalar_int = 0, scalar_float = 1, chunk = 2, none = 3 };

struct arg_bind {
	arg_kind kind = arg_kind::none;
	int64_t i = 0;
	double f = 0.0;
	int64_t chunk = -1;
	// access of a chunk argument as the planner inferred it (executor data-liveness analysis;
	// unknown for plans that arrive through mt_exec_submit)
	box region;
	int8_t access = 0; // bit 0: reads, bit 1: writes; 0 = unknown
};

// One task; the fields a kind does not use stay default. See include/manta_b200.h mt_task.
struct task {
	int64_t id = -1;
	int worker = 0;
	task_kind kind = task_kind::create;
	device_id resource;
	std::vector<int64_t> deps; // ascending, same worker, already emitted
	// create / delete / send / recv
	int64_t chunk = -1;
	box region;
	device_id home;
	dtype type = dtype::f32;
	fill_kind fill = fill_kind::none;
	reduce_op fill_op = reduce_op::plus;
	// execute
	const struct kernel_entry* kern = nullptr; // global or context-local registry entry
	device_id device;
	box sb_blocks, sb_threads;
	// every thread of sb_threads lies inside the launch grid (no partial trailing block): only
	// then may a dense_writes kernel's write region count as overwritten (executor spill tier)
	bool sb_inside_grid = false;
	point block_size;
	std::vector<arg_bind> args;
	// copy
	int64_t src = -1, dst = -1;
	box src_region, dst_region;
	// send / recv (host_write / host_read: tag = host address, src_region = host array box,
	// region = the box copied)
	int peer = -1;
	uint64_t tag = 0;
	// reduce / allreduce (group = tag, members with data = inputs, own member = output)
	reduce_op op = reduce_op::plus;
	std::vector<int64_t> inputs;
	int64_t output = -1;
};

inline const char* task_kind_name(task_kind k) {
	switch(k) {
	case task_kind::create: return "create";
	case task_kind::del: return "delete";
	case task_kind::execute: return "execute";
	case task_kind::copy: return "copy";
	case task_kind::send: return "send";
	case task_kind::recv: return "recv";
	case task_kind::reduce: return "reduce";
	case task_kind::allreduce: return "allreduce";
	case task_kind::host_write: return "host_write";
	case task_kind::host_read: return "host_read";
	}
	return "?";
}

} // namespace mtb
