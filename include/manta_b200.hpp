// manta_b200.hpp — header-only C++ host API over the C-ABI (include/manta_b200.h).
//
// Mirrors the reference's C++ interface for the hot path so code written against
// proj/include/manta reads the same against the B200 runtime:
//   manta_b200::driver          ~ manta::driver          (planner.hpp:51-78)
//   manta_b200::system_runtime  ~ manta::system_runtime  (runtime.hpp:70-98)
//   manta_b200::*_dist          ~ distribution.hpp:62-92
//   manta_b200::{parse_error, validation_error, plan_error, execution_error}
//                               ~ errors.hpp:9-35
// Every call goes through the extern "C" entry points; nothing here touches CUDA directly.
#pragma once

#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <vector>

#include "manta_b200.h"

namespace manta_b200 {

struct error : std::runtime_error {
	using std::runtime_error::runtime_error;
};
struct parse_error : error {
	using error::error;
};
struct validation_error : error {
	using error::error;
};
struct plan_error : error {
	using error::error;
};
struct execution_error : error {
	using error::error;
};

inline void check(int rc) {
	if(rc == MT_OK) return;
	const std::string msg = mt_last_error();
	switch(rc) {
	case MT_EPARSE: throw parse_error(msg);
	case MT_EVALIDATION: throw validation_error(msg);
	case MT_EPLAN: throw plan_error(msg);
	case MT_EEXEC: throw execution_error(msg);
	default: throw error(msg);
	}
}

using array_id = int64_t;
using chunk_id = int64_t;
using task_id = int64_t;

struct device_id {
	int worker = 0;
	int device = 0;
};

// [lo, hi) box; `rect({0, 0}, {n, m})` like the reference's rect
struct rect {
	mt_rect r{};
	rect() = default;
	rect(std::initializer_list<int64_t> lo, std::initializer_list<int64_t> hi) {
		r.rank = static_cast<int32_t>(lo.size());
		int k = 0;
		for(auto v : lo) r.lo[k++] = v;
		k = 0;
		for(auto v : hi) r.hi[k++] = v;
	}
	int rank() const { return r.rank; }
};

enum class dtype : int32_t { i32 = MT_I32, i64 = MT_I64, f32 = MT_F32, f64 = MT_F64, bf16 = MT_BF16 };

struct fill_spec {
	int32_t kind = MT_FILL_NONE;
	static fill_spec none() { return {MT_FILL_NONE}; }
	static fill_spec zero() { return {MT_FILL_ZERO}; }
	static fill_spec one() { return {MT_FILL_ONE}; }
};

using data_distribution = std::vector<mt_chunk_desc>;
using work_distribution = std::vector<mt_superblock>;

inline std::vector<mt_device> to_devs(const std::vector<device_id>& d) {
	std::vector<mt_device> v;
	for(auto x : d) v.push_back({x.worker, x.device});
	return v;
}

inline data_distribution tile_data_dist(const rect& domain, std::vector<int64_t> extents, std::vector<int64_t> halo, const std::vector<device_id>& devices,
    chunk_id first_id = 0) {
	auto devs = to_devs(devices);
	int64_t n = 0;
	check(mt_dist_tile(&domain.r, extents.data(), halo.data(), devs.data(), static_cast<int32_t>(devs.size()), first_id, nullptr, 0, &n));
	data_distribution out(static_cast<size_t>(n));
	check(mt_dist_tile(&domain.r, extents.data(), halo.data(), devs.data(), static_cast<int32_t>(devs.size()), first_id, out.data(), n, &n));
	return out;
}

inline data_distribution stencil_dist(const rect& domain, std::vector<int64_t> extents, std::vector<int64_t> halo, const std::vector<device_id>& devices) {
	return tile_data_dist(domain, std::move(extents), std::move(halo), devices);
}

inline data_distribution row_dist(const rect& domain, int64_t rows, const std::vector<device_id>& devices) {
	std::vector<int64_t> ext, halo(static_cast<size_t>(domain.rank()), 0);
	for(int k = 0; k < domain.rank(); ++k) ext.push_back(domain.r.hi[k] - domain.r.lo[k]);
	ext[0] = rows;
	return tile_data_dist(domain, ext, halo, devices);
}

inline data_distribution replicated_dist(const rect& domain, const std::vector<device_id>& devices) {
	auto devs = to_devs(devices);
	int64_t n = 0;
	check(mt_dist_replicated(&domain.r, devs.data(), static_cast<int32_t>(devs.size()), 0, nullptr, 0, &n));
	data_distribution out(static_cast<size_t>(n));
	check(mt_dist_replicated(&domain.r, devs.data(), static_cast<int32_t>(devs.size()), 0, out.data(), n, &n));
	return out;
}

inline data_distribution single_dist(const rect& domain, device_id home) {
	int64_t n = 0;
	data_distribution out(1);
	check(mt_dist_single(&domain.r, mt_device{home.worker, home.device}, 0, out.data(), 1, &n));
	return out;
}

inline work_distribution block_work_dist(const rect& grid, std::vector<int64_t> block, std::vector<int64_t> tps, const std::vector<device_id>& devices) {
	auto devs = to_devs(devices);
	int64_t n = 0;
	check(mt_work_block(&grid.r, block.data(), tps.data(), devs.data(), static_cast<int32_t>(devs.size()), nullptr, 0, &n));
	work_distribution out(static_cast<size_t>(n));
	check(mt_work_block(&grid.r, block.data(), tps.data(), devs.data(), static_cast<int32_t>(devs.size()), out.data(), n, &n));
	return out;
}

struct launch_arg {
	mt_launch_arg a{};
	static launch_arg scalar(int64_t v) {
		launch_arg x;
		x.a.kind = MT_LARG_INT;
		x.a.i = v;
		return x;
	}
	static launch_arg scalar(double v) {
		launch_arg x;
		x.a.kind = MT_LARG_FLOAT;
		x.a.f = v;
		return x;
	}
	static launch_arg array(array_id id) {
		launch_arg x;
		x.a.kind = MT_LARG_ARRAY;
		x.a.array = id;
		return x;
	}
};

struct launch_result {
	task_id first_task = 0;
	task_id past_last_task = 0;
};

// memory_config (memory.hpp:43-55): capacities of the device pool, the pinned-host spill tier and
// the disk tier below it (0 = the runtime's default: 90% of free HBM / no host tier / no disk tier)
struct memory_config {
	uint64_t device_capacity = 0;
	uint64_t host_capacity = 0;
	uint64_t disk_capacity = 0;
	uint64_t staging_threshold = 0; // informational on the GPU executor
	std::string spill_dir;          // "" = the system temp directory
};

struct driver_config {
	int workers = 1;
	int devices_per_worker = 1;
	bool suppress_conflict_deps = false;
	bool compat_deps = false; // B200 extension: reference whole-chunk edges
	bool execute = true;      // B200 extension: planner and executor in one context
	int num_gpus = 0;
	memory_config memory{};
};

// driver + executor in one context (the reference's harness pattern, test_runtime.cpp:12-43)
class driver {
  public:
	explicit driver(driver_config cfg) {
		mt_config c{};
		c.workers = cfg.workers;
		c.devices_per_worker = cfg.devices_per_worker;
		c.suppress_conflict_deps = cfg.suppress_conflict_deps;
		c.compat_deps = cfg.compat_deps;
		c.execute = cfg.execute;
		c.num_gpus = cfg.num_gpus;
		c.device_capacity = cfg.memory.device_capacity;
		c.host_capacity = cfg.memory.host_capacity;
		c.disk_capacity = cfg.memory.disk_capacity;
		c.staging_threshold = cfg.memory.staging_threshold;
		spill_dir_ = cfg.memory.spill_dir;
		c.spill_dir = spill_dir_.empty() ? nullptr : spill_dir_.c_str();
		check(mt_ctx_create(&c, &ctx_));
	}
	~driver() { mt_ctx_destroy(ctx_); }
	driver(const driver&) = delete;
	driver& operator=(const driver&) = delete;

	std::vector<device_id> devices() const {
		mt_device d[1024];
		int32_t n = 0;
		check(mt_ctx_devices(ctx_, d, 1024, &n));
		std::vector<device_id> v;
		for(int32_t i = 0; i < n; ++i) v.push_back({d[i].worker, d[i].device});
		return v;
	}

	array_id create_array(const rect& domain, dtype type, const data_distribution& dist, fill_spec fill) {
		array_id id = -1;
		check(mt_array_create(ctx_, &domain.r, static_cast<int32_t>(type), dist.data(), static_cast<int64_t>(dist.size()), fill.kind, &id));
		return id;
	}
	void delete_array(array_id id) { check(mt_array_delete(ctx_, id)); }

	launch_result launch(const std::string& kernel, const rect& grid, std::vector<int64_t> block, const work_distribution& work,
	    const std::vector<launch_arg>& args, const std::string& annotation) {
		std::vector<mt_launch_arg> a;
		for(const auto& x : args) a.push_back(x.a);
		launch_result r;
		check(mt_launch(ctx_, kernel.c_str(), &grid.r, block.data(), work.data(), static_cast<int64_t>(work.size()), a.data(),
		    static_cast<int32_t>(a.size()), annotation.c_str(), &r.first_task, &r.past_last_task));
		return r;
	}

	// take_pending() + system_runtime::submit()
	void flush() { check(mt_flush(ctx_)); }
	void synchronize() { check(mt_sync(ctx_)); }

	template <typename T>
	std::vector<T> read(array_id id, size_t count) {
		std::vector<T> out(count);
		check(mt_array_read(ctx_, id, out.data(), count * sizeof(T)));
		return out;
	}
	// B200 extensions: upload a whole array, and queue host transfers ordered against the
	// launches by the dependency tracking (buffers must stay valid until synchronize())
	template <typename T>
	void write(array_id id, const std::vector<T>& data) {
		check(mt_array_write(ctx_, id, data.data(), data.size() * sizeof(T)));
	}
	void write_async(array_id id, const void* host, uint64_t bytes) { check(mt_array_write_async(ctx_, id, host, bytes)); }
	void read_async(array_id id, void* host, uint64_t bytes) { check(mt_array_read_async(ctx_, id, host, bytes)); }
	// per-task device timestamps in report_json() (run_report::to_json, runtime.cpp:613-636)
	void trace(bool on) { check(mt_exec_trace(mt_ctx_exec(ctx_), on ? 1 : 0)); }
	std::string report_json() {
		int64_t n = 0;
		check(mt_exec_report_json(mt_ctx_exec(ctx_), nullptr, 0, &n));
		std::string out(static_cast<size_t>(n) + 1, '\0');
		check(mt_exec_report_json(mt_ctx_exec(ctx_), out.data(), n + 1, &n));
		out.resize(static_cast<size_t>(n));
		return out;
	}

	mt_ctx* handle() { return ctx_; }

  private:
	mt_ctx* ctx_ = nullptr;
	std::string spill_dir_;
};

// The executor alone: the drop-in for manta::system_runtime (consumes flat task records)
class system_runtime {
  public:
	system_runtime(int workers, int devices_per_worker, int num_gpus = 0) {
		mt_config c{};
		c.workers = workers;
		c.devices_per_worker = devices_per_worker;
		c.execute = 1;
		c.num_gpus = num_gpus;
		check(mt_exec_create(&c, &ex_));
	}
	~system_runtime() { mt_exec_destroy(ex_); }
	system_runtime(const system_runtime&) = delete;
	system_runtime& operator=(const system_runtime&) = delete;

	void submit(const std::vector<mt_task>& tasks, const std::vector<int64_t>& pool, const std::vector<mt_arg_binding>& args) {
		check(mt_exec_submit(ex_, tasks.data(), static_cast<int64_t>(tasks.size()), pool.data(), args.data()));
	}
	void synchronize() { check(mt_exec_sync(ex_)); }
	std::vector<unsigned char> read_chunk(chunk_id id, size_t bytes) {
		std::vector<unsigned char> out(bytes);
		check(mt_exec_read_chunk(ex_, id, out.data(), bytes));
		return out;
	}

  private:
	mt_exec* ex_ = nullptr;
};

} // namespace manta_b200
