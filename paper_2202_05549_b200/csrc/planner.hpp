// The driver: turns array/launch/delete requests into per-worker task DAGs.
//
// Task sequence, ids, kinds, chunk bindings, regions, tags and reduce input order are those
// of the reference driver (proj/src/planner.cpp:30-520) for the same request sequence; only
// the dependency lists differ, and only in region mode (see deps.hpp). Planning cost is
// O(S log C) per launch (indexed chunk queries, sweep-based overlap checks) rather than the
// reference's O(S^2 + S*C), so many launches can be planned ahead of GPU execution.
#pragma once

#include <deque>
#include <map>
#include <memory>
#include <unordered_map>
#include <vector>

#include "deps.hpp"
#include "plan.hpp"
#include "registry.hpp"

namespace mtb {

struct planner_config {
	int workers = 1;
	int devices_per_worker = 1;
	bool suppress_conflict_deps = false;
	bool compat_deps = false;
	bool retain_plan = true; // keep every emitted task for mt_plan_export (else drop them once taken)
	bool record_accesses = false;
	// cross-worker reduce trees as one allreduce task per worker (B200 extension; the
	// default keeps the reference's send-to-root tree, planner.cpp:389-517)
	bool collective_reduce = false;
	// replay the plan of an identical earlier launch when the conflict state of every chunk it
	// touches is that launch's state with task ids moved (iterative loops: plan once, replay)
	bool plan_cache = true;
};

struct launch_arg {
	enum kind_t { int_k, float_k, array_k } kind = array_k;
	int64_t i = 0;
	double f = 0.0;
	int64_t array = -1;
};

struct array_rec {
	int64_t id = -1;
	box domain;
	dtype type = dtype::f32;
	std::vector<chunk_desc> chunks; // ascending id
	chunk_index index;
};

struct chunk_meta {
	chunk_desc desc;
	dtype type = dtype::f32;
	bool temp = false;
};

class planner {
  public:
	explicit planner(const planner_config& cfg);

	const std::vector<device_id>& devices() const { return devices_; }
	const planner_config& config() const { return cfg_; }

	const array_rec& create_array(const box& domain, dtype type, std::vector<chunk_desc> chunks, fill_kind fill);
	void delete_array(int64_t id);
	// the array's chunks were filled outside the plan (mt_array_write's synchronous upload)
	void mark_filled(int64_t id);
	std::pair<int64_t, int64_t> launch(const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
	    const std::vector<launch_arg>& args, const annotation& ann);

	// B200 extension: asynchronous host <-> array transfers planned as tasks, so they are
	// ordered against launches by the same dependency tracking. write: every chunk's region
	// from the host array (row-major over the domain); read: a disjoint cover of the domain
	// (each cell from the lowest-id chunk holding it) into the host array. Returns the task
	// range like launch().
	std::pair<int64_t, int64_t> host_transfer(int64_t array_id, uint64_t host_addr, bool write, const box* host_box = nullptr);

	std::vector<task> take_pending(); // copies (the C++ adapter / tests)
	// hands every task emitted since the previous call to `f` (by reference, in id order, no
	// copies), then drops them from memory unless the plan is retained
	template <class F> void consume_pending(F&& f) {
		for(int64_t id = pending_from_; id < next_task_; ++id) f(plan_[static_cast<size_t>(id - plan_base_)]);
		pending_from_ = next_task_;
		if(!cfg_.retain_plan) {
			plan_.clear();
			plan_base_ = next_task_;
		}
	}
	// context-local kernels shadow the global registry (the reference registers synthesized
	// gather kernels per scenario, scenario.cpp:368-389)
	void add_local_kernel(kernel_entry e);
	const kernel_entry* find_kernel(const std::string& id) const;
	const array_rec& array(int64_t id) const;
	const chunk_meta& chunk(int64_t id) const;
	const std::deque<task>& plan() const { return plan_; } // tasks [plan_base(), next_id()); appends never move them
	int64_t plan_base() const { return plan_base_; }
	int64_t next_id() const { return next_task_; }
	struct access_rec {
		int64_t task, chunk;
		box region;
		bool write;
	};
	const std::vector<access_rec>& accesses() const { return accesses_; }
	uint64_t plan_cache_hits() const { return memo_hits_; }

  private:
	planner_config cfg_;
	std::vector<device_id> devices_;
	dep_tracker deps_;
	std::map<int64_t, std::unique_ptr<array_rec>> arrays_;
	int64_t next_array_ = 0;
	int64_t next_chunk_ = 0;
	int64_t next_task_ = 0;
	std::unordered_map<int64_t, chunk_meta> chunks_;
	std::deque<task> plan_;
	int64_t plan_base_ = 0;    // id of plan_.front()
	int64_t pending_from_ = 0; // first id not yet handed to the executor
	std::map<std::pair<int, int>, uint64_t> tags_;
	uint64_t collectives_ = 0; // allreduce group ids, in plan order
	std::unordered_map<int64_t, std::vector<int64_t>> temp_users_;
	std::vector<std::vector<int64_t>> spare_users_;
	std::vector<std::unique_ptr<kernel_entry>> local_kernels_;
	std::vector<access_rec> accesses_;

	std::pair<int64_t, int64_t> plan_launch(const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
	    const std::vector<launch_arg>& args, const annotation& ann);

	// ---- launch-plan memo (plan cache) ----------------------------------------------------
	struct launch_memo {
		std::string kernel;
		box grid;
		point block;
		std::vector<superblock> work;
		std::vector<launch_arg> args;
		const annotation* ann = nullptr;
		int64_t first = 0;
		std::vector<task> tasks;
		std::map<std::pair<int, int>, uint64_t> tags_before, tags_used; // per (src, dst) worker pair
		std::vector<int64_t> chunks;
		std::vector<dep_tracker::snapshot> before, after;
		std::vector<access_rec> accesses;
	};
	std::deque<launch_memo> memos_;
	bool recording_ = false;
	std::vector<int64_t> rec_chunks_;
	std::vector<dep_tracker::snapshot> rec_before_;
	uint64_t memo_hits_ = 0;
	bool same_call(const launch_memo& m, const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
	    const std::vector<launch_arg>& args, const annotation& ann) const;
	bool replay(const launch_memo& m, std::pair<int64_t, int64_t>& out);

	int64_t emit(task&& t);
	int64_t new_temp(const box& region, device_id home, dtype type);
	// users of a launch's temporaries (the delete task waits for them); the lists' storage is
	// recycled across temporaries
	void touch(int64_t temp, int64_t t) {
		auto [it, fresh] = temp_users_.try_emplace(temp);
		if(fresh && !spare_users_.empty()) {
			it->second = std::move(spare_users_.back());
			spare_users_.pop_back();
		}
		it->second.push_back(t);
	}
	// the delete task of a temporary: waits for its users; the temporary's metadata is dropped
	// with it unless the plan is retained for inspection (mt_chunk_meta)
	void emit_delete_temp(int worker, device_id dev, int64_t temp);
	void record(int64_t chunk, int64_t t, bool write, const box& region, bool check_filled, std::vector<int64_t>& out);
	int64_t transfer(int64_t src, int64_t dst, const box& region, std::vector<int64_t> src_deps, std::vector<int64_t> dst_deps);
	int64_t emit_create(int worker, device_id dev, int64_t chunk, fill_kind fill, reduce_op op);
};

} // namespace mtb
