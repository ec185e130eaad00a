// Process-global kernel registry: signatures for the planner's validation and the device
// launchers for the executor (the reference's kernel_registry, kernels.hpp:94-105, with the
// std::function CPU body replaced by an ahead-of-time compiled sm_100a launcher).
#pragma once

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/manta_b200.h"
#include "geometry.hpp"

namespace mtb {

struct param_sig {
	std::string name;
	bool is_array = false;
	dtype type = dtype::f32;
	int rank = 0;
	bool writable = false;
};

struct kernel_entry {
	std::string id;
	std::vector<param_sig> params;
	mt_launcher_fn launcher = nullptr;
	const void* user = nullptr; // passed to the launcher as mt_launch_ctx::user
	// every cell of a declared `write` region (inside the array domain) is written by the
	// kernel; lets the spill tier skip restoring data that is about to be overwritten
	bool dense_writes = false;
	// param index whose writes the launcher can store a second time into a neighbouring chunk
	// (mt_launch_ctx mirrors: halo copies fused into the producing kernel); -1: none
	int mirror_param = -1;
};

class kernel_table {
  public:
	static kernel_table& get();

	int add(kernel_entry e);        // throws validation_error on duplicates / bad ranks
	int find(const std::string& id) const; // -1 when absent
	const kernel_entry& at(int index) const;
	int size() const;
	void set_dense_writes(const std::string& id); // see kernel_entry::dense_writes
	void set_mirror_param(const std::string& id, int param); // see kernel_entry::mirror_param

  private:
	kernel_table();
	mutable std::mutex mu_;
	std::vector<kernel_entry*> entries_; // stable addresses
	std::unordered_map<std::string, int> by_name_;
};

// defined in kernels/builtin.cu: registers every builtin kernel once
void register_builtin_kernels(kernel_table& t);

} // namespace mtb
