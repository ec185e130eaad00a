#include "registry.hpp"

namespace mtb {

kernel_table& kernel_table::get() {
	static kernel_table* t = [] {
		auto* table = new kernel_table();
		register_builtin_kernels(*table);
		return table;
	}();
	return *t;
}

kernel_table::kernel_table() = default;

int kernel_table::add(kernel_entry e) {
	if(e.id.empty()) throw validation_error("kernel id must not be empty");
	if(e.id.size() >= MT_KERNEL_NAME_MAX) throw validation_error("kernel id too long");
	for(const auto& p : e.params)
		if(p.is_array && (p.rank < 1 || p.rank > kMaxRank))
			throw validation_error("kernel \"" + e.id + "\" parameter \"" + p.name + "\" has unsupported rank");
	std::lock_guard<std::mutex> lock(mu_);
	if(by_name_.count(e.id)) throw validation_error("kernel \"" + e.id + "\" is already registered");
	const int index = static_cast<int>(entries_.size());
	by_name_[e.id] = index;
	entries_.push_back(new kernel_entry(std::move(e)));
	return index;
}

int kernel_table::find(const std::string& id) const {
	std::lock_guard<std::mutex> lock(mu_);
	const auto it = by_name_.find(id);
	return it == by_name_.end() ? -1 : it->second;
}

const kernel_entry& kernel_table::at(int index) const {
	std::lock_guard<std::mutex> lock(mu_);
	if(index < 0 || index >= static_cast<int>(entries_.size())) throw validation_error("bad kernel index");
	return *entries_[static_cast<size_t>(index)];
}

void kernel_table::set_dense_writes(const std::string& id) {
	std::lock_guard<std::mutex> lock(mu_);
	const auto it = by_name_.find(id);
	if(it == by_name_.end()) throw validation_error("unknown kernel \"" + id + "\"");
	entries_[static_cast<size_t>(it->second)]->dense_writes = true;
}

void kernel_table::set_mirror_param(const std::string& id, int param) {
	std::lock_guard<std::mutex> lock(mu_);
	const auto it = by_name_.find(id);
	if(it == by_name_.end()) throw validation_error("unknown kernel \"" + id + "\"");
	entries_[static_cast<size_t>(it->second)]->mirror_param = param;
}

int kernel_table::size() const {
	std::lock_guard<std::mutex> lock(mu_);
	return static_cast<int>(entries_.size());
}

} // namespace mtb
