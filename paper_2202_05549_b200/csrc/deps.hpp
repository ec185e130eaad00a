// Conflict tracking for planned chunk accesses.
//
// The reference tracks one (last_writer, readers_since_write) pair per chunk
// (proj/src/array_registry.cpp:41-60), so a halo copy into row 1024 of a chunk orders after
// every task that touched ANY row of that chunk; a distributed stencil launch collapses into
// a serial chain (SURVEY finding 3). Here every chunk is a set of disjoint cells, each with
// its own writer and readers; an access conflicts only with the cells its box intersects.
//
//   * compat mode treats every access as touching the whole chunk and therefore emits
//     exactly the reference's edges (plan-parity tests use it);
//   * region mode emits a subset of those edges whose transitive closure still orders every
//     pair of conflicting accesses (each dropped edge is to a task whose cells were
//     overwritten, and the overwriting task is itself ordered after it).
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "geometry.hpp"

namespace mtb {

class dep_tracker {
  public:
	explicit dep_tracker(bool compat) : compat_(compat) {}

	void add_chunk(int64_t chunk, const box& region);
	void drop_chunk(int64_t chunk);
	bool known(int64_t chunk) const { return chunks_.count(chunk) != 0; }

	// Create task: `creator` becomes the writer of the whole chunk (array_registry.cpp:24-28)
	void mark_created(int64_t chunk, int64_t creator, bool filled);
	bool filled(int64_t chunk) const;

	// Records an access over `region` (clipped to the chunk) and appends the tasks the
	// accessor must wait for to `deps` (unsorted, may contain duplicates).
	void read(int64_t chunk, int64_t task, const box& region, std::vector<int64_t>& deps);
	void write(int64_t chunk, int64_t task, const box& region, std::vector<int64_t>& deps);

	size_t cell_count(int64_t chunk) const;

  private:
	struct cell {
		box region;
		int64_t writer = -1;
		std::vector<int64_t> readers; // ascending
	};
	struct state {
		box region;
		bool filled = false;
		std::vector<cell> cells; // disjoint, covering `region`
	};

	bool compat_;
	std::unordered_map<int64_t, state> chunks_;

	state& get(int64_t chunk);
	const state& get(int64_t chunk) const;
	static void split(const cell& c, const box& cut, std::vector<cell>& out_inside, std::vector<cell>& out_outside);
	static void coalesce(std::vector<cell>& cells);
};

} // namespace mtb
