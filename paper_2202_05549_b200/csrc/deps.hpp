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
//
// Cost. The reference's registry is O(1) per access (array_registry.cpp:41-60). Cells of a
// chunk are kept in an ordered map keyed by their low corner along one index axis (the axis
// the accesses split, chosen and re-chosen from the cells' shapes), with a count of cell
// extents along that axis: an access visits only cells whose low corner lies within
// (max extent) of its box, and coalesces only the cells around the box it touched. Band
// accesses of one chunk by S superblocks cost O(log S) each instead of O(S^2).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <unordered_map>
#include <utility>
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
	// host upload outside the plan (mt_array_write): the chunk holds defined data from now on
	void mark_filled(int64_t chunk);

	// Records an access over `region` (clipped to the chunk) and appends the tasks the
	// accessor must wait for to `deps` (unsorted, may contain duplicates).
	void read(int64_t chunk, int64_t task, const box& region, std::vector<int64_t>& deps);
	void write(int64_t chunk, int64_t task, const box& region, std::vector<int64_t>& deps);

	size_t cell_count(int64_t chunk) const;
	int index_axis(int64_t chunk) const;

	// Launch-plan memo support (planner.cpp, plan cache): a chunk's complete conflict state, and
	// the test / restore of "the same state with every task id moved by delta".
	struct snapshot;
	snapshot save(int64_t chunk) const;
	bool matches(int64_t chunk, const snapshot& s, int64_t delta) const;
	void restore(int64_t chunk, const snapshot& s, int64_t delta);

  private:
	// Ascending task ids. Up to kInline live in the cell itself: the cells of band and halo
	// accesses carry one to three readers, and splitting a cell copies its list, so an inline
	// list keeps the planner's hot path free of heap traffic (the allocator was a quarter of
	// the planning time at 1024 superblocks per chunk).
	class reader_list {
	  public:
		reader_list() = default;
		reader_list(const reader_list&) = default;
		reader_list& operator=(const reader_list&) = default;
		reader_list(reader_list&& o) noexcept { *this = std::move(o); }
		reader_list& operator=(reader_list&& o) noexcept {
			if(this == &o) return *this;
			n_ = o.n_;
			heap_on_ = o.heap_on_;
			heap_ = std::move(o.heap_);
			if(!heap_on_) std::copy(o.inline_, o.inline_ + n_, inline_);
			o.n_ = 0;
			o.heap_on_ = false;
			o.heap_.clear();
			return *this;
		}
		int64_t* begin() { return heap_on_ ? heap_.data() : inline_; }
		int64_t* end() { return begin() + n_; }
		const int64_t* begin() const { return heap_on_ ? heap_.data() : inline_; }
		const int64_t* end() const { return begin() + n_; }
		size_t size() const { return n_; }
		int64_t operator[](size_t i) const { return begin()[i]; }
		void insert(int64_t task); // keeps the order, ignores a task already present
		bool operator==(const reader_list& o) const;
		bool operator!=(const reader_list& o) const { return !(*this == o); }

	  private:
		static constexpr uint32_t kInline = 6;
		int64_t inline_[kInline] = {};
		uint32_t n_ = 0;
		bool heap_on_ = false;
		std::vector<int64_t> heap_;
	};
	// Readers of part of a cell: (task, the box it read, inside the cell). A read never splits
	// cells; a later write depends on a partial reader only when their boxes overlap, which is
	// the edge set the split cells gave, without restructuring the map on every halo read.
	struct partial_read {
		int64_t task;
		box region;
		bool operator==(const partial_read& o) const { return task == o.task && region == o.region; }
	};
	static constexpr size_t kMaxPartial = 8; // past this a partial read splits the cell
	struct cell {
		box region;
		int64_t writer = -1;
		reader_list readers;               // read the whole cell
		std::vector<partial_read> partial; // read part of it (ascending task, then first come)
	};
	using key = std::array<int64_t, kMaxRank>; // low corner, index axis first
	struct state {
		box region;
		bool filled = false;
		int axis = 0;                        // index axis
		std::map<key, cell> cells;           // disjoint, covering `region`
		// (cell extent along `axis`, count), ascending extent; a handful of distinct values
		std::vector<std::pair<int64_t, int64_t>> extents;
		int64_t probes = 0, hits = 0;        // scan efficiency since the last axis check
	};

	bool compat_;
	std::unordered_map<int64_t, state> chunks_;

  public:
	struct snapshot {
		state st;
	};

  private:

	state& get(int64_t chunk);
	const state& get(int64_t chunk) const;
	static key key_of(const state& s, const box& b);
	static int64_t reach(const state& s) { return s.extents.empty() ? 0 : s.extents.back().first; }
	static void count_extent(state& s, int64_t e, int64_t by);
	static void insert(state& s, cell&& c);
	static cell take(state& s, std::map<key, cell>::iterator it);
	// map nodes taken out of a cell map, kept per thread for the next insert (splitting and
	// coalescing cells then reuses nodes instead of going through the allocator)
	static std::vector<std::map<key, cell>::node_type>& spare_nodes();
	// moves every cell overlapping `q` out of the map into `out`
	static void extract(state& s, const box& q, std::vector<cell>& out);
	static void reindex(state& s);
	static void split(cell&& c, const box& cut, std::vector<cell>& inside, std::vector<cell>& outside);
	// partial readers of c clipped to c's region (a clip covering all of it makes a full reader)
	static void clip_partial(cell& c);
	void settle(state& s, const box& touched);
};

} // namespace mtb
