// Work and data distributions (the reference's L2 layer, proj/src/distribution.cpp).
//
// Behaviour parity: superblock tiling round-robin over devices (:110-134), tiled chunks with
// clipped halos (:136-178), replicated / single (:180-195), coverage + disjointness
// validation (:10-73), intersect query in ascending id (:197-205), enclosing-chunk
// preference same device > same worker > lowest id (:207-220).
//
// B200 changes: validation is O(S log S) (sweep) for work and O(cells painted) for data
// (coordinate-compressed bitmap instead of the reference's per-cell scan over all chunks),
// and intersect queries go through a per-array index (chunk_index) instead of a linear scan,
// so planning 400-800-chunk out-of-core launches stays in microseconds.
#pragma once

#include <vector>

#include "geometry.hpp"

namespace mtb {

struct superblock {
	box blocks; // thread-block index space
	device_id device;
};

struct chunk_desc {
	int64_t id = -1;
	box region;
	device_id home;
};

void validate_work(const std::vector<superblock>& sbs, const box& block_grid);
void validate_chunks(const std::vector<chunk_desc>& chunks, const box& domain);

std::vector<superblock> block_work_dist(const box& grid, const point& block, const point& threads_per_sb, const std::vector<device_id>& devices);
std::vector<chunk_desc> tile_dist(const box& domain, const point& extents, const point& halo, const std::vector<device_id>& devices, int64_t first_id);
std::vector<chunk_desc> replicated_dist(const box& domain, const std::vector<device_id>& devices, int64_t first_id);
std::vector<chunk_desc> single_dist(const box& domain, device_id home, int64_t first_id);

// Spatial index over one array's chunks. Queries return chunk positions (indices into the
// array's chunk list, which is in ascending id order) intersecting a box, ascending.
class chunk_index {
  public:
	void build(const std::vector<chunk_desc>& chunks);
	void query(const box& region, std::vector<int>& out) const;

  private:
	const std::vector<chunk_desc>* chunks_ = nullptr;
	// chunks sorted by lo[0] plus the running max of hi[0] for pruning
	std::vector<int> by_lo0_;
	std::vector<int64_t> max_hi0_;
};

// Among `candidates` (positions into `chunks`, ascending), the one whose region encloses
// `region` with the best preference; -1 if none encloses it.
int select_enclosing(const std::vector<chunk_desc>& chunks, const std::vector<int>& candidates, const box& region, device_id executor);

} // namespace mtb
