#include "distribution.hpp"

#include <numeric>

namespace mtb {

std::string to_string(const point& p) {
	std::string s = "(";
	for(int k = 0; k < p.rank; ++k) s += (k ? "," : "") + std::to_string(p[k]);
	return s + ")";
}

std::string to_string(const box& b) {
	std::string s;
	for(int k = 0; k < b.rank(); ++k) s += (k ? "x[" : "[") + std::to_string(b.lo[k]) + "," + std::to_string(b.hi[k]) + ")";
	return s;
}

void validate_work(const std::vector<superblock>& sbs, const box& block_grid) {
	int64_t covered = 0;
	for(size_t i = 0; i < sbs.size(); ++i) {
		const box& r = sbs[i].blocks;
		if(r.is_empty()) throw validation_error("superblock " + std::to_string(i) + " is empty");
		if(!encloses(block_grid, r)) throw validation_error("superblock " + std::to_string(i) + " exceeds the launch grid");
		covered += r.volume();
	}
	// pairwise disjointness by a sweep along axis 0
	std::vector<size_t> order(sbs.size());
	std::iota(order.begin(), order.end(), size_t{0});
	std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return sbs[a].blocks.lo[0] < sbs[b].blocks.lo[0]; });
	for(size_t x = 0; x < order.size(); ++x) {
		const box& a = sbs[order[x]].blocks;
		for(size_t y = x + 1; y < order.size() && sbs[order[y]].blocks.lo[0] < a.hi[0]; ++y) {
			if(overlaps(a, sbs[order[y]].blocks)) {
				const size_t i = std::min(order[x], order[y]), j = std::max(order[x], order[y]);
				throw validation_error("superblocks " + std::to_string(i) + " and " + std::to_string(j) + " overlap");
			}
		}
	}
	if(covered != block_grid.volume()) throw validation_error("superblocks do not cover the launch grid");
}

void validate_chunks(const std::vector<chunk_desc>& chunks, const box& domain) {
	if(chunks.empty()) throw validation_error("data distribution has no chunks");
	for(const auto& c : chunks) {
		if(c.region.is_empty()) throw validation_error("chunk " + std::to_string(c.id) + " is empty");
		if(!encloses(domain, c.region)) throw validation_error("chunk " + std::to_string(c.id) + " exceeds the array domain");
	}
	// coverage: compress coordinates per axis, paint each chunk's cells, sum painted volume
	const int rank = domain.rank();
	std::vector<int64_t> cuts[kMaxRank];
	for(int k = 0; k < rank; ++k) {
		cuts[k].reserve(2 * chunks.size() + 2);
		cuts[k].push_back(domain.lo[k]);
		cuts[k].push_back(domain.hi[k]);
		for(const auto& c : chunks) {
			cuts[k].push_back(c.region.lo[k]);
			cuts[k].push_back(c.region.hi[k]);
		}
		std::sort(cuts[k].begin(), cuts[k].end());
		cuts[k].erase(std::unique(cuts[k].begin(), cuts[k].end()), cuts[k].end());
	}
	size_t dims[kMaxRank] = {1, 1, 1};
	size_t cells = 1;
	for(int k = 0; k < rank; ++k) {
		dims[k] = cuts[k].size() - 1;
		cells *= dims[k];
	}
	if(cells > (size_t{1} << 28)) throw validation_error("data distribution too irregular to validate");
	std::vector<uint8_t> painted(cells, 0);
	const auto pos = [&](int k, int64_t v) { return static_cast<size_t>(std::lower_bound(cuts[k].begin(), cuts[k].end(), v) - cuts[k].begin()); };
	for(const auto& c : chunks) {
		size_t lo[kMaxRank] = {0, 0, 0}, hi[kMaxRank] = {1, 1, 1};
		for(int k = 0; k < rank; ++k) {
			lo[k] = pos(k, c.region.lo[k]);
			hi[k] = pos(k, c.region.hi[k]);
		}
		for(size_t a = lo[0]; a < hi[0]; ++a)
			for(size_t b = lo[1]; b < hi[1]; ++b)
				for(size_t d = lo[2]; d < hi[2]; ++d) painted[(a * dims[1] + b) * dims[2] + d] = 1;
	}
	int64_t covered = 0;
	for(size_t a = 0; a < dims[0]; ++a)
		for(size_t b = 0; b < dims[1]; ++b)
			for(size_t d = 0; d < dims[2]; ++d) {
				if(!painted[(a * dims[1] + b) * dims[2] + d]) continue;
				int64_t v = cuts[0][a + 1] - cuts[0][a];
				if(rank > 1) v *= cuts[1][b + 1] - cuts[1][b];
				if(rank > 2) v *= cuts[2][d + 1] - cuts[2][d];
				covered += v;
			}
	if(covered != domain.volume()) throw validation_error("data distribution does not cover the array domain");
}

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// tiles of `ext` over `dom` in row-major tile order
template <typename Fn>
void tiles(const box& dom, const point& ext, Fn&& fn) {
	const int rank = dom.rank();
	int64_t count[kMaxRank] = {1, 1, 1};
	for(int k = 0; k < rank; ++k) {
		if(ext[k] <= 0) throw validation_error("chunk/superblock extents must be positive");
		count[k] = ceil_div(dom.extent(k), ext[k]);
	}
	int64_t index = 0;
	for(int64_t a = 0; a < count[0]; ++a)
		for(int64_t b = 0; b < count[1]; ++b)
			for(int64_t c = 0; c < count[2]; ++c) {
				const int64_t t[kMaxRank] = {a, b, c};
				box r;
				r.lo = point::zeros(rank);
				r.hi = point::zeros(rank);
				for(int k = 0; k < rank; ++k) {
					r.lo[k] = dom.lo[k] + t[k] * ext[k];
					r.hi[k] = std::min(dom.hi[k], r.lo[k] + ext[k]);
				}
				fn(index++, r);
			}
}

} // namespace

std::vector<superblock> block_work_dist(const box& grid, const point& block, const point& tps, const std::vector<device_id>& devices) {
	if(devices.empty()) throw validation_error("no devices");
	if(grid.rank() != block.rank || grid.rank() != tps.rank) throw validation_error("axis-count mismatch in work distribution");
	point per_sb = point::zeros(grid.rank()), blocks = point::zeros(grid.rank());
	for(int k = 0; k < grid.rank(); ++k) {
		if(block[k] <= 0) throw validation_error("block size must be positive");
		if(tps[k] % block[k] != 0)
			throw validation_error("superblock extent " + std::to_string(tps[k]) + " is not a multiple of block size " + std::to_string(block[k]) + " on axis "
			                       + std::to_string(k));
		per_sb[k] = tps[k] / block[k];
		blocks[k] = ceil_div(grid.extent(k), block[k]);
	}
	const box bgrid = box::extents(blocks);
	std::vector<superblock> out;
	tiles(bgrid, per_sb, [&](int64_t i, const box& r) { out.push_back({r, devices[static_cast<size_t>(i) % devices.size()]}); });
	validate_work(out, bgrid);
	return out;
}

std::vector<chunk_desc> tile_dist(const box& domain, const point& ext, const point& halo, const std::vector<device_id>& devices, int64_t first_id) {
	if(devices.empty()) throw validation_error("no devices");
	if(domain.rank() != ext.rank || domain.rank() != halo.rank) throw validation_error("axis-count mismatch in data distribution");
	for(int k = 0; k < domain.rank(); ++k)
		if(halo[k] < 0) throw validation_error("halo must be non-negative");
	std::vector<chunk_desc> out;
	tiles(domain, ext, [&](int64_t i, const box& interior) {
		box r = interior;
		for(int k = 0; k < domain.rank(); ++k) {
			r.lo[k] = std::max(domain.lo[k], r.lo[k] - halo[k]);
			r.hi[k] = std::min(domain.hi[k], r.hi[k] + halo[k]);
		}
		out.push_back({first_id + i, r, devices[static_cast<size_t>(i) % devices.size()]});
	});
	validate_chunks(out, domain);
	return out;
}

std::vector<chunk_desc> replicated_dist(const box& domain, const std::vector<device_id>& devices, int64_t first_id) {
	if(devices.empty()) throw validation_error("no devices");
	std::vector<chunk_desc> out;
	for(size_t i = 0; i < devices.size(); ++i) out.push_back({first_id + static_cast<int64_t>(i), domain, devices[i]});
	validate_chunks(out, domain);
	return out;
}

std::vector<chunk_desc> single_dist(const box& domain, device_id home, int64_t first_id) {
	std::vector<chunk_desc> out{{first_id, domain, home}};
	validate_chunks(out, domain);
	return out;
}

void chunk_index::build(const std::vector<chunk_desc>& chunks) {
	chunks_ = &chunks;
	by_lo0_.resize(chunks.size());
	std::iota(by_lo0_.begin(), by_lo0_.end(), 0);
	std::stable_sort(by_lo0_.begin(), by_lo0_.end(), [&](int a, int b) { return chunks[static_cast<size_t>(a)].region.lo[0] < chunks[static_cast<size_t>(b)].region.lo[0]; });
	max_hi0_.resize(chunks.size());
	int64_t m = INT64_MIN;
	for(size_t i = 0; i < by_lo0_.size(); ++i) {
		m = std::max(m, chunks[static_cast<size_t>(by_lo0_[i])].region.hi[0]);
		max_hi0_[i] = m;
	}
}

void chunk_index::query(const box& region, std::vector<int>& out) const {
	out.clear();
	if(region.is_empty()) return;
	const auto& chunks = *chunks_;
	// chunks with lo[0] < region.hi[0]; among those skip prefixes whose max hi[0] <= region.lo[0]
	const auto end = std::lower_bound(by_lo0_.begin(), by_lo0_.end(), region.hi[0],
	    [&](int c, int64_t v) { return chunks[static_cast<size_t>(c)].region.lo[0] < v; });
	const size_t n = static_cast<size_t>(end - by_lo0_.begin());
	const size_t start = static_cast<size_t>(std::upper_bound(max_hi0_.begin(), max_hi0_.begin() + static_cast<std::ptrdiff_t>(n), region.lo[0]) - max_hi0_.begin());
	for(size_t i = start; i < n; ++i) {
		const int c = by_lo0_[i];
		if(overlaps(chunks[static_cast<size_t>(c)].region, region)) out.push_back(c);
	}
	std::sort(out.begin(), out.end());
}

int select_enclosing(const std::vector<chunk_desc>& chunks, const std::vector<int>& candidates, const box& region, device_id executor) {
	int best = -1, best_score = -1;
	for(const int c : candidates) {
		const auto& d = chunks[static_cast<size_t>(c)];
		if(!encloses(d.region, region)) continue;
		const int score = d.home == executor ? 2 : (d.home.worker == executor.worker ? 1 : 0);
		if(score > best_score) {
			best = c;
			best_score = score;
		}
	}
	return best;
}

} // namespace mtb
