#include "deps.hpp"

namespace mtb {

void dep_tracker::add_chunk(int64_t chunk, const box& region) {
	state s;
	s.region = region;
	s.cells.push_back(cell{region, -1, {}});
	chunks_[chunk] = std::move(s);
}

void dep_tracker::drop_chunk(int64_t chunk) { chunks_.erase(chunk); }

dep_tracker::state& dep_tracker::get(int64_t chunk) {
	const auto it = chunks_.find(chunk);
	if(it == chunks_.end()) throw validation_error("unknown chunk " + std::to_string(chunk));
	return it->second;
}

const dep_tracker::state& dep_tracker::get(int64_t chunk) const {
	const auto it = chunks_.find(chunk);
	if(it == chunks_.end()) throw validation_error("unknown chunk " + std::to_string(chunk));
	return it->second;
}

void dep_tracker::mark_created(int64_t chunk, int64_t creator, bool filled) {
	state& s = get(chunk);
	s.cells.assign(1, cell{s.region, creator, {}});
	s.filled = filled;
}

bool dep_tracker::filled(int64_t chunk) const { return get(chunk).filled; }

size_t dep_tracker::cell_count(int64_t chunk) const { return get(chunk).cells.size(); }

// c minus cut (cut intersects c): slabs peeled axis by axis, plus the inside part
void dep_tracker::split(const cell& c, const box& cut, std::vector<cell>& inside, std::vector<cell>& outside) {
	box rest = c.region;
	for(int k = 0; k < rest.rank(); ++k) {
		if(rest.lo[k] < cut.lo[k]) {
			cell piece = c;
			piece.region = rest;
			piece.region.hi[k] = cut.lo[k];
			outside.push_back(std::move(piece));
			rest.lo[k] = cut.lo[k];
		}
		if(cut.hi[k] < rest.hi[k]) {
			cell piece = c;
			piece.region = rest;
			piece.region.lo[k] = cut.hi[k];
			outside.push_back(std::move(piece));
			rest.hi[k] = cut.hi[k];
		}
	}
	cell in = c;
	in.region = rest;
	inside.push_back(std::move(in));
}

// merges neighbouring cells with identical state whose union is a box
void dep_tracker::coalesce(std::vector<cell>& cells) {
	bool merged = true;
	while(merged && cells.size() > 1) {
		merged = false;
		for(size_t a = 0; a < cells.size() && !merged; ++a) {
			for(size_t b = a + 1; b < cells.size() && !merged; ++b) {
				cell& x = cells[a];
				const cell& y = cells[b];
				if(x.writer != y.writer || x.readers != y.readers) continue;
				const int rank = x.region.rank();
				int axis = -1;
				bool ok = true;
				for(int k = 0; k < rank && ok; ++k) {
					if(x.region.lo[k] == y.region.lo[k] && x.region.hi[k] == y.region.hi[k]) continue;
					if(axis >= 0) ok = false;
					else if(x.region.hi[k] == y.region.lo[k] || y.region.hi[k] == x.region.lo[k]) axis = k;
					else ok = false;
				}
				if(!ok || axis < 0) continue;
				x.region.lo[axis] = std::min(x.region.lo[axis], y.region.lo[axis]);
				x.region.hi[axis] = std::max(x.region.hi[axis], y.region.hi[axis]);
				cells.erase(cells.begin() + static_cast<std::ptrdiff_t>(b));
				merged = true;
			}
		}
	}
}

void dep_tracker::read(int64_t chunk, int64_t task, const box& region_in, std::vector<int64_t>& deps) {
	state& s = get(chunk);
	const box region = compat_ ? s.region : intersect(region_in, s.region);
	if(region.is_empty()) return;
	// scratch lists reused across calls (the planner is single-threaded per context; thread_local
	// keeps contexts on different threads apart); untouched cells are moved, not copied
	static thread_local std::vector<cell> keep, inside;
	keep.clear();
	inside.clear();
	for(auto& c : s.cells) {
		if(!overlaps(c.region, region)) {
			keep.push_back(std::move(c));
			continue;
		}
		if(c.writer >= 0) deps.push_back(c.writer);
		split(c, region, inside, keep);
	}
	for(auto& c : inside) {
		const auto it = std::lower_bound(c.readers.begin(), c.readers.end(), task);
		if(it == c.readers.end() || *it != task) c.readers.insert(it, task);
		keep.push_back(std::move(c));
	}
	s.cells.swap(keep);
	keep.clear();
	coalesce(s.cells);
}

void dep_tracker::write(int64_t chunk, int64_t task, const box& region_in, std::vector<int64_t>& deps) {
	state& s = get(chunk);
	const box region = compat_ ? s.region : intersect(region_in, s.region);
	if(region.is_empty()) return;
	static thread_local std::vector<cell> keep, inside;
	keep.clear();
	inside.clear();
	for(auto& c : s.cells) {
		if(!overlaps(c.region, region)) {
			keep.push_back(std::move(c));
			continue;
		}
		if(c.writer >= 0) deps.push_back(c.writer);
		for(const auto r : c.readers)
			if(r != task) deps.push_back(r);
		split(c, region, inside, keep);
	}
	keep.push_back(cell{region, task, {}});
	s.cells.swap(keep);
	keep.clear();
	s.filled = true;
	coalesce(s.cells);
}

} // namespace mtb
