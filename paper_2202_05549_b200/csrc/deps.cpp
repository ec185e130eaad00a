#include "deps.hpp"

#include <algorithm>
#include <limits>

namespace mtb {

void dep_tracker::add_chunk(int64_t chunk, const box& region) {
	state s;
	s.region = region;
	insert(s, cell{region, -1, {}});
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
	s.cells.clear();
	s.extents.clear();
	insert(s, cell{s.region, creator, {}});
	s.filled = filled;
}

bool dep_tracker::filled(int64_t chunk) const { return get(chunk).filled; }

void dep_tracker::mark_filled(int64_t chunk) { get(chunk).filled = true; }

size_t dep_tracker::cell_count(int64_t chunk) const { return get(chunk).cells.size(); }

int dep_tracker::index_axis(int64_t chunk) const { return get(chunk).axis; }

dep_tracker::key dep_tracker::key_of(const state& s, const box& b) {
	key k{0, 0, 0};
	const int r = b.rank();
	for(int i = 0; i < r; ++i) k[i] = b.lo[(s.axis + i) % r];
	return k;
}

void dep_tracker::insert(state& s, cell&& c) {
	++s.extents[c.region.hi[s.axis] - c.region.lo[s.axis]];
	const key k = key_of(s, c.region);
	s.cells.emplace(k, std::move(c));
}

dep_tracker::cell dep_tracker::take(state& s, std::map<key, cell>::iterator it) {
	cell c = std::move(it->second);
	s.cells.erase(it);
	const auto e = s.extents.find(c.region.hi[s.axis] - c.region.lo[s.axis]);
	if(--e->second == 0) s.extents.erase(e);
	return c;
}

// Cells are disjoint, so a cell overlapping q along the index axis has its low corner in
// (q.lo - max_extent, q.hi): the scan starts there and stops at q.hi.
void dep_tracker::extract(state& s, const box& q, std::vector<cell>& out) {
	const int ax = s.axis;
	const int64_t reach = s.extents.empty() ? 0 : s.extents.rbegin()->first;
	key from{std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min()};
	from[0] = q.lo[ax] - reach + 1;
	auto it = s.cells.lower_bound(from);
	int64_t probes = 0;
	while(it != s.cells.end() && it->first[0] < q.hi[ax]) {
		++probes;
		if(overlaps(it->second.region, q)) {
			++s.hits;
			const auto cur = it++;
			out.push_back(take(s, cur));
			continue;
		}
		++it;
	}
	s.probes += probes;
}

// Re-picks the index axis when scans visit many cells they do not touch: the axis along which
// the longest cell covers the smallest fraction of the chunk.
void dep_tracker::reindex(state& s) {
	const int r = s.region.rank();
	const bool wasteful = s.probes > 8 * (s.hits + 16);
	s.probes = s.hits = 0;
	if(!wasteful || r == 1 || s.cells.size() < 64) return;
	int best = s.axis;
	double best_frac = 2.0;
	for(int a = 0; a < r; ++a) {
		int64_t longest = 0;
		for(const auto& [k, c] : s.cells) longest = std::max(longest, c.region.hi[a] - c.region.lo[a]);
		const double frac = static_cast<double>(longest) / static_cast<double>(std::max<int64_t>(1, s.region.hi[a] - s.region.lo[a]));
		if(frac < best_frac - 1e-12) best_frac = frac, best = a;
	}
	if(best == s.axis) return;
	std::vector<cell> all;
	all.reserve(s.cells.size());
	for(auto& [k, c] : s.cells) all.push_back(std::move(c));
	s.cells.clear();
	s.extents.clear();
	s.axis = best;
	for(auto& c : all) insert(s, std::move(c));
}

// c minus cut (cut intersects c): slabs peeled axis by axis, plus the inside part
void dep_tracker::split(cell&& c, const box& cut, std::vector<cell>& inside, std::vector<cell>& outside) {
	box rest = c.region;
	for(int k = 0; k < rest.rank(); ++k) {
		if(rest.lo[k] < cut.lo[k]) {
			cell piece{rest, c.writer, c.readers};
			piece.region.hi[k] = cut.lo[k];
			outside.push_back(std::move(piece));
			rest.lo[k] = cut.lo[k];
		}
		if(cut.hi[k] < rest.hi[k]) {
			cell piece{rest, c.writer, c.readers};
			piece.region.lo[k] = cut.hi[k];
			outside.push_back(std::move(piece));
			rest.hi[k] = cut.hi[k];
		}
	}
	c.region = rest;
	inside.push_back(std::move(c));
}

// true (and the merged box in `out`) when two cells' union is a box
static bool mergeable(const box& x, const box& y, box& out) {
	const int rank = x.rank();
	int axis = -1;
	for(int k = 0; k < rank; ++k) {
		if(x.lo[k] == y.lo[k] && x.hi[k] == y.hi[k]) continue;
		if(axis >= 0) return false;
		if(x.hi[k] == y.lo[k] || y.hi[k] == x.lo[k]) axis = k;
		else return false;
	}
	if(axis < 0) return false;
	out = x;
	out.lo[axis] = std::min(x.lo[axis], y.lo[axis]);
	out.hi[axis] = std::max(x.hi[axis], y.hi[axis]);
	return true;
}

// coalesces the cells that touch `touched` (the box grown by one on every axis): any pair of
// mergeable cells created by this access has a member inside it. Cells stay in the map unless
// two of them merge.
void dep_tracker::settle(state& s, const box& touched) {
	box grown = touched;
	for(int k = 0; k < grown.rank(); ++k) --grown.lo[k], ++grown.hi[k];
	grown = intersect(grown, s.region);
	static thread_local std::vector<std::map<key, cell>::iterator> near;
	for(bool again = true; again;) {
		again = false;
		near.clear();
		const int ax = s.axis;
		const int64_t reach = s.extents.empty() ? 0 : s.extents.rbegin()->first;
		key from{std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min()};
		from[0] = grown.lo[ax] - reach + 1;
		for(auto it = s.cells.lower_bound(from); it != s.cells.end() && it->first[0] < grown.hi[ax]; ++it) {
			++s.probes;
			if(overlaps(it->second.region, grown)) near.push_back(it);
		}
		for(size_t a = 0; a < near.size() && !again; ++a) {
			for(size_t b = a + 1; b < near.size() && !again; ++b) {
				const cell& x = near[a]->second;
				const cell& y = near[b]->second;
				box u;
				if(x.writer != y.writer || x.readers != y.readers || !mergeable(x.region, y.region, u)) continue;
				cell m = take(s, near[a]);
				take(s, near[b]);
				m.region = u;
				insert(s, std::move(m));
				again = true;
			}
		}
	}
	near.clear();
	reindex(s);
}

void dep_tracker::read(int64_t chunk, int64_t task, const box& region_in, std::vector<int64_t>& deps) {
	state& s = get(chunk);
	const box region = compat_ ? s.region : intersect(region_in, s.region);
	if(region.is_empty()) return;
	// scratch lists reused across calls (the planner is single-threaded per context; thread_local
	// keeps contexts on different threads apart)
	static thread_local std::vector<cell> hit, inside, outside;
	hit.clear();
	inside.clear();
	outside.clear();
	// cells inside the box only gain a reader (in place); cells it cuts are split
	const int ax = s.axis;
	const int64_t reach = s.extents.empty() ? 0 : s.extents.rbegin()->first;
	key from{std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min()};
	from[0] = region.lo[ax] - reach + 1;
	int64_t probes = 0;
	for(auto it = s.cells.lower_bound(from); it != s.cells.end() && it->first[0] < region.hi[ax];) {
		++probes;
		cell& c = it->second;
		if(!overlaps(c.region, region)) {
			++it;
			continue;
		}
		++s.hits;
		if(c.writer >= 0) deps.push_back(c.writer);
		if(encloses(region, c.region)) {
			const auto r = std::lower_bound(c.readers.begin(), c.readers.end(), task);
			if(r == c.readers.end() || *r != task) c.readers.insert(r, task);
			++it;
			continue;
		}
		const auto cur = it++;
		hit.push_back(take(s, cur));
	}
	s.probes += probes;
	if(hit.empty()) return;
	for(auto& c : hit) split(std::move(c), region, inside, outside);
	for(auto& c : inside) {
		const auto it = std::lower_bound(c.readers.begin(), c.readers.end(), task);
		if(it == c.readers.end() || *it != task) c.readers.insert(it, task);
		insert(s, std::move(c));
	}
	for(auto& c : outside) insert(s, std::move(c));
	hit.clear();
	inside.clear();
	outside.clear();
	settle(s, region);
}

void dep_tracker::write(int64_t chunk, int64_t task, const box& region_in, std::vector<int64_t>& deps) {
	state& s = get(chunk);
	const box region = compat_ ? s.region : intersect(region_in, s.region);
	if(region.is_empty()) return;
	static thread_local std::vector<cell> hit, inside, outside;
	hit.clear();
	inside.clear();
	outside.clear();
	extract(s, region, hit);
	for(auto& c : hit) {
		if(c.writer >= 0) deps.push_back(c.writer);
		for(const auto r : c.readers)
			if(r != task) deps.push_back(r);
		split(std::move(c), region, inside, outside);
	}
	for(auto& c : outside) insert(s, std::move(c));
	insert(s, cell{region, task, {}});
	hit.clear();
	inside.clear();
	outside.clear();
	s.filled = true;
	settle(s, region);
}

dep_tracker::snapshot dep_tracker::save(int64_t chunk) const { return snapshot{get(chunk)}; }

bool dep_tracker::matches(int64_t chunk, const snapshot& snap, int64_t delta) const {
	const auto it = chunks_.find(chunk);
	if(it == chunks_.end()) return false;
	const state& a = it->second;
	const state& b = snap.st;
	if(a.filled != b.filled || a.axis != b.axis || a.cells.size() != b.cells.size() || a.region != b.region) return false;
	for(auto x = a.cells.begin(), y = b.cells.begin(); x != a.cells.end(); ++x, ++y) {
		const cell& c = x->second;
		const cell& d = y->second;
		if(x->first != y->first || c.region != d.region || c.readers.size() != d.readers.size()) return false;
		if(c.writer != (d.writer < 0 ? d.writer : d.writer + delta)) return false;
		for(size_t k = 0; k < c.readers.size(); ++k)
			if(c.readers[k] != d.readers[k] + delta) return false;
	}
	return true;
}

void dep_tracker::restore(int64_t chunk, const snapshot& snap, int64_t delta) {
	state& a = get(chunk);
	a = snap.st;
	a.probes = a.hits = 0;
	for(auto& [k, c] : a.cells) {
		if(c.writer >= 0) c.writer += delta;
		for(auto& r : c.readers) r += delta;
	}
}

} // namespace mtb
