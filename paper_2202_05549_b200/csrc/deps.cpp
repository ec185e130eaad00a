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

void dep_tracker::reader_list::insert(int64_t task) {
	int64_t* const p = std::lower_bound(begin(), end(), task);
	if(p != end() && *p == task) return;
	const size_t at = static_cast<size_t>(p - begin());
	if(!heap_on_ && n_ < kInline) {
		std::copy_backward(inline_ + at, inline_ + n_, inline_ + n_ + 1);
		inline_[at] = task;
		++n_;
		return;
	}
	if(!heap_on_) {
		heap_.assign(inline_, inline_ + n_);
		heap_on_ = true;
	}
	heap_.insert(heap_.begin() + static_cast<std::ptrdiff_t>(at), task);
	++n_;
}

bool dep_tracker::reader_list::operator==(const reader_list& o) const { return n_ == o.n_ && std::equal(begin(), end(), o.begin()); }

void dep_tracker::count_extent(state& s, int64_t e, int64_t by) {
	auto& v = s.extents;
	auto it = std::lower_bound(v.begin(), v.end(), e, [](const std::pair<int64_t, int64_t>& x, int64_t y) { return x.first < y; });
	if(it != v.end() && it->first == e) {
		if((it->second += by) == 0) v.erase(it);
	} else {
		v.insert(it, {e, by});
	}
}

std::vector<std::map<dep_tracker::key, dep_tracker::cell>::node_type>& dep_tracker::spare_nodes() {
	static thread_local std::vector<std::map<key, cell>::node_type> spare;
	return spare;
}

void dep_tracker::insert(state& s, cell&& c) {
	count_extent(s, c.region.hi[s.axis] - c.region.lo[s.axis], 1);
	const key k = key_of(s, c.region);
	auto& spare = spare_nodes();
	if(!spare.empty()) {
		auto nh = std::move(spare.back());
		spare.pop_back();
		nh.key() = k;
		nh.mapped() = std::move(c);
		s.cells.insert(std::move(nh));
		return;
	}
	s.cells.emplace(k, std::move(c));
}

dep_tracker::cell dep_tracker::take(state& s, std::map<key, cell>::iterator it) {
	auto nh = s.cells.extract(it);
	cell c = std::move(nh.mapped());
	auto& spare = spare_nodes();
	if(spare.size() < 4096) spare.push_back(std::move(nh));
	count_extent(s, c.region.hi[s.axis] - c.region.lo[s.axis], -1);
	return c;
}

// Cells are disjoint, so a cell overlapping q along the index axis has its low corner in
// (q.lo - max_extent, q.hi): the scan starts there and stops at q.hi.
void dep_tracker::extract(state& s, const box& q, std::vector<cell>& out) {
	const int ax = s.axis;
	const int64_t reach = dep_tracker::reach(s);
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
			cell piece{rest, c.writer, c.readers, c.partial};
			piece.region.hi[k] = cut.lo[k];
			clip_partial(piece);
			outside.push_back(std::move(piece));
			rest.lo[k] = cut.lo[k];
		}
		if(cut.hi[k] < rest.hi[k]) {
			cell piece{rest, c.writer, c.readers, c.partial};
			piece.region.lo[k] = cut.hi[k];
			clip_partial(piece);
			outside.push_back(std::move(piece));
			rest.hi[k] = cut.hi[k];
		}
	}
	c.region = rest;
	clip_partial(c);
	inside.push_back(std::move(c));
}

void dep_tracker::clip_partial(cell& c) {
	if(c.partial.empty()) return;
	size_t out = 0;
	for(size_t i = 0; i < c.partial.size(); ++i) {
		partial_read p = c.partial[i];
		if(!overlaps(p.region, c.region)) continue;
		p.region = intersect(p.region, c.region);
		if(p.region == c.region) {
			c.readers.insert(p.task);
			continue;
		}
		c.partial[out++] = p;
	}
	c.partial.resize(out);
	// a task now a full reader needs no partial entries
	if(!c.partial.empty())
		c.partial.erase(std::remove_if(c.partial.begin(), c.partial.end(),
		                    [&](const partial_read& p) { return std::binary_search(c.readers.begin(), c.readers.end(), p.task); }),
		    c.partial.end());
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
		const int64_t reach = dep_tracker::reach(s);
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
				if(x.writer != y.writer || x.readers != y.readers || !x.partial.empty() || !y.partial.empty() || !mergeable(x.region, y.region, u)) continue;
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
	// cells the box encloses gain a full reader, cells it cuts a partial one; the map is not
	// touched (no split, no coalescing)
	const int ax = s.axis;
	const int64_t reach = dep_tracker::reach(s);
	key from{std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min(), std::numeric_limits<int64_t>::min()};
	from[0] = region.lo[ax] - reach + 1;
	int64_t probes = 0;
	static thread_local std::vector<key> split_later;
	static thread_local std::vector<cell> inside, outside;
	split_later.clear();
	for(auto it = s.cells.lower_bound(from); it != s.cells.end() && it->first[0] < region.hi[ax]; ++it) {
		++probes;
		cell& c = it->second;
		if(!overlaps(c.region, region)) continue;
		++s.hits;
		if(c.writer >= 0) deps.push_back(c.writer);
		if(encloses(region, c.region)) {
			c.readers.insert(task);
			continue;
		}
		if(std::binary_search(c.readers.begin(), c.readers.end(), task)) continue;
		const box part = intersect(region, c.region);
		bool covered = false;
		for(const auto& p : c.partial)
			if(p.task == task && encloses(p.region, part)) covered = true;
		if(covered) continue;
		if(c.partial.size() < kMaxPartial) {
			c.partial.push_back({task, part});
			continue;
		}
		// too many partial readers on one cell (band reads of one big chunk): cut the box out of
		// it, so the cell map converges to the read pattern and the lists stay short
		split_later.push_back(it->first);
	}
	s.probes += probes;
	for(const key& k : split_later) {
		const auto it = s.cells.find(k);
		cell c = take(s, it);
		split(std::move(c), region, inside, outside);
		for(auto& piece : inside) {
			piece.readers.insert(task);
			insert(s, std::move(piece));
		}
		for(auto& piece : outside) insert(s, std::move(piece));
		inside.clear();
		outside.clear();
	}
	if(!split_later.empty()) {
		split_later.clear();
		settle(s, region);
		return;
	}
	reindex(s);
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
		for(const auto& p : c.partial)
			if(p.task != task && overlaps(p.region, region)) deps.push_back(p.task);
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
		if(x->first != y->first || c.region != d.region || c.readers.size() != d.readers.size() || c.partial.size() != d.partial.size()) return false;
		if(c.writer != (d.writer < 0 ? d.writer : d.writer + delta)) return false;
		for(size_t k = 0; k < c.readers.size(); ++k)
			if(c.readers[k] != d.readers[k] + delta) return false;
		for(size_t k = 0; k < c.partial.size(); ++k)
			if(c.partial[k].task != d.partial[k].task + delta || c.partial[k].region != d.partial[k].region) return false;
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
		for(auto& p : c.partial) p.task += delta;
	}
}

} // namespace mtb
