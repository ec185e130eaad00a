// Geometry, element types and error kinds of the B200 planner.
//
// Semantics follow the reference's L0 layer (proj/include/manta/geometry.hpp:15-118,
// dtype.hpp:13-55, errors.hpp:9-35): half-open boxes with canonical emptiness, closed
// intervals for linear-expression evaluation (a negative coefficient swaps the ends), and
// four error kinds that surface through the C-ABI as MT_E* codes. Everything is a fixed-size
// value type so the planner's hot loops never allocate.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace mtb {

constexpr int kMaxRank = 3;

// ---- errors ---------------------------------------------------------------------------

struct error : std::runtime_error {
	using std::runtime_error::runtime_error;
};
struct parse_error : error {
	parse_error(int line, int col, const std::string& what)
	    : error("parse error at " + std::to_string(line) + ":" + std::to_string(col) + ": " + what), line(line), col(col) {}
	int line, col;
};
struct validation_error : error {
	using error::error;
};
struct plan_error : error {
	using error::error;
};
struct execution_error : error {
	using error::error;
};

// ---- element types --------------------------------------------------------------------

enum class dtype : int32_t { i32 = 0, i64 = 1, f32 = 2, f64 = 3, bf16 = 4 };

inline size_t dtype_size(dtype t) {
	switch(t) {
	case dtype::i32: return 4;
	case dtype::i64: return 8;
	case dtype::f32: return 4;
	case dtype::f64: return 8;
	case dtype::bf16: return 2;
	}
	throw validation_error("unknown element type");
}
inline const char* dtype_name(dtype t) {
	switch(t) {
	case dtype::i32: return "i32";
	case dtype::i64: return "i64";
	case dtype::f32: return "f32";
	case dtype::f64: return "f64";
	case dtype::bf16: return "bf16";
	}
	return "?";
}
inline bool dtype_integral(dtype t) { return t == dtype::i32 || t == dtype::i64; }

// ---- points and boxes -----------------------------------------------------------------

struct point {
	int rank = 1;
	std::array<int64_t, kMaxRank> v{0, 0, 0};

	static point zeros(int rank) {
		if(rank < 1 || rank > kMaxRank) throw validation_error("axis count must be between 1 and 3, got " + std::to_string(rank));
		point p;
		p.rank = rank;
		return p;
	}
	static point of(int rank, const int64_t* c) {
		point p = zeros(rank);
		for(int k = 0; k < rank; ++k) p.v[k] = c[k];
		return p;
	}
	int64_t& operator[](int k) { return v[static_cast<size_t>(k)]; }
	int64_t operator[](int k) const { return v[static_cast<size_t>(k)]; }
	bool operator==(const point& o) const {
		if(rank != o.rank) return false;
		for(int k = 0; k < rank; ++k)
			if(v[k] != o.v[k]) return false;
		return true;
	}
};

std::string to_string(const point& p);

// [lo, hi); any lo >= hi axis makes it empty, and all empty boxes of a rank are equal.
struct box {
	point lo, hi;

	box() = default;
	box(const point& l, const point& h) : lo(l), hi(h) {
		if(l.rank != h.rank) throw validation_error("rect lo/hi axis counts differ");
		for(int k = 0; k < l.rank; ++k)
			if(l[k] > h[k]) throw validation_error("rect has lo > hi on axis " + std::to_string(k));
	}
	static box empty(int rank) { return box(point::zeros(rank), point::zeros(rank)); }
	static box extents(const point& e) { return box(point::zeros(e.rank), e); }

	int rank() const { return lo.rank; }
	bool is_empty() const {
		for(int k = 0; k < lo.rank; ++k)
			if(hi[k] <= lo[k]) return true;
		return false;
	}
	int64_t extent(int k) const { return hi[k] - lo[k]; }
	int64_t volume() const {
		if(is_empty()) return 0;
		int64_t v = 1;
		for(int k = 0; k < rank(); ++k)
			if(__builtin_mul_overflow(v, extent(k), &v)) throw validation_error("rect volume overflows int64");
		return v;
	}
	bool operator==(const box& o) const {
		if(rank() != o.rank()) return false;
		const bool ea = is_empty(), eb = o.is_empty();
		if(ea || eb) return ea && eb;
		return lo == o.lo && hi == o.hi;
	}
	bool operator!=(const box& o) const { return !(*this == o); }
};

std::string to_string(const box& b);

inline void require_same_rank(const box& a, const box& b) {
	if(a.rank() != b.rank()) throw validation_error("axis-count mismatch: " + std::to_string(a.rank()) + " vs " + std::to_string(b.rank()));
}

inline box intersect(const box& a, const box& b) {
	require_same_rank(a, b);
	box r;
	r.lo = point::zeros(a.rank());
	r.hi = point::zeros(a.rank());
	for(int k = 0; k < a.rank(); ++k) {
		r.lo[k] = std::max(a.lo[k], b.lo[k]);
		r.hi[k] = std::min(a.hi[k], b.hi[k]);
		if(r.hi[k] <= r.lo[k]) return box::empty(a.rank());
	}
	return r;
}

inline bool overlaps(const box& a, const box& b) {
	for(int k = 0; k < a.rank(); ++k)
		if(std::max(a.lo[k], b.lo[k]) >= std::min(a.hi[k], b.hi[k])) return false;
	return true;
}

// every point of `inner` lies in `outer`; an empty inner box is contained in anything
inline bool encloses(const box& outer, const box& inner) {
	require_same_rank(outer, inner);
	if(inner.is_empty()) return true;
	for(int k = 0; k < outer.rank(); ++k)
		if(inner.lo[k] < outer.lo[k] || inner.hi[k] > outer.hi[k]) return false;
	return true;
}

inline box hull(const box& a, const box& b) {
	require_same_rank(a, b);
	if(a.is_empty()) return b.is_empty() ? box::empty(a.rank()) : b;
	if(b.is_empty()) return a;
	box r = a;
	for(int k = 0; k < a.rank(); ++k) {
		r.lo[k] = std::min(a.lo[k], b.lo[k]);
		r.hi[k] = std::max(a.hi[k], b.hi[k]);
	}
	return r;
}

// closed interval [lo, hi]; lo > hi encodes empty
struct span {
	int64_t lo = 0, hi = -1;
	bool is_empty() const { return lo > hi; }
	static span scaled(int64_t c, span s) {
		if(s.is_empty()) return {};
		return c < 0 ? span{c * s.hi, c * s.lo} : span{c * s.lo, c * s.hi};
	}
	static span sum(span a, span b) {
		if(a.is_empty() || b.is_empty()) return {};
		return {a.lo + b.lo, a.hi + b.hi};
	}
};

struct device_id {
	int worker = 0;
	int device = 0;
	bool operator==(const device_id& o) const { return worker == o.worker && device == o.device; }
	bool operator!=(const device_id& o) const { return !(*this == o); }
	bool operator<(const device_id& o) const { return worker != o.worker ? worker < o.worker : device < o.device; }
};

inline std::string to_string(const device_id& d) { return "w" + std::to_string(d.worker) + "d" + std::to_string(d.device); }

} // namespace mtb
