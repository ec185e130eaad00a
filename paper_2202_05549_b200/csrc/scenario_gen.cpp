// Random scenario generator for the fuzz campaign (make_fuzz_scenario,
// proj/src/scenario.cpp:653-807, with its helpers var_name / random_expr / random_index at
// :617-650). The campaign (`python -m paper_2202_05549_b200 fuzz`) runs each scenario through
// the B200 planner + executor and compares it with the same scenario in oracle mode (one
// device, sequential), like run_fuzz_campaign (scenario.cpp:809-846).
//
// The draws use std::mt19937_64 and std::uniform_int_distribution in the reference's order,
// so a case seed yields the reference's scenario (pinned by tests/test_cli.py against the
// reference's own generator). Output is JSON in the scenario file format (scenario.cpp:131-167).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/manta_b200.h"

namespace {

using rng_t = std::mt19937_64;

std::string var_name(int axis) { return axis == 0 ? "i" : axis == 1 ? "j" : "k"; }

std::string random_expr(rng_t& rng, int rank) {
	std::uniform_int_distribution<int> coeff(-3, 3);
	std::uniform_int_distribution<int> constant(-5, 5);
	std::uniform_int_distribution<int> axis(0, rank - 1);
	const int c = coeff(rng);
	std::string s = std::to_string(c) + "*" + var_name(axis(rng));
	const int k = constant(rng);
	if(k >= 0) s += "+";
	return s + std::to_string(k);
}

std::string random_index(rng_t& rng, int rank) {
	std::uniform_int_distribution<int> form(0, 4);
	std::uniform_int_distribution<int> width(0, 3);
	switch(form(rng)) {
	case 0: return random_expr(rng, rank);
	case 1: return ":";
	case 2: return random_expr(rng, rank) + ":";
	case 3: return ":" + random_expr(rng, rank);
	default: {
		const std::string center = random_expr(rng, rank);
		// the reference builds this in one operator+ chain; g++ evaluates the right-hand
		// width(rng) first, so the upper width is drawn before the lower one
		const int hi = width(rng);
		const int lo = width(rng);
		return center + "-" + std::to_string(lo) + ":" + center + "+" + std::to_string(hi);
	}
	}
}

struct array_gen {
	std::string name;
	std::vector<int64_t> domain;
	std::string kind;
	int64_t rows = 0, cols = 0;
	std::vector<int64_t> extents, halo;
};

struct launch_gen {
	std::vector<int64_t> grid, block, superblock;
	std::string annotation;
	std::vector<std::string> args;
};

std::string ints(const std::vector<int64_t>& v) {
	std::string s = "[";
	for(size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
	return s + "]";
}

std::string quoted(const std::string& s) {
	std::string o = "\"";
	for(char c : s) {
		if(c == '"' || c == '\\') o += '\\';
		o += c;
	}
	return o + "\"";
}

std::string make_fuzz_scenario_json(uint64_t case_seed) {
	rng_t rng(case_seed);
	std::uniform_int_distribution<int> workers_dist(1, 2);
	std::uniform_int_distribution<int> devices_dist(1, 2);
	std::uniform_int_distribution<int> arrays_dist(3, 5);
	std::uniform_int_distribution<int> rank_dist(1, 2);
	using i64_dist = std::uniform_int_distribution<int64_t>;

	const int workers = workers_dist(rng);
	const int devices = devices_dist(rng);
	const uint64_t seed = rng();
	uint64_t device_capacity = 256ull << 20, host_capacity = 1ull << 30; // system_spec defaults (scenario.hpp:66-73)

	const int array_count = arrays_dist(rng);
	uint64_t total_bytes = 0;
	std::vector<array_gen> arrays;
	for(int a = 0; a < array_count; ++a) {
		array_gen g;
		g.name = "a" + std::to_string(a);
		const int rank = rank_dist(rng);
		if(rank == 1) {
			g.domain = {i64_dist(16, 96)(rng)};
		} else {
			const int64_t d0 = i64_dist(6, 20)(rng);
			const int64_t d1 = i64_dist(6, 20)(rng);
			g.domain = {d0, d1};
		}
		uint64_t volume = 1;
		for(auto e : g.domain) volume *= static_cast<uint64_t>(e);
		total_bytes += volume * 8;
		const int kind = std::uniform_int_distribution<int>(0, rank == 2 ? 5 : 4)(rng);
		switch(kind) {
		case 0:
			g.kind = "row";
			g.rows = i64_dist(1, std::max<int64_t>(1, g.domain[0] / 2))(rng);
			break;
		case 1:
			g.kind = "tile";
			for(auto e : g.domain) g.extents.push_back(i64_dist(1, std::max<int64_t>(1, e / 2))(rng));
			break;
		case 2:
			g.kind = "stencil";
			for(auto e : g.domain) {
				g.extents.push_back(i64_dist(2, std::max<int64_t>(2, e / 2))(rng));
				g.halo.push_back(i64_dist(0, 2)(rng));
			}
			break;
		case 3: g.kind = "replicated"; break;
		case 4: g.kind = "single"; break;
		default:
			g.kind = "col";
			g.cols = i64_dist(1, std::max<int64_t>(1, g.domain[1] / 2))(rng);
			break;
		}
		arrays.push_back(std::move(g));
	}

	auto binding = [&](int rank) {
		std::string b = "global ";
		if(rank == 1) return b + "i";
		b += "[i";
		for(int k = 1; k < rank; ++k) b += ", " + var_name(k);
		return b + "]";
	};
	auto identity = [&](int rank) {
		std::string s = "i";
		for(int k = 1; k < rank; ++k) s += "," + var_name(k);
		return s;
	};

	std::vector<launch_gen> launches;
	const int launch_count = std::uniform_int_distribution<int>(2, 4)(rng);
	int previous_dst = 0;
	for(int l = 0; l < launch_count; ++l) {
		const int dst = l == 0 ? 0 : std::uniform_int_distribution<int>(0, array_count - 1)(rng);
		const array_gen& d = arrays[static_cast<size_t>(dst)];
		const int rank = static_cast<int>(d.domain.size());
		launch_gen L;
		L.grid = d.domain;
		for(int k = 0; k < rank; ++k) {
			const int64_t bs = i64_dist(1, 6)(rng);
			L.block.push_back(bs);
			L.superblock.push_back(bs * i64_dist(1, 4)(rng));
		}
		std::string ann = binding(rank) + " => ";
		if(l > 0) {
			std::vector<int> sources{previous_dst};
			const int extra = std::uniform_int_distribution<int>(0, array_count - 1)(rng);
			if(extra != previous_dst) sources.push_back(extra);
			bool first = true;
			for(int src : sources) {
				if(src == dst) continue;
				const array_gen& s = arrays[static_cast<size_t>(src)];
				if(!first) ann += ", ";
				first = false;
				ann += "read " + s.name + "[";
				for(size_t k = 0; k < s.domain.size(); ++k) ann += (k ? "," : "") + random_index(rng, rank);
				ann += "]";
				L.args.push_back(s.name);
			}
			if(!first) ann += ", ";
		}
		const bool reduce = l > 0 && std::uniform_int_distribution<int>(0, 3)(rng) == 0;
		if(reduce) {
			static const char* ops[] = {"+", "min", "max"};
			ann += std::string("reduce(") + ops[std::uniform_int_distribution<int>(0, 2)(rng)] + ") " + d.name + "[";
			for(int k = 0; k < rank; ++k) {
				std::uniform_int_distribution<int> coeff(0, 2);
				const int c = coeff(rng);
				const int v = std::uniform_int_distribution<int>(0, rank - 1)(rng);
				ann += (k ? "," : "") + std::to_string(c) + "*" + var_name(v);
			}
			ann += "]";
		} else {
			ann += "write " + d.name + "[" + identity(rank) + "]";
		}
		L.args.push_back(d.name);
		L.annotation = ann;
		launches.push_back(std::move(L));
		previous_dst = dst;
	}

	if(std::uniform_int_distribution<int>(0, 1)(rng) == 0) {
		uint64_t worst_fan_in = 1;
		for(const auto& l : launches) {
			uint64_t superblocks = 1;
			for(size_t k = 0; k < l.grid.size(); ++k) {
				const int64_t blocks = (l.grid[k] + l.block[k] - 1) / l.block[k];
				const int64_t per_sb = l.superblock[k] / l.block[k];
				superblocks *= static_cast<uint64_t>((blocks + per_sb - 1) / per_sb);
			}
			worst_fan_in = std::max(worst_fan_in, superblocks);
		}
		const uint64_t floor = 2 * (worst_fan_in + 8) * 4096;
		device_capacity = std::max(floor, total_bytes / 2);
		host_capacity = device_capacity * 4;
	}

	std::ostringstream os;
	os << "{\"system\": {\"workers\": " << workers << ", \"devices\": " << devices << ", \"device_capacity\": " << device_capacity
	   << ", \"host_capacity\": " << host_capacity << ", \"disk_capacity\": " << (4ull << 30) << ", \"staging_threshold\": " << (64ull << 20)
	   << "},\n \"arrays\": [";
	for(size_t a = 0; a < arrays.size(); ++a) {
		const auto& g = arrays[a];
		os << (a ? ",\n  " : "\n  ") << "{\"name\": " << quoted(g.name) << ", \"domain\": " << ints(g.domain) << ", \"type\": \"i64\", \"distribution\": {\"kind\": "
		   << quoted(g.kind);
		if(g.kind == "row") os << ", \"rows\": " << g.rows;
		if(g.kind == "col") os << ", \"cols\": " << g.cols;
		if(g.kind == "tile" || g.kind == "stencil") os << ", \"extents\": " << ints(g.extents);
		if(g.kind == "stencil") os << ", \"halo\": " << ints(g.halo);
		os << "}, \"fill\": 1.0}";
	}
	os << "],\n \"launches\": [";
	for(size_t i = 0; i < launches.size(); ++i) {
		const auto& L = launches[i];
		os << (i ? ",\n  " : "\n  ") << "{\"kernel\": \"gather\", \"grid\": " << ints(L.grid) << ", \"block\": " << ints(L.block)
		   << ", \"superblock\": " << ints(L.superblock) << ", \"annotation\": " << quoted(L.annotation) << ", \"args\": [";
		for(size_t k = 0; k < L.args.size(); ++k) os << (k ? ", " : "") << quoted(L.args[k]);
		os << "], \"repeat\": 1}";
	}
	os << "],\n \"seed\": " << seed << "}\n";
	return os.str();
}

} // namespace

extern "C" int mt_fuzz_scenario_json(uint64_t seed, char* buf, int64_t cap, int64_t* len) {
	try {
		const std::string s = make_fuzz_scenario_json(seed);
		*len = static_cast<int64_t>(s.size());
		if(buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
		return MT_OK;
	} catch(...) {
		return MT_EINTERNAL;
	}
}
