// ORACLE / TEST INFRASTRUCTURE — not part of the product.
//
// C-ABI shim over the UNMODIFIED reference implementation (/root/reference/proj, compiled
// from its own sources by oracle/Makefile into oracle/_ref/libmanta_ref.so). It exports
// the entry points of include/manta_b200.h with the prefix `mr_` so the parity tests can
// drive the reference planner (manta::driver, planner.hpp:51-78) and the reference CPU
// executor (manta::system_runtime, runtime.hpp:70-98) through the same binding as the
// B200 product, and bench.py can time the reference CPU executor as its baseline.
//
// Kernels the reference lacks (heat2d, histogram, int32 k-means, the f32/i32 pattern
// generators) are restated here through the reference's own plugin API
// (kernel_registry::register_kernel, kernels.hpp:99), following the conventions of the
// builtins they extend: stencil1d (kernels.cpp:147-165) for zero padding and guards,
// kmeans_* (kernels.cpp:267-346) and row_reduce (kernels.cpp:195-215) for reduce partials,
// ramp2d / ipattern2d (kernels.cpp:439-496) for deterministic inputs, mix64
// (kernels.cpp:103-110) for hashed inputs. The test-only kernels of
// tests/unit/test_runtime.cpp:130-142 and :167-178 are registered too.

#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "manta/planner.hpp"
#include "manta/runtime.hpp"
#include "manta/scenario.hpp"

#include "../include/manta_b200.h"

using namespace manta;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
	g_last_error = msg;
	return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
	try {
		fn();
		return MT_OK;
	} catch(const parse_error& e) {
		return fail(MT_EPARSE, e.what());
	} catch(const validation_error& e) {
		return fail(MT_EVALIDATION, e.what());
	} catch(const plan_error& e) {
		return fail(MT_EPLAN, e.what());
	} catch(const execution_error& e) {
		return fail(MT_EEXEC, e.what());
	} catch(const std::exception& e) {
		return fail(MT_EINTERNAL, e.what());
	}
}

// ---- conversions ---------------------------------------------------------------------

point to_point(int rank, const int64_t* v) {
	point p = point::zeros(rank);
	for(int k = 0; k < rank; ++k) p[k] = v[k];
	return p;
}

rect to_rect(const mt_rect& r) { return rect(to_point(r.rank, r.lo), to_point(r.rank, r.hi)); }

mt_rect from_rect(const rect& r) {
	mt_rect o{};
	o.rank = r.rank();
	for(int k = 0; k < r.rank(); ++k) {
		o.lo[k] = r.lo[k];
		o.hi[k] = r.hi[k];
	}
	return o;
}

mt_rect from_point(const point& p) {
	mt_rect o{};
	o.rank = p.rank;
	for(int k = 0; k < p.rank; ++k) o.lo[k] = p[k];
	return o;
}

dtype to_dtype(int32_t t) {
	switch(t) {
	case MT_I32: return dtype::i32;
	case MT_I64: return dtype::i64;
	case MT_F32: return dtype::f32;
	case MT_F64: return dtype::f64;
	}
	throw validation_error("the reference has no element type " + std::to_string(t));
}

int32_t from_dtype(dtype t) {
	switch(t) {
	case dtype::i32: return MT_I32;
	case dtype::i64: return MT_I64;
	case dtype::f32: return MT_F32;
	case dtype::f64: return MT_F64;
	}
	return -1;
}

reduce_op to_op(int32_t op) { return static_cast<reduce_op>(op); }

fill_spec to_fill(int32_t kind, int32_t op) {
	switch(kind) {
	case MT_FILL_NONE: return fill_spec::none();
	case MT_FILL_ZERO: return fill_spec::zero();
	case MT_FILL_ONE: return fill_spec::one();
	case MT_FILL_IDENTITY: return fill_spec::identity_of(to_op(op));
	}
	throw validation_error("bad fill kind");
}

device_id to_dev(mt_device d) { return device_id{d.worker, d.device}; }
mt_device from_dev(device_id d) { return mt_device{d.worker, d.device}; }

data_distribution to_dist(const mt_chunk_desc* chunks, int64_t n) {
	data_distribution dist;
	for(int64_t i = 0; i < n; ++i) dist.chunks.push_back({chunks[i].id, to_rect(chunks[i].region), to_dev(chunks[i].home)});
	return dist;
}

int emit_chunks(const data_distribution& d, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	const auto n = static_cast<int64_t>(d.chunks.size());
	for(int64_t i = 0; i < n && i < cap; ++i) {
		out[i].id = d.chunks[static_cast<size_t>(i)].id;
		out[i].region = from_rect(d.chunks[static_cast<size_t>(i)].region);
		out[i].home = from_dev(d.chunks[static_cast<size_t>(i)].home);
	}
	*n_out = n;
	return MT_OK;
}

std::vector<device_id> to_devs(const mt_device* d, int32_t n) {
	std::vector<device_id> v;
	for(int32_t i = 0; i < n; ++i) v.push_back(to_dev(d[i]));
	return v;
}

// task -> flat record
void flatten(const task& t, mt_task& o, std::vector<int64_t>& pool, std::vector<mt_arg_binding>& args) {
	std::memset(&o, 0, sizeof(o));
	o.id = t.id;
	o.worker = t.worker;
	o.kind = static_cast<int32_t>(t.op.index());
	o.resource = from_dev(t.resource);
	o.deps_off = static_cast<int64_t>(pool.size());
	o.ndeps = static_cast<int64_t>(t.deps.size());
	for(auto d : t.deps) pool.push_back(d);
	o.chunk = -1;
	o.src = o.dst = o.output = -1;
	if(const auto* c = std::get_if<create_task>(&t.op)) {
		o.chunk = c->chunk.id;
		o.region = from_rect(c->chunk.region);
		o.home = from_dev(c->chunk.home);
		o.dtype = from_dtype(c->type);
		o.fill = static_cast<int32_t>(c->fill.kind);
		o.fill_op = static_cast<int32_t>(c->fill.op);
	} else if(const auto* d = std::get_if<delete_task>(&t.op)) {
		o.chunk = d->chunk;
	} else if(const auto* e = std::get_if<execute_task>(&t.op)) {
		std::strncpy(o.kernel, e->kernel.c_str(), MT_KERNEL_NAME_MAX - 1);
		o.device = from_dev(e->device);
		o.sb_blocks = from_rect(e->superblock_blocks);
		o.sb_threads = from_rect(e->superblock_threads);
		o.block_size = from_point(e->block_size);
		o.args_off = static_cast<int64_t>(args.size());
		o.nargs = static_cast<int64_t>(e->args.size());
		for(const auto& b : e->args) {
			mt_arg_binding a{};
			a.kind = static_cast<int32_t>(b.kind);
			a.i = b.scalar_int;
			a.f = b.scalar_float;
			a.chunk = b.chunk;
			args.push_back(a);
		}
	} else if(const auto* c = std::get_if<copy_task>(&t.op)) {
		o.src = c->src;
		o.dst = c->dst;
		o.src_region = from_rect(c->src_region);
		o.dst_region = from_rect(c->dst_region);
	} else if(const auto* s = std::get_if<send_task>(&t.op)) {
		o.chunk = s->chunk;
		o.region = from_rect(s->region);
		o.peer = s->peer_worker;
		o.tag = s->tag;
	} else if(const auto* r = std::get_if<recv_task>(&t.op)) {
		o.chunk = r->chunk;
		o.region = from_rect(r->region);
		o.peer = r->peer_worker;
		o.tag = r->tag;
	} else if(const auto* r = std::get_if<reduce_task>(&t.op)) {
		o.op = static_cast<int32_t>(r->op);
		o.inputs_off = static_cast<int64_t>(pool.size());
		o.ninputs = static_cast<int64_t>(r->inputs.size());
		for(auto c : r->inputs) pool.push_back(c);
		o.output = r->output;
	}
}

// flat record -> task
task unflatten(const mt_task& o, const int64_t* pool, const mt_arg_binding* args) {
	task t;
	t.id = o.id;
	t.worker = o.worker;
	t.resource = to_dev(o.resource);
	for(int64_t i = 0; i < o.ndeps; ++i) t.deps.push_back(pool[o.deps_off + i]);
	switch(o.kind) {
	case MT_TASK_CREATE:
		t.op = create_task{chunk_descriptor{o.chunk, to_rect(o.region), to_dev(o.home)}, to_dtype(o.dtype), to_fill(o.fill, o.fill_op)};
		break;
	case MT_TASK_DELETE: t.op = delete_task{o.chunk}; break;
	case MT_TASK_EXECUTE: {
		execute_task e;
		e.kernel = o.kernel;
		e.device = to_dev(o.device);
		e.superblock_blocks = to_rect(o.sb_blocks);
		e.superblock_threads = to_rect(o.sb_threads);
		e.block_size = to_point(o.block_size.rank, o.block_size.lo);
		for(int64_t i = 0; i < o.nargs; ++i) {
			const auto& a = args[o.args_off + i];
			arg_binding b;
			b.kind = static_cast<arg_binding::kind_t>(a.kind);
			b.scalar_int = a.i;
			b.scalar_float = a.f;
			b.chunk = a.chunk;
			e.args.push_back(b);
		}
		t.op = std::move(e);
		break;
	}
	case MT_TASK_COPY: t.op = copy_task{o.src, o.dst, to_rect(o.src_region), to_rect(o.dst_region)}; break;
	case MT_TASK_SEND: t.op = send_task{o.chunk, to_rect(o.region), o.peer, o.tag}; break;
	case MT_TASK_RECV: t.op = recv_task{o.chunk, to_rect(o.region), o.peer, o.tag}; break;
	case MT_TASK_REDUCE: {
		reduce_task r;
		r.op = to_op(o.op);
		for(int64_t i = 0; i < o.ninputs; ++i) r.inputs.push_back(pool[o.inputs_off + i]);
		r.output = o.output;
		t.op = std::move(r);
		break;
	}
	default: throw validation_error("bad task kind");
	}
	return t;
}

// ---- kernels restated through the reference plugin API -------------------------------

std::uint64_t mix64(std::uint64_t h) {
	h ^= h >> 33;
	h *= 0xff51afd7ed558ccdULL;
	h ^= h >> 33;
	h *= 0xc4ceb9fe1a85ec53ULL;
	h ^= h >> 33;
	return h;
}

// 2D 5-point heat step, f32 arithmetic in a fixed order (no contraction; the Makefile
// passes -ffp-contract=off), zero padding outside [0,rows)x[0,cols) like stencil1d.
kernel_def make_heat2d() {
	kernel_def def;
	def.id = "heat2d";
	def.params = {param_spec::scalar("rows", dtype::i64), param_spec::scalar("cols", dtype::i64), param_spec::scalar("alpha", dtype::f64),
	    param_spec::array("out", dtype::f32, 2, true), param_spec::array("in", dtype::f32, 2, false)};
	def.body = [](const kernel_context& ctx) {
		const auto rows = ctx.scalar_int(0);
		const auto cols = ctx.scalar_int(1);
		const float a = static_cast<float>(ctx.scalar_float(2));
		const auto& out = ctx.view(3);
		const auto& in = ctx.view(4);
		ctx.for_each_thread([&](const point& g) {
			const std::int64_t i = g[0], j = g[1];
			if(i >= rows || j >= cols) return;
			const float c = in.at<float>({i, j});
			const float up = i > 0 ? in.at<float>({i - 1, j}) : 0.0f;
			const float dn = i + 1 < rows ? in.at<float>({i + 1, j}) : 0.0f;
			const float lf = j > 0 ? in.at<float>({i, j - 1}) : 0.0f;
			const float rt = j + 1 < cols ? in.at<float>({i, j + 1}) : 0.0f;
			const float s = ((up + dn) + (lf + rt)) - 4.0f * c;
			out.at<float>({i, j}) = c + a * s;
		});
	};
	return def;
}

// f32 form of ramp2d (kernels.cpp:475-496): value computed in f64, rounded once to f32
kernel_def make_ramp2d_f32() {
	kernel_def def;
	def.id = "ramp2d_f32";
	def.params = {param_spec::scalar("rows", dtype::i64), param_spec::scalar("cols", dtype::i64), param_spec::scalar("mod", dtype::i64),
	    param_spec::scalar("base", dtype::f64), param_spec::scalar("scale", dtype::f64), param_spec::array("out", dtype::f32, 2, true)};
	def.body = [](const kernel_context& ctx) {
		const auto rows = ctx.scalar_int(0);
		const auto cols = ctx.scalar_int(1);
		const auto mod = ctx.scalar_int(2);
		const double base = ctx.scalar_float(3);
		const double scale = ctx.scalar_float(4);
		const auto& out = ctx.view(5);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= rows || g[1] >= cols) return;
			const double v = base + scale * static_cast<double>((g[0] * 31 + g[1] * 17 + 7) % mod) / static_cast<double>(mod);
			out.at<float>(g) = static_cast<float>(v);
		});
	};
	return def;
}

// hashed bin indices for the histogram: x[i] = mix64(i ^ seed) mod bins, as i32
kernel_def make_hpattern1d() {
	kernel_def def;
	def.id = "hpattern1d";
	def.params = {param_spec::scalar("n", dtype::i64), param_spec::scalar("bins", dtype::i64), param_spec::scalar("seed", dtype::i64),
	    param_spec::array("out", dtype::i32, 1, true)};
	def.body = [](const kernel_context& ctx) {
		const auto n = ctx.scalar_int(0);
		const auto bins = static_cast<std::uint64_t>(ctx.scalar_int(1));
		const auto seed = static_cast<std::uint64_t>(ctx.scalar_int(2));
		const auto& out = ctx.view(3);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= n) return;
			out.at<std::int32_t>(g) = static_cast<std::int32_t>(mix64(static_cast<std::uint64_t>(g[0]) ^ seed) % bins);
		});
	};
	return def;
}

// histogram into a reduce(+) partial (the row_reduce / kmeans_update convention):
// out-of-range values are ignored, counts wrap like every integer reduce
kernel_def make_histogram() {
	kernel_def def;
	def.id = "histogram";
	def.params = {param_spec::scalar("n", dtype::i64), param_spec::scalar("bins", dtype::i64), param_spec::array("x", dtype::i32, 1, false),
	    param_spec::array("hist", dtype::i64, 1, true)};
	def.body = [](const kernel_context& ctx) {
		const auto n = ctx.scalar_int(0);
		const auto bins = ctx.scalar_int(1);
		const auto& x = ctx.view(2);
		const auto& hist = ctx.view(3);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= n) return;
			const std::int64_t b = x.at<std::int32_t>(g);
			if(b < 0 || b >= bins) return;
			auto& cell = hist.at<std::int64_t>({b});
			cell = static_cast<std::int64_t>(static_cast<std::uint64_t>(cell) + 1u);
		});
	};
	return def;
}

kernel_def make_ipattern2d_i32() {
	kernel_def def;
	def.id = "ipattern2d_i32";
	def.params = {param_spec::scalar("rows", dtype::i64), param_spec::scalar("cols", dtype::i64), param_spec::scalar("mod", dtype::i64),
	    param_spec::array("out", dtype::i32, 2, true)};
	def.body = [](const kernel_context& ctx) {
		const auto rows = ctx.scalar_int(0);
		const auto cols = ctx.scalar_int(1);
		const auto mod = ctx.scalar_int(2);
		const auto& out = ctx.view(3);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= rows || g[1] >= cols) return;
			out.at<std::int32_t>(g) = static_cast<std::int32_t>((g[0] * 31 + g[1] * 17 + 7) % mod);
		});
	};
	return def;
}

// k-means over i32 points (the BASELINE C4 layout); distances in i64, ties -> lowest c
kernel_def make_kmeans_assign_i32() {
	kernel_def def;
	def.id = "kmeans_assign_i32";
	def.params = {param_spec::scalar("n", dtype::i64), param_spec::scalar("k", dtype::i64), param_spec::scalar("d", dtype::i64),
	    param_spec::array("assign", dtype::i32, 1, true), param_spec::array("points", dtype::i32, 2, false),
	    param_spec::array("centroids", dtype::i32, 2, false)};
	def.body = [](const kernel_context& ctx) {
		const auto n = ctx.scalar_int(0);
		const auto k = ctx.scalar_int(1);
		const auto d = ctx.scalar_int(2);
		const auto& assign = ctx.view(3);
		const auto& points = ctx.view(4);
		const auto& centroids = ctx.view(5);
		ctx.for_each_thread([&](const point& g) {
			const std::int64_t i = g[0];
			if(i >= n) return;
			std::int64_t best = 0;
			std::int64_t best_dist = std::numeric_limits<std::int64_t>::max();
			for(std::int64_t c = 0; c < k; ++c) {
				std::int64_t dist = 0;
				for(std::int64_t t = 0; t < d; ++t) {
					const std::int64_t diff = static_cast<std::int64_t>(points.at<std::int32_t>({i, t})) - centroids.at<std::int32_t>({c, t});
					dist += diff * diff;
				}
				if(dist < best_dist) {
					best_dist = dist;
					best = c;
				}
			}
			assign.at<std::int32_t>({i}) = static_cast<std::int32_t>(best);
		});
	};
	return def;
}

kernel_def make_kmeans_update_i32() {
	kernel_def def;
	def.id = "kmeans_update_i32";
	def.params = {param_spec::scalar("n", dtype::i64), param_spec::scalar("d", dtype::i64), param_spec::array("points", dtype::i32, 2, false),
	    param_spec::array("assign", dtype::i32, 1, false), param_spec::array("sums", dtype::i64, 2, true), param_spec::array("counts", dtype::i64, 1, true)};
	def.body = [](const kernel_context& ctx) {
		const auto n = ctx.scalar_int(0);
		const auto d = ctx.scalar_int(1);
		const auto& points = ctx.view(2);
		const auto& assign = ctx.view(3);
		const auto& sums = ctx.view(4);
		const auto& counts = ctx.view(5);
		ctx.for_each_thread([&](const point& g) {
			const std::int64_t i = g[0];
			if(i >= n) return;
			const std::int64_t c = assign.at<std::int32_t>({i});
			for(std::int64_t t = 0; t < d; ++t) {
				auto& s = sums.at<std::int64_t>({c, t});
				s = static_cast<std::int64_t>(static_cast<std::uint64_t>(s) + static_cast<std::uint64_t>(static_cast<std::int64_t>(points.at<std::int32_t>({i, t}))));
			}
			auto& cnt = counts.at<std::int64_t>({c});
			cnt = static_cast<std::int64_t>(static_cast<std::uint64_t>(cnt) + 1u);
		});
	};
	return def;
}

kernel_def make_kmeans_finalize_i32() {
	kernel_def def;
	def.id = "kmeans_finalize_i32";
	def.params = {param_spec::scalar("k", dtype::i64), param_spec::scalar("d", dtype::i64), param_spec::array("centroids", dtype::i32, 2, true),
	    param_spec::array("sums", dtype::i64, 2, false), param_spec::array("counts", dtype::i64, 1, false)};
	def.body = [](const kernel_context& ctx) {
		const auto k = ctx.scalar_int(0);
		const auto d = ctx.scalar_int(1);
		const auto& centroids = ctx.view(2);
		const auto& sums = ctx.view(3);
		const auto& counts = ctx.view(4);
		ctx.for_each_thread([&](const point& g) {
			const std::int64_t c = g[0], t = g[1];
			if(c >= k || t >= d) return;
			const std::int64_t count = counts.at<std::int64_t>({c});
			if(count > 0) centroids.at<std::int32_t>({c, t}) = static_cast<std::int32_t>(sums.at<std::int64_t>({c, t}) / count);
		});
	};
	return def;
}

// tests/unit/test_runtime.cpp:130-142
kernel_def make_row_reduce_i64() {
	kernel_def def;
	def.id = "row_reduce_i64";
	def.params = {param_spec::scalar("rows", dtype::i64), param_spec::scalar("cols", dtype::i64), param_spec::array("A", dtype::i64, 2, false),
	    param_spec::array("sum", dtype::i64, 1, true)};
	def.body = [](const kernel_context& ctx) {
		const auto rows = ctx.scalar_int(0);
		const auto cols = ctx.scalar_int(1);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= rows || g[1] >= cols) return;
			ctx.view(3).at<std::int64_t>({g[0]}) += ctx.view(2).at<std::int64_t>(g);
		});
	};
	return def;
}

// tests/unit/test_runtime.cpp:167-178
kernel_def make_partial_min() {
	kernel_def def;
	def.id = "partial_min";
	def.params = {param_spec::scalar("n", dtype::i64), param_spec::array("src", dtype::i64, 1, false), param_spec::array("dst", dtype::i64, 1, true)};
	def.body = [](const kernel_context& ctx) {
		const auto n = ctx.scalar_int(0);
		ctx.for_each_thread([&](const point& g) {
			if(g[0] >= n || g[0] >= 4) return;
			auto& cell = ctx.view(2).at<std::int64_t>(g);
			cell = std::min(cell, ctx.view(1).at<std::int64_t>(g) + g[0]);
		});
	};
	return def;
}

kernel_registry make_registry() {
	kernel_registry reg = kernel_registry::with_builtins();
	reg.register_kernel(make_heat2d());
	reg.register_kernel(make_ramp2d_f32());
	reg.register_kernel(make_hpattern1d());
	reg.register_kernel(make_histogram());
	reg.register_kernel(make_ipattern2d_i32());
	reg.register_kernel(make_kmeans_assign_i32());
	reg.register_kernel(make_kmeans_update_i32());
	reg.register_kernel(make_kmeans_finalize_i32());
	reg.register_kernel(make_row_reduce_i64());
	reg.register_kernel(make_partial_min());
	return reg;
}

const kernel_registry& registry() {
	static const kernel_registry reg = make_registry();
	return reg;
}

// array_view bounds checking in the reference executor (memory.hpp:54, default on); the bench
// times the CPU baseline both ways
bool g_bounds_check = true;

system_config make_system_config(const mt_config& c) {
	system_config sys;
	sys.memory.bounds_check = g_bounds_check;
	sys.workers = c.workers;
	sys.devices_per_worker = c.devices_per_worker;
	if(c.device_capacity) sys.memory.device_capacity = c.device_capacity;
	if(c.host_capacity) sys.memory.host_capacity = c.host_capacity;
	if(c.staging_threshold) sys.memory.staging_threshold = c.staging_threshold;
	if(c.disk_capacity) sys.memory.disk_capacity = c.disk_capacity;
	sys.memory.disk_in_memory = true;
	if(c.schedule_seed) sys.ready_seed = c.schedule_seed;
	sys.progress_timeout = std::chrono::milliseconds(600000);
	return sys;
}

} // namespace

struct mt_exec {
	std::unique_ptr<system_runtime> rt;
};

struct mt_ctx {
	mt_config cfg{};
	std::unique_ptr<driver> drv;
	mt_exec exec;
	bool has_exec = false;
};

namespace {
// the reference's access_annotation (annotation.hpp:15-87) in the canonical text of
// mt_annotation_describe (capi.cpp), for the parser-parity test
void describe_expr(std::string& o, const linear_expr& e) {
	o += "[" + std::to_string(e.constant) + ",[";
	for(size_t t = 0; t < e.terms.size(); ++t) {
		if(t) o += ",";
		o += "[\"" + e.terms[t].first + "\"," + std::to_string(e.terms[t].second) + "]";
	}
	o += "]]";
}

std::string describe(const access_annotation& a) {
	static const char* space[] = {"global", "block", "local"};
	static const char* kind[] = {"read", "write", "readwrite", "reduce"};
	static const char* op[] = {"+", "*", "min", "max"};
	std::string o = "{\"bindings\":[";
	for(size_t b = 0; b < a.bindings.size(); ++b) {
		if(b) o += ",";
		o += "[\"" + std::string(space[static_cast<int>(a.bindings[b].space)]) + "\",[";
		for(size_t v = 0; v < a.bindings[b].variables.size(); ++v) o += std::string(v ? "," : "") + "\"" + a.bindings[b].variables[v] + "\"";
		o += "]]";
	}
	o += "],\"accesses\":[";
	for(size_t i = 0; i < a.accesses.size(); ++i) {
		const auto& acc = a.accesses[i];
		if(i) o += ",";
		o += "[\"" + acc.argument + "\",\"" + kind[static_cast<int>(acc.mode.kind)] + "\",\"" + op[static_cast<int>(acc.mode.op)] + "\",[";
		for(size_t k = 0; k < acc.indices.size(); ++k) {
			const auto& ix = acc.indices[k];
			if(k) o += ",";
			if(ix.kind == index_spec::kind_t::single) {
				o += "[\"single\",";
				describe_expr(o, *ix.single);
				o += "]";
				continue;
			}
			o += "[\"slice\",";
			if(ix.slice_lower) describe_expr(o, *ix.slice_lower);
			else o += "null";
			o += ",";
			if(ix.slice_upper) describe_expr(o, *ix.slice_upper);
			else o += "null";
			o += "]";
		}
		o += "]]";
	}
	return o + "]}";
}
} // namespace

extern "C" {

const char* mr_last_error(void) { return g_last_error.c_str(); }
const char* mr_version(void) { return "manta-reference (proj/, C++20 CPU executor)"; }

int mr_annotation_describe(const char* text, char* out, int64_t cap, int64_t* len) {
	return guarded([&] {
		const std::string s = describe(parse_annotation(text ? text : ""));
		*len = static_cast<int64_t>(s.size());
		if(out && cap > static_cast<int64_t>(s.size())) std::memcpy(out, s.c_str(), s.size() + 1);
	});
}

int mr_dist_tile(const mt_rect* domain, const int64_t* extents, const int64_t* halo, const mt_device* devices, int32_t ndev, int64_t first_id,
    mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] {
		const rect dom = to_rect(*domain);
		const auto d = tile_data_dist(dom, to_point(dom.rank(), extents), to_point(dom.rank(), halo), to_devs(devices, ndev), first_id);
		emit_chunks(d, out, cap, n_out);
	});
}

int mr_dist_replicated(const mt_rect* domain, const mt_device* devices, int32_t ndev, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(replicated_dist(to_rect(*domain), to_devs(devices, ndev), first_id), out, cap, n_out); });
}

int mr_dist_single(const mt_rect* domain, mt_device home, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(single_dist(to_rect(*domain), to_dev(home), first_id), out, cap, n_out); });
}

int mr_work_block(const mt_rect* grid, const int64_t* block, const int64_t* tps, const mt_device* devices, int32_t ndev, mt_superblock* out,
    int64_t cap, int64_t* n_out) {
	return guarded([&] {
		const rect g = to_rect(*grid);
		const auto w = block_work_dist(g, to_point(g.rank(), block), to_point(g.rank(), tps), to_devs(devices, ndev));
		const auto n = static_cast<int64_t>(w.superblocks.size());
		for(int64_t i = 0; i < n && i < cap; ++i) {
			out[i].blocks = from_rect(w.superblocks[static_cast<size_t>(i)].blocks);
			out[i].device = from_dev(w.superblocks[static_cast<size_t>(i)].device);
		}
		*n_out = n;
	});
}

int mr_ctx_create(const mt_config* cfg, mt_ctx** out) {
	return guarded([&] {
		auto ctx = std::make_unique<mt_ctx>();
		ctx->cfg = *cfg;
		driver_config dc;
		dc.workers = cfg->workers;
		dc.devices_per_worker = cfg->devices_per_worker;
		dc.suppress_conflict_deps = cfg->suppress_conflict_deps != 0;
		ctx->drv = std::make_unique<driver>(dc, registry());
		if(cfg->execute) {
			ctx->exec.rt = std::make_unique<system_runtime>(make_system_config(*cfg), registry());
			ctx->has_exec = true;
		}
		*out = ctx.release();
	});
}

int mr_ctx_destroy(mt_ctx* ctx) {
	delete ctx;
	return MT_OK;
}

int mr_ctx_devices(mt_ctx* ctx, mt_device* out, int32_t cap, int32_t* n_out) {
	const auto& d = ctx->drv->devices();
	for(size_t i = 0; i < d.size() && static_cast<int32_t>(i) < cap; ++i) out[i] = from_dev(d[i]);
	*n_out = static_cast<int32_t>(d.size());
	return MT_OK;
}

int mr_array_create(mt_ctx* ctx, const mt_rect* domain, int32_t dt, const mt_chunk_desc* chunks, int64_t nchunks, int32_t fill, int64_t* out_id) {
	return guarded([&] { *out_id = ctx->drv->create_array(to_rect(*domain), to_dtype(dt), to_dist(chunks, nchunks), to_fill(fill, 0)).id; });
}

int mr_array_delete(mt_ctx* ctx, int64_t id) {
	return guarded([&] { ctx->drv->delete_array(id); });
}

int mr_array_chunks(mt_ctx* ctx, int64_t id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(ctx->drv->registry().get(id).distribution, out, cap, n_out); });
}

int mr_launch(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* annotation, int64_t* first, int64_t* last) {
	return guarded([&] {
		const rect g = to_rect(*grid);
		work_distribution w;
		for(int64_t i = 0; i < nwork; ++i) w.superblocks.push_back({to_rect(work[i].blocks), to_dev(work[i].device)});
		std::vector<launch_arg> la;
		for(int32_t i = 0; i < nargs; ++i) {
			switch(args[i].kind) {
			case MT_LARG_INT: la.push_back(launch_arg::scalar(static_cast<std::int64_t>(args[i].i))); break;
			case MT_LARG_FLOAT: la.push_back(launch_arg::scalar(args[i].f)); break;
			default: la.push_back(launch_arg::array(args[i].array)); break;
			}
		}
		const auto ann = parse_annotation(annotation);
		const auto r = ctx->drv->launch(kernel, g, to_point(g.rank(), block), w, la, ann);
		*first = r.first_task;
		*last = r.past_last_task;
	});
}

int mr_flush(mt_ctx* ctx) {
	return guarded([&] {
		auto pending = ctx->drv->take_pending();
		if(ctx->has_exec) ctx->exec.rt->submit(pending);
	});
}

// the repeat / swap loop of apply_scenario (scenario.cpp:407-441) over the reference driver
int mr_launch_repeat(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* annotation, int32_t repeat, int64_t swap_a, int64_t swap_b, int32_t flush_every, int64_t* first,
    int64_t* last) {
	if(repeat < 1) {
		g_last_error = "repeat must be at least 1";
		return MT_EVALIDATION;
	}
	std::vector<mt_launch_arg> a(args, args + nargs);
	int64_t lo = -1, hi = -1;
	for(int32_t rep = 0; rep < repeat; ++rep) {
		int64_t f = 0, l = 0;
		if(const int rc = mr_launch(ctx, kernel, grid, block, work, nwork, a.data(), nargs, annotation, &f, &l)) return rc;
		if(rep == 0) lo = f;
		hi = l;
		if(flush_every > 0 && (rep + 1) % flush_every == 0)
			if(const int rc = mr_flush(ctx)) return rc;
		for(auto& x : a) {
			if(x.kind != MT_LARG_ARRAY) continue;
			if(x.array == swap_a)
				x.array = swap_b;
			else if(x.array == swap_b)
				x.array = swap_a;
		}
	}
	if(flush_every == 0)
		if(const int rc = mr_flush(ctx)) return rc;
	*first = lo;
	*last = hi;
	return MT_OK;
}

int mr_sync(mt_ctx* ctx) {
	return guarded([&] {
		auto pending = ctx->drv->take_pending();
		if(!ctx->has_exec) return;
		ctx->exec.rt->submit(pending);
		ctx->exec.rt->synchronize();
	});
}

int mr_array_read(mt_ctx* ctx, int64_t id, void* host, uint64_t bytes) {
	return guarded([&] {
		if(!ctx->has_exec) throw validation_error("context does not execute");
		ctx->exec.rt->submit(ctx->drv->take_pending());
		ctx->exec.rt->synchronize();
		const auto& h = ctx->drv->registry().get(id);
		const uint64_t need = static_cast<uint64_t>(h.domain.volume()) * dtype_size(h.type);
		if(bytes < need) throw validation_error("host buffer too small");
		auto full = array_view::over_region(static_cast<std::byte*>(host), h.type, h.domain, false);
		for(const auto& c : h.distribution.chunks) {
			auto cb = ctx->exec.rt->read_chunk(c.id);
			copy_region(array_view::over_region(cb.data(), h.type, c.region, false), full, c.region);
		}
	});
}

int mr_array_write(mt_ctx*, int64_t, const void*, uint64_t) { return fail(MT_EVALIDATION, "the reference runtime has no host upload path"); }

int mr_array_check_replicas(mt_ctx* ctx, int64_t id, int32_t* coherent) {
	return guarded([&] {
		if(!ctx->has_exec) throw validation_error("context does not execute");
		ctx->exec.rt->submit(ctx->drv->take_pending());
		ctx->exec.rt->synchronize();
		const auto& h = ctx->drv->registry().get(id);
		const auto& chunks = h.distribution.chunks;
		*coherent = 1;
		for(size_t i = 0; i < chunks.size(); ++i) {
			for(size_t j = i + 1; j < chunks.size(); ++j) {
				const rect ov = intersect(chunks[i].region, chunks[j].region);
				if(ov.is_empty()) continue;
				auto bi = ctx->exec.rt->read_chunk(chunks[i].id);
				auto bj = ctx->exec.rt->read_chunk(chunks[j].id);
				if(pack_region(array_view::over_region(bi.data(), h.type, chunks[i].region, false), ov)
				    != pack_region(array_view::over_region(bj.data(), h.type, chunks[j].region, false), ov)) {
					*coherent = 0;
					return;
				}
			}
		}
	});
}

int mr_plan_export(mt_ctx* ctx, int64_t first, int64_t last, mt_task* tasks, int64_t task_cap, int64_t* ntasks, int64_t* pool, int64_t pool_cap,
    int64_t* npool, mt_arg_binding* args, int64_t args_cap, int64_t* nargs) {
	return guarded([&] {
		std::vector<mt_task> ts;
		std::vector<int64_t> p;
		std::vector<mt_arg_binding> a;
		for(const auto* t : ctx->drv->plan().in_id_order()) {
			if(t->id < first || t->id >= last) continue;
			mt_task o;
			flatten(*t, o, p, a);
			ts.push_back(o);
		}
		*ntasks = static_cast<int64_t>(ts.size());
		*npool = static_cast<int64_t>(p.size());
		*nargs = static_cast<int64_t>(a.size());
		if(task_cap >= *ntasks && tasks) std::memcpy(tasks, ts.data(), ts.size() * sizeof(mt_task));
		if(pool_cap >= *npool && pool) std::memcpy(pool, p.data(), p.size() * sizeof(int64_t));
		if(args_cap >= *nargs && args) std::memcpy(args, a.data(), a.size() * sizeof(mt_arg_binding));
	});
}

int64_t mr_plan_size(mt_ctx* ctx) { return static_cast<int64_t>(ctx->drv->plan().task_count()); }

int mr_chunk_meta(mt_ctx* ctx, int64_t chunk, mt_chunk_desc* desc, int32_t* dt, int32_t* temp) {
	return guarded([&] {
		const auto& m = ctx->drv->chunk(chunk);
		desc->id = m.descriptor.id;
		desc->region = from_rect(m.descriptor.region);
		desc->home = from_dev(m.descriptor.home);
		*dt = from_dtype(m.type);
		*temp = m.temp ? 1 : 0;
	});
}

mt_exec* mr_ctx_exec(mt_ctx* ctx) { return ctx->has_exec ? &ctx->exec : nullptr; }

int mr_exec_create(const mt_config* cfg, mt_exec** out) {
	return guarded([&] {
		auto ex = std::make_unique<mt_exec>();
		ex->rt = std::make_unique<system_runtime>(make_system_config(*cfg), registry());
		*out = ex.release();
	});
}

int mr_exec_destroy(mt_exec* ex) {
	delete ex;
	return MT_OK;
}

int mr_exec_submit(mt_exec* ex, const mt_task* tasks, int64_t n, const int64_t* pool, const mt_arg_binding* args) {
	return guarded([&] {
		std::vector<task> ts;
		for(int64_t i = 0; i < n; ++i) ts.push_back(unflatten(tasks[i], pool, args));
		ex->rt->submit(ts);
	});
}

int mr_exec_sync(mt_exec* ex) {
	return guarded([&] { ex->rt->synchronize(); });
}

int mr_exec_read_chunk(mt_exec* ex, int64_t chunk, void* dst, uint64_t bytes) {
	return guarded([&] {
		auto b = ex->rt->read_chunk(chunk);
		if(bytes < b.size()) throw validation_error("host buffer too small");
		std::memcpy(dst, b.data(), b.size());
	});
}

int mr_exec_write_chunk(mt_exec*, int64_t, const void*, uint64_t) { return fail(MT_EVALIDATION, "the reference runtime has no host upload path"); }

int mr_exec_report_json(mt_exec* ex, char* buf, int64_t cap, int64_t* len) {
	return guarded([&] {
		const auto s = ex->rt->report().to_json();
		*len = static_cast<int64_t>(s.size());
		if(buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
	});
}

int mr_kernel_register(const char*, const mt_param_spec*, int32_t, mt_launcher_fn) {
	return fail(MT_EVALIDATION, "the reference shim registers its CPU kernels at build time");
}

int mr_kernel_count(void) {
	return 0;
}

// Hardware threads the reference executor can use on this host (bench cpu_baseline).
int mr_host_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }
void mr_set_bounds_check(int32_t on) { g_bounds_check = on != 0; }

// ---- scenario harness of the reference (scenario.hpp:160-171), used as the parity oracle ----

// make_fuzz_scenario (scenario.cpp:653-812) rendered as scenario JSON
int mr_fuzz_scenario_json(uint64_t seed, char* buf, int64_t cap, int64_t* len) {
	return guarded([&] {
		const std::string s = scenario_to_json_text(make_fuzz_scenario(seed));
		*len = static_cast<int64_t>(s.size());
		if(buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
	});
}

namespace {
run_overrides make_overrides(int32_t workers, int32_t devices, int32_t oracle_mode, int32_t suppress) {
	run_overrides ov;
	if(workers > 0) ov.workers = workers;
	if(devices > 0) ov.devices = devices;
	ov.oracle_mode = oracle_mode != 0;
	ov.suppress_conflict_deps = suppress != 0;
	ov.disk_in_memory = true;
	return ov;
}
} // namespace

// plan_scenario (scenario.cpp:455-463) + plan export
int mr_scenario_plan(const char* json, int32_t workers, int32_t devices, int32_t oracle_mode, int32_t suppress, mt_task* tasks, int64_t task_cap,
    int64_t* ntasks, int64_t* pool, int64_t pool_cap, int64_t* npool, mt_arg_binding* args, int64_t args_cap, int64_t* nargs) {
	return guarded([&] {
		const auto sp = plan_scenario(scenario_from_json_text(json), make_overrides(workers, devices, oracle_mode, suppress));
		std::vector<mt_task> ts;
		std::vector<int64_t> p;
		std::vector<mt_arg_binding> a;
		for(const auto* t : sp.drv->plan().in_id_order()) {
			mt_task o;
			flatten(*t, o, p, a);
			ts.push_back(o);
		}
		*ntasks = static_cast<int64_t>(ts.size());
		*npool = static_cast<int64_t>(p.size());
		*nargs = static_cast<int64_t>(a.size());
		if(task_cap >= *ntasks && tasks) std::memcpy(tasks, ts.data(), ts.size() * sizeof(mt_task));
		if(pool_cap >= *npool && pool) std::memcpy(pool, p.data(), p.size() * sizeof(int64_t));
		if(args_cap >= *nargs && args) std::memcpy(args, a.data(), a.size() * sizeof(mt_arg_binding));
	});
}

// export_dot (task.cpp:72-110) of the scenario's plan, to pin the product CLI's --dot output
int mr_scenario_dot(const char* json, int32_t workers, int32_t devices, char* buf, int64_t cap, int64_t* len) {
	return guarded([&] {
		const auto sp = plan_scenario(scenario_from_json_text(json), make_overrides(workers, devices, 0, 0));
		const std::string s = export_dot(sp.drv->plan());
		*len = static_cast<int64_t>(s.size());
		if(buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
	});
}

// run_scenario (scenario.cpp:513-552): final arrays concatenated in scenario order
int mr_scenario_run(const char* json, int32_t workers, int32_t devices, int32_t oracle_mode, int64_t ready_seed, int32_t use_seed, void* out,
    int64_t cap, int64_t* len, int32_t* coherent) {
	return guarded([&] {
		auto ov = make_overrides(workers, devices, oracle_mode, 0);
		if(use_seed) ov.ready_seed = static_cast<uint64_t>(ready_seed);
		const auto r = run_scenario(scenario_from_json_text(json), ov);
		int64_t total = 0;
		for(const auto& a : r.arrays) total += static_cast<int64_t>(a.bytes.size());
		*len = total;
		*coherent = r.replicas_coherent ? 1 : 0;
		if(!out || cap < total) return;
		auto* p = static_cast<char*>(out);
		for(const auto& a : r.arrays) {
			std::memcpy(p, a.bytes.data(), a.bytes.size());
			p += a.bytes.size();
		}
	});
}

} // extern "C"
