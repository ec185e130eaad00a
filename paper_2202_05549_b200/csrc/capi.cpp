// extern "C" boundary: include/manta_b200.h implemented over the C++ planner and the GPU
// executor. Every entry point converts exceptions into MT_E* codes (errors.hpp:9-35 kinds)
// and keeps the message in a thread-local buffer for mt_last_error().
#include <cstring>
#include <memory>
#include <unordered_map>

#include "executor.hpp"
#include "planner.hpp"
#include "rtc.hpp"

using namespace mtb;

namespace mtb {
std::shared_ptr<void> make_gather_kernel(const std::string& annotation_text, const std::vector<dtype>& types, const std::vector<box>& domains,
    kernel_entry& out);
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
	g_err = m;
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

box to_box(const mt_rect& r) { return box(point::of(r.rank, r.lo), point::of(r.rank, r.hi)); }

mt_rect from_box(const box& b) {
	mt_rect r{};
	r.rank = b.rank();
	for(int k = 0; k < b.rank(); ++k) {
		r.lo[k] = b.lo[k];
		r.hi[k] = b.hi[k];
	}
	return r;
}

mt_rect from_point(const point& p) {
	mt_rect r{};
	r.rank = p.rank;
	for(int k = 0; k < p.rank; ++k) r.lo[k] = p[k];
	return r;
}

device_id to_dev(mt_device d) { return {d.worker, d.device}; }
mt_device from_dev(device_id d) { return {d.worker, d.device}; }

std::vector<device_id> to_devs(const mt_device* d, int32_t n) {
	std::vector<device_id> v;
	for(int32_t i = 0; i < n; ++i) v.push_back(to_dev(d[i]));
	return v;
}

dtype to_dtype(int32_t t) {
	if(t < MT_I32 || t > MT_BF16) throw validation_error("unknown element type " + std::to_string(t));
	return static_cast<dtype>(t);
}

void emit_chunks(const std::vector<chunk_desc>& v, mt_chunk_desc* out, int64_t cap, int64_t* n) {
	*n = static_cast<int64_t>(v.size());
	for(size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = mt_chunk_desc{v[i].id, from_box(v[i].region), from_dev(v[i].home)};
}

void flatten(const task& t, mt_task& o, std::vector<int64_t>& pool, std::vector<mt_arg_binding>& args) {
	std::memset(&o, 0, sizeof(o));
	o.id = t.id;
	o.worker = t.worker;
	o.kind = static_cast<int32_t>(t.kind);
	o.resource = from_dev(t.resource);
	o.deps_off = static_cast<int64_t>(pool.size());
	o.ndeps = static_cast<int64_t>(t.deps.size());
	pool.insert(pool.end(), t.deps.begin(), t.deps.end());
	o.chunk = t.chunk;
	o.src = t.src;
	o.dst = t.dst;
	o.output = t.output;
	switch(t.kind) {
	case task_kind::create:
		o.region = from_box(t.region);
		o.home = from_dev(t.home);
		o.dtype = static_cast<int32_t>(t.type);
		o.fill = static_cast<int32_t>(t.fill);
		o.fill_op = static_cast<int32_t>(t.fill_op);
		break;
	case task_kind::execute: {
		std::strncpy(o.kernel, t.kern->id.c_str(), MT_KERNEL_NAME_MAX - 1);
		o.device = from_dev(t.device);
		o.sb_blocks = from_box(t.sb_blocks);
		o.sb_threads = from_box(t.sb_threads);
		o.block_size = from_point(t.block_size);
		o.args_off = static_cast<int64_t>(args.size());
		o.nargs = static_cast<int64_t>(t.args.size());
		for(const auto& a : t.args) {
			mt_arg_binding b{};
			b.kind = static_cast<int32_t>(a.kind);
			b.i = a.i;
			b.f = a.f;
			b.chunk = a.chunk;
			args.push_back(b);
		}
		break;
	}
	case task_kind::copy:
		o.src_region = from_box(t.src_region);
		o.dst_region = from_box(t.dst_region);
		break;
	case task_kind::send:
	case task_kind::recv:
		o.region = from_box(t.region);
		o.peer = t.peer;
		o.tag = t.tag;
		break;
	case task_kind::host_write:
	case task_kind::host_read:
		o.region = from_box(t.region);
		o.src_region = from_box(t.src_region);
		o.dtype = static_cast<int32_t>(t.type);
		o.tag = t.tag;
		break;
	case task_kind::allreduce:
		o.region = from_box(t.region);
		o.dtype = static_cast<int32_t>(t.type);
		o.tag = t.tag;
		[[fallthrough]];
	case task_kind::reduce:
		o.op = static_cast<int32_t>(t.op);
		o.inputs_off = static_cast<int64_t>(pool.size());
		o.ninputs = static_cast<int64_t>(t.inputs.size());
		pool.insert(pool.end(), t.inputs.begin(), t.inputs.end());
		break;
	case task_kind::del: break;
	}
}

task unflatten(const mt_task& o, const int64_t* pool, const mt_arg_binding* args) {
	task t;
	t.id = o.id;
	t.worker = o.worker;
	if(o.kind < 0 || o.kind > MT_TASK_HOST_READ) throw validation_error("bad task kind");
	t.kind = static_cast<task_kind>(o.kind);
	t.resource = to_dev(o.resource);
	for(int64_t i = 0; i < o.ndeps; ++i) t.deps.push_back(pool[o.deps_off + i]);
	t.chunk = o.chunk;
	switch(t.kind) {
	case task_kind::create:
		t.region = to_box(o.region);
		t.home = to_dev(o.home);
		t.type = to_dtype(o.dtype);
		t.fill = static_cast<fill_kind>(o.fill);
		t.fill_op = static_cast<reduce_op>(o.fill_op);
		break;
	case task_kind::execute: {
		{
			const int idx = kernel_table::get().find(o.kernel);
			if(idx < 0) throw plan_error(std::string("unknown kernel \"") + o.kernel + "\"");
			t.kern = &kernel_table::get().at(idx);
		}
		t.device = to_dev(o.device);
		t.sb_blocks = to_box(o.sb_blocks);
		t.sb_threads = to_box(o.sb_threads);
		t.block_size = point::of(o.block_size.rank, o.block_size.lo);
		for(int64_t i = 0; i < o.nargs; ++i) {
			const auto& a = args[o.args_off + i];
			t.args.push_back(arg_bind{static_cast<arg_kind>(a.kind), a.i, a.f, a.chunk});
		}
		break;
	}
	case task_kind::copy:
		t.src = o.src;
		t.dst = o.dst;
		t.src_region = to_box(o.src_region);
		t.dst_region = to_box(o.dst_region);
		break;
	case task_kind::send:
	case task_kind::recv:
		t.region = to_box(o.region);
		t.peer = o.peer;
		t.tag = o.tag;
		break;
	case task_kind::host_write:
	case task_kind::host_read:
		t.region = to_box(o.region);
		t.src_region = to_box(o.src_region);
		t.type = to_dtype(o.dtype);
		t.tag = o.tag;
		break;
	case task_kind::allreduce:
		t.region = to_box(o.region);
		t.type = to_dtype(o.dtype);
		t.tag = o.tag;
		[[fallthrough]];
	case task_kind::reduce:
		t.op = static_cast<reduce_op>(o.op);
		for(int64_t i = 0; i < o.ninputs; ++i) t.inputs.push_back(pool[o.inputs_off + i]);
		t.output = o.output;
		break;
	case task_kind::del: break;
	}
	return t;
}

executor_config exec_cfg(const mt_config& c) {
	executor_config e;
	e.workers = c.workers;
	e.devices_per_worker = c.devices_per_worker;
	e.num_gpus = c.num_gpus;
	e.streams_per_device = c.streams_per_device > 0 ? c.streams_per_device : 4;
	e.device_capacity = c.device_capacity;
	e.host_capacity = c.host_capacity;
	e.lookahead = c.lookahead_tasks > 0 ? c.lookahead_tasks : 512;
	e.disk_capacity = c.disk_capacity;
	if(c.spill_dir) e.spill_dir = c.spill_dir;
	e.schedule_seed = c.schedule_seed;
	e.staging_threshold = c.staging_threshold;
	if(c.single_worker) {
		// one process per worker: this process executes worker_rank only, on GPU ordinal
		// gpu_base (+ device index); every rank plans the identical full plan
		if(c.worker_rank < 0 || c.worker_rank >= c.workers) throw validation_error("worker_rank outside the configured workers");
		e.first_worker = c.worker_rank;
		e.local_workers = 1;
		e.gpu_base = c.gpu_base;
		if(e.num_gpus == 0) e.num_gpus = c.devices_per_worker;
	}
	return e;
}

} // namespace

struct mt_exec {
	std::unique_ptr<executor> ex;
	// chunk geometry for host transfers (from create tasks)
	std::unordered_map<int64_t, std::pair<box, dtype>> chunk_geom;
	std::vector<uint8_t> peer_blob;
};

struct mt_ctx {
	mt_config cfg{};
	std::unique_ptr<planner> plan;
	std::unique_ptr<mt_exec> exec;
	std::unordered_map<std::string, annotation> ann_cache;
	std::vector<std::shared_ptr<void>> owned; // descriptors of context-local kernels
};

namespace {

void submit_tasks(mt_exec& e, const std::vector<task>& ts) {
	for(const auto& t : ts)
		if(t.kind == task_kind::create) e.chunk_geom[t.chunk] = {t.region, t.type};
	e.ex->submit(ts);
}

void flush(mt_ctx* ctx) {
	nvtx3::scoped_range_in<mtb::nvtx_domain> range{"mt_flush"};
	if(!ctx->exec) {
		ctx->plan->consume_pending([](const task&) {});
		return;
	}
	mt_exec& e = *ctx->exec;
	bool any = false;
	ctx->plan->consume_pending([&](const task& t) {
		if(t.kind == task_kind::create) e.chunk_geom[t.chunk] = {t.region, t.type};
		e.ex->submit_one(t);
		any = true;
	});
	if(any) e.ex->end_submit();
}

mt_exec& need_exec(mt_ctx* ctx) {
	if(!ctx->exec) throw validation_error("context was created with execute = 0");
	return *ctx->exec;
}

} // namespace

namespace {
// canonical text of a parsed annotation (bindings, accesses, folded linear expressions), the
// same rendering ref_shim.cpp gives the reference's access_annotation
void describe_expr(std::string& o, const mtb::lin_expr& e, const mtb::annotation& a) {
	o += "[" + std::to_string(e.constant) + ",[";
	for(size_t t = 0; t < e.terms.size(); ++t) {
		if(t) o += ",";
		o += "[\"" + a.vars[static_cast<size_t>(e.terms[t].slot)].name + "\"," + std::to_string(e.terms[t].coeff) + "]";
	}
	o += "]]";
}

std::string describe(const mtb::annotation& a) {
	static const char* space[] = {"global", "block", "local"};
	static const char* kind[] = {"read", "write", "readwrite", "reduce"};
	static const char* op[] = {"+", "*", "min", "max"};
	std::string o = "{\"bindings\":[";
	for(size_t v = 0; v < a.vars.size(); ++v) {
		const auto& b = a.vars[v];
		if(b.axis == 0) o += std::string(v ? "]]," : "") + "[\"" + space[static_cast<int>(b.space)] + "\",[";
		else o += ",";
		o += "\"" + b.name + "\"";
	}
	if(!a.vars.empty()) o += "]]";
	o += "],\"accesses\":[";
	for(size_t i = 0; i < a.accesses.size(); ++i) {
		const auto& acc = a.accesses[i];
		if(i) o += ",";
		o += "[\"" + acc.argument + "\",\"" + kind[static_cast<int>(acc.mode.kind)] + "\",\"" + op[static_cast<int>(acc.mode.op)] + "\",[";
		for(size_t k = 0; k < acc.indices.size(); ++k) {
			const auto& ix = acc.indices[k];
			if(k) o += ",";
			if(!ix.is_slice) {
				o += "[\"single\",";
				describe_expr(o, ix.single, a);
				o += "]";
				continue;
			}
			o += "[\"slice\",";
			if(ix.has_lower) describe_expr(o, ix.lower, a);
			else o += "null";
			o += ",";
			if(ix.has_upper) describe_expr(o, ix.upper, a);
			else o += "null";
			o += "]";
		}
		o += "]]";
	}
	return o + "]}";
}
} // namespace

extern "C" {

const char* mt_last_error(void) { return g_err.c_str(); }
const char* mt_version(void) { return "manta-b200 0.1 (sm_100a)"; }

int mt_dist_tile(const mt_rect* domain, const int64_t* extents, const int64_t* halo, const mt_device* devices, int32_t ndev, int64_t first_id,
    mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] {
		const box d = to_box(*domain);
		emit_chunks(tile_dist(d, point::of(d.rank(), extents), point::of(d.rank(), halo), to_devs(devices, ndev), first_id), out, cap, n_out);
	});
}

int mt_dist_replicated(const mt_rect* domain, const mt_device* devices, int32_t ndev, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(replicated_dist(to_box(*domain), to_devs(devices, ndev), first_id), out, cap, n_out); });
}

int mt_dist_single(const mt_rect* domain, mt_device home, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(single_dist(to_box(*domain), to_dev(home), first_id), out, cap, n_out); });
}

int mt_work_block(const mt_rect* grid, const int64_t* block, const int64_t* tps, const mt_device* devices, int32_t ndev, mt_superblock* out,
    int64_t cap, int64_t* n_out) {
	return guarded([&] {
		const box g = to_box(*grid);
		const auto w = block_work_dist(g, point::of(g.rank(), block), point::of(g.rank(), tps), to_devs(devices, ndev));
		*n_out = static_cast<int64_t>(w.size());
		for(size_t i = 0; i < w.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = mt_superblock{from_box(w[i].blocks), from_dev(w[i].device)};
	});
}

int mt_ctx_create(const mt_config* cfg, mt_ctx** out) {
	return guarded([&] {
		auto ctx = std::make_unique<mt_ctx>();
		ctx->cfg = *cfg;
		planner_config pc;
		pc.workers = cfg->workers;
		pc.devices_per_worker = cfg->devices_per_worker;
		pc.suppress_conflict_deps = cfg->suppress_conflict_deps != 0;
		pc.compat_deps = cfg->compat_deps != 0;
		pc.record_accesses = cfg->record_accesses != 0;
		pc.collective_reduce = cfg->collective_reduce != 0;
		pc.plan_cache = cfg->plan_cache_off == 0;
		pc.retain_plan = cfg->drop_executed_tasks == 0;
		ctx->plan = std::make_unique<planner>(pc);
		if(cfg->execute) {
			ctx->exec = std::make_unique<mt_exec>();
			ctx->exec->ex = std::make_unique<executor>(exec_cfg(*cfg));
		}
		*out = ctx.release();
	});
}

int mt_ctx_destroy(mt_ctx* ctx) {
	return guarded([&] { delete ctx; });
}

int mt_ctx_devices(mt_ctx* ctx, mt_device* out, int32_t cap, int32_t* n_out) {
	const auto& d = ctx->plan->devices();
	*n_out = static_cast<int32_t>(d.size());
	for(size_t i = 0; i < d.size() && static_cast<int32_t>(i) < cap; ++i) out[i] = from_dev(d[i]);
	return MT_OK;
}

int mt_array_create(mt_ctx* ctx, const mt_rect* domain, int32_t dt, const mt_chunk_desc* chunks, int64_t nchunks, int32_t fill, int64_t* out_id) {
	return guarded([&] {
		std::vector<chunk_desc> v;
		for(int64_t i = 0; i < nchunks; ++i) v.push_back({chunks[i].id, to_box(chunks[i].region), to_dev(chunks[i].home)});
		if(fill < MT_FILL_NONE || fill > MT_FILL_ONE) throw validation_error("fill must be none, zero or one");
		*out_id = ctx->plan->create_array(to_box(*domain), to_dtype(dt), std::move(v), static_cast<fill_kind>(fill)).id;
	});
}

int mt_array_delete(mt_ctx* ctx, int64_t id) {
	return guarded([&] { ctx->plan->delete_array(id); });
}

int mt_array_chunks(mt_ctx* ctx, int64_t id, mt_chunk_desc* out, int64_t cap, int64_t* n_out) {
	return guarded([&] { emit_chunks(ctx->plan->array(id).chunks, out, cap, n_out); });
}

int mt_launch(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* ann_text, int64_t* first, int64_t* last) {
	return mt_launch_repeat(ctx, kernel, grid, block, work, nwork, args, nargs, ann_text, 1, -1, -1, -1, first, last);
}

int mt_launch_repeat(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* ann_text, int32_t repeat, int64_t swap_a, int64_t swap_b, int32_t flush_every, int64_t* first,
    int64_t* last) {
	return guarded([&] {
		nvtx3::scoped_range_in<mtb::nvtx_domain> range{kernel ? kernel : "mt_launch"}; // planning of the launch(es) (NVTX, visible in nsys)
		if(repeat < 1) throw validation_error("repeat must be at least 1");
		const box g = to_box(*grid);
		std::vector<superblock> w;
		w.reserve(static_cast<size_t>(nwork));
		for(int64_t i = 0; i < nwork; ++i) w.push_back({to_box(work[i].blocks), to_dev(work[i].device)});
		std::vector<launch_arg> la(static_cast<size_t>(nargs));
		for(int32_t i = 0; i < nargs; ++i) {
			la[static_cast<size_t>(i)].kind = args[i].kind == MT_LARG_INT ? launch_arg::int_k : args[i].kind == MT_LARG_FLOAT ? launch_arg::float_k : launch_arg::array_k;
			la[static_cast<size_t>(i)].i = args[i].kind == MT_LARG_INT ? args[i].i : 0;
			la[static_cast<size_t>(i)].f = args[i].kind == MT_LARG_FLOAT ? args[i].f : 0.0;
			la[static_cast<size_t>(i)].array = args[i].array;
		}
		auto it = ctx->ann_cache.find(ann_text);
		if(it == ctx->ann_cache.end()) it = ctx->ann_cache.emplace(ann_text, parse_annotation(ann_text)).first;
		const point blk = point::of(g.rank(), block);
		int64_t lo = -1, hi = -1;
		for(int32_t rep = 0; rep < repeat; ++rep) {
			const auto r = ctx->plan->launch(kernel, g, blk, w, la, it->second);
			if(rep == 0) lo = r.first;
			hi = r.second;
			if(flush_every > 0 && (rep + 1) % flush_every == 0) flush(ctx);
			if(swap_a >= 0 || swap_b >= 0)
				for(auto& a : la) {
					if(a.kind != launch_arg::array_k) continue;
					if(a.array == swap_a)
						a.array = swap_b;
					else if(a.array == swap_b)
						a.array = swap_a;
				}
		}
		if(flush_every == 0) flush(ctx);
		*first = lo;
		*last = hi;
	});
}

int mt_flush(mt_ctx* ctx) {
	return guarded([&] { flush(ctx); });
}

int mt_sync(mt_ctx* ctx) {
	return guarded([&] {
		flush(ctx);
		if(ctx->exec) ctx->exec->ex->sync();
	});
}

int mt_array_read(mt_ctx* ctx, int64_t id, void* host, uint64_t bytes) {
	return guarded([&] {
		mt_exec& e = need_exec(ctx);
		flush(ctx);
		e.ex->sync();
		const array_rec& a = ctx->plan->array(id);
		if(bytes < static_cast<uint64_t>(a.domain.volume()) * dtype_size(a.type)) throw validation_error("host buffer too small");
		for(const auto& c : a.chunks)
			if(e.ex->has_chunk(c.id)) e.ex->download(c.id, host, a.domain, c.region); // single_worker: local chunks only
	});
}

int mt_array_write(mt_ctx* ctx, int64_t id, const void* host, uint64_t bytes) {
	return guarded([&] {
		mt_exec& e = need_exec(ctx);
		const array_rec& a = ctx->plan->array(id);
		if(bytes < static_cast<uint64_t>(a.domain.volume()) * dtype_size(a.type)) throw validation_error("host buffer too small");
		// synchronous upload outside the plan: every queued task (a copy on another GPU may
		// still read these chunks) completes first
		flush(ctx);
		e.ex->sync();
		for(const auto& c : a.chunks)
			if(e.ex->has_chunk(c.id)) e.ex->upload(c.id, host, a.domain); // single_worker: local chunks only
		// the chunks now hold defined data: later launches may read them
		ctx->plan->mark_filled(id);
	});
}

int mt_array_write_async(mt_ctx* ctx, int64_t id, const void* host, uint64_t bytes) {
	return guarded([&] { // plan-only contexts just plan the transfer
		const array_rec& a = ctx->plan->array(id);
		if(bytes < static_cast<uint64_t>(a.domain.volume()) * dtype_size(a.type)) throw validation_error("host buffer too small");
		ctx->plan->host_transfer(id, reinterpret_cast<uint64_t>(host), true);
		flush(ctx);
	});
}

int mt_array_read_async(mt_ctx* ctx, int64_t id, void* host, uint64_t bytes) {
	return guarded([&] {
		const array_rec& a = ctx->plan->array(id);
		if(bytes < static_cast<uint64_t>(a.domain.volume()) * dtype_size(a.type)) throw validation_error("host buffer too small");
		ctx->plan->host_transfer(id, reinterpret_cast<uint64_t>(host), false);
		flush(ctx);
	});
}

namespace {
int host_box_transfer(mt_ctx* ctx, int64_t id, const mt_rect* host_box, uint64_t host, uint64_t bytes, bool write) {
	return guarded([&] {
		const array_rec& a = ctx->plan->array(id);
		if(!host_box) throw validation_error("host box is required");
		const box hb = to_box(*host_box);
		if(hb.rank() != a.domain.rank() || hb.is_empty() || !encloses(a.domain, hb)) throw validation_error("host box must be a non-empty box inside the array's domain");
		if(bytes < static_cast<uint64_t>(hb.volume()) * dtype_size(a.type)) throw validation_error("host buffer too small");
		ctx->plan->host_transfer(id, host, write, &hb);
		flush(ctx);
	});
}
} // namespace

int mt_array_write_box_async(mt_ctx* ctx, int64_t id, const mt_rect* host_box, const void* host, uint64_t bytes) {
	return host_box_transfer(ctx, id, host_box, reinterpret_cast<uint64_t>(host), bytes, true);
}

int mt_array_read_box_async(mt_ctx* ctx, int64_t id, const mt_rect* host_box, void* host, uint64_t bytes) {
	return host_box_transfer(ctx, id, host_box, reinterpret_cast<uint64_t>(host), bytes, false);
}

int mt_array_check_replicas(mt_ctx* ctx, int64_t id, int32_t* coherent) {
	return guarded([&] {
		mt_exec& e = need_exec(ctx);
		flush(ctx);
		e.ex->sync();
		const array_rec& a = ctx->plan->array(id);
		const size_t elem = dtype_size(a.type);
		*coherent = 1;
		for(size_t i = 0; i < a.chunks.size() && *coherent; ++i) {
			for(size_t j = i + 1; j < a.chunks.size() && *coherent; ++j) {
				const box ov = intersect(a.chunks[i].region, a.chunks[j].region);
				if(ov.is_empty() || !e.ex->has_chunk(a.chunks[i].id) || !e.ex->has_chunk(a.chunks[j].id)) continue;
				std::vector<char> x(static_cast<size_t>(ov.volume()) * elem), y(x.size());
				e.ex->download(a.chunks[i].id, x.data(), ov, ov);
				e.ex->download(a.chunks[j].id, y.data(), ov, ov);
				if(std::memcmp(x.data(), y.data(), x.size()) != 0) *coherent = 0;
			}
		}
	});
}

int mt_plan_export(mt_ctx* ctx, int64_t first, int64_t last, mt_task* tasks, int64_t task_cap, int64_t* ntasks, int64_t* pool, int64_t pool_cap,
    int64_t* npool, mt_arg_binding* args, int64_t args_cap, int64_t* nargs) {
	return guarded([&] {
		std::vector<mt_task> ts;
		std::vector<int64_t> p;
		std::vector<mt_arg_binding> a;
		for(const auto& t : ctx->plan->plan()) {
			if(t.id < first || t.id >= last) continue;
			mt_task o;
			flatten(t, o, p, a);
			ts.push_back(o);
		}
		*ntasks = static_cast<int64_t>(ts.size());
		*npool = static_cast<int64_t>(p.size());
		*nargs = static_cast<int64_t>(a.size());
		if(tasks && task_cap >= *ntasks) std::memcpy(tasks, ts.data(), ts.size() * sizeof(mt_task));
		if(pool && pool_cap >= *npool) std::memcpy(pool, p.data(), p.size() * sizeof(int64_t));
		if(args && args_cap >= *nargs) std::memcpy(args, a.data(), a.size() * sizeof(mt_arg_binding));
	});
}

int64_t mt_plan_size(mt_ctx* ctx) { return ctx->plan->next_id(); }

uint64_t mt_plan_cache_hits(mt_ctx* ctx) { return ctx->plan->plan_cache_hits(); }

int mt_annotation_describe(const char* text, char* out, int64_t cap, int64_t* len) {
	return guarded([&] {
		const std::string s = describe(mtb::parse_annotation(text ? text : ""));
		*len = static_cast<int64_t>(s.size());
		if(out && cap > static_cast<int64_t>(s.size())) std::memcpy(out, s.c_str(), s.size() + 1);
	});
}

int mt_plan_accesses(mt_ctx* ctx, mt_access* out, int64_t cap, int64_t* n_out) {
	return guarded([&] {
		const auto& a = ctx->plan->accesses();
		*n_out = static_cast<int64_t>(a.size());
		for(size_t i = 0; i < a.size() && static_cast<int64_t>(i) < cap; ++i) {
			mt_access r{};
			r.task = a[i].task;
			r.chunk = a[i].chunk;
			r.region = from_box(a[i].region);
			r.write = a[i].write ? 1 : 0;
			out[i] = r;
		}
	});
}

int mt_chunk_meta(mt_ctx* ctx, int64_t chunk, mt_chunk_desc* desc, int32_t* dt, int32_t* temp) {
	return guarded([&] {
		const auto& m = ctx->plan->chunk(chunk);
		*desc = mt_chunk_desc{m.desc.id, from_box(m.desc.region), from_dev(m.desc.home)};
		*dt = static_cast<int32_t>(m.type);
		*temp = m.temp ? 1 : 0;
	});
}

mt_exec* mt_ctx_exec(mt_ctx* ctx) { return ctx->exec.get(); }

int mt_exec_create(const mt_config* cfg, mt_exec** out) {
	return guarded([&] {
		auto e = std::make_unique<mt_exec>();
		e->ex = std::make_unique<executor>(exec_cfg(*cfg));
		*out = e.release();
	});
}

int mt_exec_destroy(mt_exec* ex) {
	return guarded([&] { delete ex; });
}

int mt_exec_submit(mt_exec* ex, const mt_task* tasks, int64_t n, const int64_t* pool, const mt_arg_binding* args) {
	return guarded([&] {
		std::vector<task> ts;
		ts.reserve(static_cast<size_t>(n));
		for(int64_t i = 0; i < n; ++i) ts.push_back(unflatten(tasks[i], pool, args));
		submit_tasks(*ex, ts);
	});
}

int mt_exec_sync(mt_exec* ex) {
	return guarded([&] { ex->ex->sync(); });
}

int mt_exec_read_chunk(mt_exec* ex, int64_t chunk, void* dst, uint64_t bytes) {
	return guarded([&] {
		const auto it = ex->chunk_geom.find(chunk);
		if(it == ex->chunk_geom.end()) throw validation_error("chunk " + std::to_string(chunk) + " was never created on this system");
		if(bytes < static_cast<uint64_t>(it->second.first.volume()) * dtype_size(it->second.second)) throw validation_error("host buffer too small");
		ex->ex->sync();
		ex->ex->download(chunk, dst, it->second.first, it->second.first);
	});
}

int mt_exec_write_chunk(mt_exec* ex, int64_t chunk, const void* src, uint64_t bytes) {
	return guarded([&] {
		const auto it = ex->chunk_geom.find(chunk);
		if(it == ex->chunk_geom.end()) throw validation_error("chunk " + std::to_string(chunk) + " was never created on this system");
		if(bytes < static_cast<uint64_t>(it->second.first.volume()) * dtype_size(it->second.second)) throw validation_error("host buffer too small");
		ex->ex->upload(chunk, src, it->second.first);
	});
}

int mt_exec_report_json(mt_exec* ex, char* buf, int64_t cap, int64_t* len) {
	return guarded([&] {
		const std::string s = ex->ex->report_json();
		*len = static_cast<int64_t>(s.size());
		if(buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
	});
}

int mt_exec_stats(mt_exec* ex, uint64_t* out, int32_t n) {
	return guarded([&] {
		const auto& c = ex->ex->counters();
		const uint64_t v[] = {c.tasks, c.kernels, c.copies, c.bytes_copied, c.bytes_sent, c.bytes_received, c.peak_device_bytes, c.evictions,
		    c.bytes_device_to_host, c.bytes_host_to_device, c.dead_drops, c.dead_skips, c.host_reclaims, c.bytes_host_in, c.bytes_host_out,
		    c.graph_captures, c.graph_replays, c.bytes_host_to_disk, c.bytes_disk_to_host, c.messages, c.message_ops, c.fused_copies, c.bytes_fused};
		for(int32_t i = 0; i < n && i < static_cast<int32_t>(sizeof(v) / sizeof(v[0])); ++i) out[i] = v[i];
	});
}

void* mt_exec_last_stream(mt_exec* ex) { return ex->ex->last_exec_stream(); }

int mt_ctx_peer_export(mt_ctx* ctx, void* buf, int64_t cap, int64_t* len) {
	return guarded([&] {
		mt_exec& e = need_exec(ctx);
		if(e.peer_blob.empty()) e.peer_blob = e.ex->peer_export();
		*len = static_cast<int64_t>(e.peer_blob.size());
		if(buf && cap >= *len) std::memcpy(buf, e.peer_blob.data(), e.peer_blob.size());
	});
}

int mt_ctx_peer_import(mt_ctx* ctx, const void* blobs, int64_t blob_len, int32_t nblobs) {
	return guarded([&] {
		mt_exec& e = need_exec(ctx);
		std::vector<std::vector<uint8_t>> v;
		const auto* p = static_cast<const uint8_t*>(blobs);
		for(int32_t i = 0; i < nblobs; ++i) v.emplace_back(p + i * blob_len, p + (i + 1) * blob_len);
		e.ex->peer_import(v);
	});
}

int mt_ctx_nccl_unique_id(mt_ctx* ctx, const char* nccl_lib, void* id128) {
	return guarded([&] { need_exec(ctx).ex->nccl_unique_id(nccl_lib, id128); });
}

int mt_ctx_nccl_init(mt_ctx* ctx, const char* nccl_lib, const void* id128) {
	return guarded([&] {
		if(!ctx->cfg.single_worker) throw validation_error("an NCCL communicator is only used with single_worker (one process per worker)");
		need_exec(ctx).ex->nccl_init(nccl_lib, id128, ctx->cfg.workers, ctx->cfg.worker_rank);
	});
}

int mt_exec_mark(mt_exec* ex, int32_t slot) {
	return guarded([&] { ex->ex->mark(slot); });
}

int mt_exec_elapsed_ms(mt_exec* ex, double* ms) {
	return guarded([&] { *ms = ex->ex->elapsed_ms(); });
}

int mt_exec_profile(mt_exec* ex, int32_t on) {
	return guarded([&] { ex->ex->set_profile(on != 0); });
}

int mt_exec_trace(mt_exec* ex, int32_t on) {
	return guarded([&] { ex->ex->set_trace(on != 0); });
}

int mt_exec_kernel_time(mt_exec* ex, const char* kernel, int64_t* count, double* total_ms) {
	return guarded([&] { ex->ex->kernel_time(kernel, count, total_ms); });
}

namespace {
kernel_entry make_entry(const char* id, const mt_param_spec* params, int32_t nparams, mt_launcher_fn launcher, const void* user) {
	kernel_entry e;
	e.id = id;
	for(int32_t i = 0; i < nparams; ++i) {
		param_sig p;
		p.name = params[i].name;
		p.is_array = params[i].kind == MT_PARAM_ARRAY;
		p.type = to_dtype(params[i].dtype);
		p.rank = params[i].rank;
		p.writable = params[i].writable != 0;
		e.params.push_back(p);
	}
	e.launcher = launcher;
	e.user = user;
	return e;
}
} // namespace

int mt_ctx_gather_register(mt_ctx* ctx, const char* id, const char* annotation_text, int32_t naccess, const int32_t* dtypes, const mt_rect* domains) {
	return guarded([&] {
		std::vector<dtype> types;
		std::vector<box> doms;
		for(int32_t i = 0; i < naccess; ++i) {
			types.push_back(to_dtype(dtypes[i]));
			doms.push_back(to_box(domains[i]));
		}
		kernel_entry e;
		e.id = id;
		ctx->owned.push_back(make_gather_kernel(annotation_text, types, doms, e));
		ctx->plan->add_local_kernel(std::move(e));
	});
}

int mt_ctx_kernel_compile(mt_ctx* ctx, const char* id, const mt_param_spec* params, int32_t nparams, const char* source) {
	return guarded([&] {
		if(!source) throw validation_error("kernel source must not be NULL");
		kernel_entry e = make_entry(id, params, nparams, nullptr, nullptr);
		ctx->owned.push_back(make_rtc_kernel(id, e.params, source, e));
		ctx->plan->add_local_kernel(std::move(e));
	});
}

int mt_wrapper_source(const char* id, const mt_param_spec* params, int32_t nparams, const int64_t* block_offset, int32_t rank, const int64_t* offsets,
    const int64_t* strides, char* out, int64_t cap, int64_t* len) {
	return guarded([&] {
		const kernel_entry e = make_entry(id, params, nparams, nullptr, nullptr);
		std::vector<std::vector<int64_t>> offs, sts;
		size_t at = 0;
		for(const auto& p : e.params) {
			if(!p.is_array) continue;
			offs.emplace_back(offsets + at, offsets + at + p.rank);
			sts.emplace_back(strides + at, strides + at + p.rank);
			at += static_cast<size_t>(p.rank);
		}
		const std::string s = wrapper_source(id, e.params, std::vector<int64_t>(block_offset, block_offset + rank), offs, sts);
		*len = static_cast<int64_t>(s.size());
		if(out && cap > *len) std::memcpy(out, s.c_str(), s.size() + 1);
	});
}

int mt_ctx_kernel_register(mt_ctx* ctx, const char* id, const mt_param_spec* params, int32_t nparams, mt_launcher_fn launcher, const void* user) {
	return guarded([&] { ctx->plan->add_local_kernel(make_entry(id, params, nparams, launcher, user)); });
}

int mt_kernel_register(const char* id, const mt_param_spec* params, int32_t nparams, mt_launcher_fn launcher) {
	return guarded([&] {
		if(!launcher) throw validation_error("kernel launcher must not be NULL");
		kernel_entry e;
		e.id = id;
		for(int32_t i = 0; i < nparams; ++i) {
			param_sig p;
			p.name = params[i].name;
			p.is_array = params[i].kind == MT_PARAM_ARRAY;
			p.type = to_dtype(params[i].dtype);
			p.rank = params[i].rank;
			p.writable = params[i].writable != 0;
			e.params.push_back(p);
		}
		e.launcher = launcher;
		kernel_table::get().add(std::move(e));
	});
}

int mt_kernel_count(void) { return kernel_table::get().size(); }

int mt_kernel_info(int32_t index, char* id, int32_t id_cap, mt_param_spec* params, int32_t cap, int32_t* nparams) {
	return guarded([&] {
		const auto& e = kernel_table::get().at(index);
		if(id && id_cap > 0) {
			std::strncpy(id, e.id.c_str(), static_cast<size_t>(id_cap) - 1);
			id[id_cap - 1] = 0;
		}
		*nparams = static_cast<int32_t>(e.params.size());
		for(int32_t i = 0; i < *nparams && i < cap; ++i) {
			const auto& p = e.params[static_cast<size_t>(i)];
			mt_param_spec s{};
			std::strncpy(s.name, p.name.c_str(), sizeof(s.name) - 1);
			s.kind = p.is_array ? MT_PARAM_ARRAY : MT_PARAM_SCALAR;
			s.dtype = static_cast<int32_t>(p.type);
			s.rank = p.rank;
			s.writable = p.writable ? 1 : 0;
			params[i] = s;
		}
	});
}

} // extern "C"
