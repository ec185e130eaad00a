// The reference-side binding a manta maintainer adds to run their plans on B200
// (INTEGRATION.md): `gpu_runtime` has manta::system_runtime's interface
// (proj/include/manta/runtime.hpp:70-98) and forwards every task through the C-ABI of
// include/manta_b200.h. main() drives the UNMODIFIED reference driver (proj/src/planner.cpp,
// linked from oracle/_ref) on the paper's iterated stencil and checks that the GPU executor
// and the reference CPU executor produce byte-identical chunks.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "manta/planner.hpp"
#include "manta/runtime.hpp"

#include "../../include/manta_b200.h"

namespace manta {

class gpu_runtime {
  public:
	gpu_runtime(int workers, int devices_per_worker) {
		mt_config c{};
		c.workers = workers;
		c.devices_per_worker = devices_per_worker;
		c.execute = 1;
		c.num_gpus = 1;
		check(mt_exec_create(&c, &ex_));
	}
	~gpu_runtime() { mt_exec_destroy(ex_); }

	void submit(const std::vector<task>& tasks) {
		std::vector<mt_task> flat;
		std::vector<int64_t> pool;
		std::vector<mt_arg_binding> args;
		for(const auto& t : tasks) flat.push_back(convert(t, pool, args));
		check(mt_exec_submit(ex_, flat.data(), static_cast<int64_t>(flat.size()), pool.data(), args.data()));
	}
	void synchronize() { check(mt_exec_sync(ex_)); }
	std::vector<std::byte> read_chunk(chunk_id id, std::size_t bytes) {
		std::vector<std::byte> out(bytes);
		check(mt_exec_read_chunk(ex_, id, out.data(), bytes));
		return out;
	}

  private:
	mt_exec* ex_ = nullptr;

	static void check(int rc) {
		if(rc == MT_OK) return;
		if(rc == MT_EEXEC) throw execution_error(mt_last_error());
		if(rc == MT_EPLAN) throw plan_error(mt_last_error());
		throw validation_error(mt_last_error());
	}
	static mt_rect R(const rect& r) {
		mt_rect o{};
		o.rank = r.rank();
		for(int k = 0; k < r.rank(); ++k) {
			o.lo[k] = r.lo[k];
			o.hi[k] = r.hi[k];
		}
		return o;
	}
	static mt_rect P(const point& p) {
		mt_rect o{};
		o.rank = p.rank;
		for(int k = 0; k < p.rank; ++k) o.lo[k] = p[k];
		return o;
	}
	static mt_device D(device_id d) { return {d.worker, d.device}; }

	static mt_task convert(const task& t, std::vector<int64_t>& pool, std::vector<mt_arg_binding>& args) {
		mt_task o{};
		o.id = t.id;
		o.worker = t.worker;
		o.kind = static_cast<int32_t>(t.op.index()); // create, delete, execute, copy, send, recv, reduce
		o.resource = D(t.resource);
		o.deps_off = static_cast<int64_t>(pool.size());
		o.ndeps = static_cast<int64_t>(t.deps.size());
		pool.insert(pool.end(), t.deps.begin(), t.deps.end());
		if(auto* c = std::get_if<create_task>(&t.op)) {
			o.chunk = c->chunk.id;
			o.region = R(c->chunk.region);
			o.home = D(c->chunk.home);
			o.dtype = static_cast<int32_t>(c->type); // i32, i64, f32, f64 share the C-ABI codes
			o.fill = static_cast<int32_t>(c->fill.kind);
			o.fill_op = static_cast<int32_t>(c->fill.op);
		} else if(auto* d = std::get_if<delete_task>(&t.op)) {
			o.chunk = d->chunk;
		} else if(auto* e = std::get_if<execute_task>(&t.op)) {
			std::strncpy(o.kernel, e->kernel.c_str(), MT_KERNEL_NAME_MAX - 1);
			o.device = D(e->device);
			o.sb_blocks = R(e->superblock_blocks);
			o.sb_threads = R(e->superblock_threads);
			o.block_size = P(e->block_size);
			o.args_off = static_cast<int64_t>(args.size());
			o.nargs = static_cast<int64_t>(e->args.size());
			for(const auto& b : e->args) args.push_back(mt_arg_binding{static_cast<int32_t>(b.kind), 0, b.scalar_int, b.scalar_float, b.chunk});
		} else if(auto* c = std::get_if<copy_task>(&t.op)) {
			o.src = c->src;
			o.dst = c->dst;
			o.src_region = R(c->src_region);
			o.dst_region = R(c->dst_region);
		} else if(auto* s = std::get_if<send_task>(&t.op)) {
			o.chunk = s->chunk;
			o.region = R(s->region);
			o.peer = s->peer_worker;
			o.tag = s->tag;
		} else if(auto* r = std::get_if<recv_task>(&t.op)) {
			o.chunk = r->chunk;
			o.region = R(r->region);
			o.peer = r->peer_worker;
			o.tag = r->tag;
		} else if(auto* r = std::get_if<reduce_task>(&t.op)) {
			o.op = static_cast<int32_t>(r->op);
			o.inputs_off = static_cast<int64_t>(pool.size());
			o.ninputs = static_cast<int64_t>(r->inputs.size());
			pool.insert(pool.end(), r->inputs.begin(), r->inputs.end());
			o.output = r->output;
		}
		return o;
	}
};

} // namespace manta

int main() {
	using namespace manta;
	const auto registry = kernel_registry::with_builtins();
	driver drv(driver_config{2, 2, false}, registry);
	system_config cfg;
	cfg.workers = 2;
	cfg.devices_per_worker = 2;
	cfg.memory.disk_in_memory = true;
	system_runtime cpu(cfg, registry);
	gpu_runtime gpu(2, 2);

	const std::int64_t n = 1 << 16;
	const auto dist = [&] { return stencil_dist(rect({0}, {n}), {n / 8}, {1}, drv.devices()); };
	auto in = drv.create_array(rect({0}, {n}), dtype::f32, dist(), fill_spec::one()).id;
	auto out = drv.create_array(rect({0}, {n}), dtype::f32, dist(), fill_spec::zero()).id;
	const auto annotation = parse_annotation("global i => read input[i-1:i+1], write output[i]");
	const auto work = block_work_dist(rect({0}, {n}), {16}, {n / 8}, drv.devices());
	for(int it = 0; it < 10; ++it) {
		drv.launch("stencil1d", rect({0}, {n}), {16}, work, {launch_arg::scalar(n), launch_arg::array(out), launch_arg::array(in)}, annotation);
		const auto pending = drv.take_pending();
		cpu.submit(pending);
		gpu.submit(pending);
		std::swap(in, out);
	}
	cpu.synchronize();
	gpu.synchronize();
	int mismatches = 0;
	for(const auto& c : drv.registry().get(in).distribution.chunks) {
		const auto want = cpu.read_chunk(c.id);
		const auto got = gpu.read_chunk(c.id, want.size());
		if(std::memcmp(want.data(), got.data(), want.size()) != 0) ++mismatches;
	}
	std::printf("%s: %d chunk mismatches (reference driver -> B200 executor vs reference CPU executor)\n", mismatches ? "FAIL" : "PASS", mismatches);
	return mismatches ? 1 : 0;
}
