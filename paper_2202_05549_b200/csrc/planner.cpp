#include "planner.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>

namespace mtb {

planner::planner(const planner_config& cfg) : cfg_(cfg), deps_(cfg.compat_deps) {
	if(cfg.workers < 1 || cfg.devices_per_worker < 1) throw validation_error("system needs at least one worker with one device");
	for(int w = 0; w < cfg.workers; ++w)
		for(int d = 0; d < cfg.devices_per_worker; ++d) devices_.push_back({w, d});
}

const array_rec& planner::array(int64_t id) const {
	const auto it = arrays_.find(id);
	if(it == arrays_.end()) throw validation_error("array " + std::to_string(id) + " is not live");
	return *it->second;
}

const chunk_meta& planner::chunk(int64_t id) const {
	const auto it = chunks_.find(id);
	if(it == chunks_.end()) throw validation_error("unknown chunk " + std::to_string(id));
	return it->second;
}

void planner::add_local_kernel(kernel_entry e) {
	if(e.id.empty()) throw validation_error("kernel id must not be empty");
	for(const auto& p : e.params)
		if(p.is_array && (p.rank < 1 || p.rank > kMaxRank))
			throw validation_error("kernel \"" + e.id + "\" parameter \"" + p.name + "\" has unsupported rank");
	for(const auto& k : local_kernels_)
		if(k->id == e.id) throw validation_error("kernel \"" + e.id + "\" is already registered");
	local_kernels_.push_back(std::make_unique<kernel_entry>(std::move(e)));
}

const kernel_entry* planner::find_kernel(const std::string& id) const {
	for(const auto& k : local_kernels_)
		if(k->id == id) return k.get();
	const auto& table = kernel_table::get();
	const int idx = table.find(id);
	return idx < 0 ? nullptr : &table.at(idx);
}

std::vector<task> planner::take_pending() {
	std::vector<task> out;
	consume_pending([&](const task& t) { out.push_back(t); });
	return out; // already in id order: ids are assigned at emission
}

int64_t planner::emit(task&& t) {
	std::sort(t.deps.begin(), t.deps.end());
	t.deps.erase(std::unique(t.deps.begin(), t.deps.end()), t.deps.end());
	t.id = next_task_++;
	plan_.push_back(std::move(t));
	return next_task_ - 1;
}

int64_t planner::new_temp(const box& region, device_id home, dtype type) {
	const int64_t id = next_chunk_++;
	chunks_[id] = chunk_meta{chunk_desc{id, region, home}, type, true};
	return id;
}

void planner::emit_delete_temp(int worker, device_id dev, int64_t temp) {
	const auto it = temp_users_.find(temp);
	task d;
	d.worker = worker;
	d.resource = dev;
	d.kind = task_kind::del;
	d.deps = it->second; // emit() sorts its own copy
	d.chunk = temp;
	emit(std::move(d));
	it->second.clear();
	if(spare_users_.size() < 4096) spare_users_.push_back(std::move(it->second));
	temp_users_.erase(it);
	if(!cfg_.retain_plan) chunks_.erase(temp);
}

int64_t planner::emit_create(int worker, device_id dev, int64_t chunk_id, fill_kind fill, reduce_op op) {
	const auto& m = chunk(chunk_id);
	task t;
	t.worker = worker;
	t.resource = dev;
	t.kind = task_kind::create;
	t.chunk = chunk_id;
	t.region = m.desc.region;
	t.home = m.desc.home;
	t.type = m.type;
	t.fill = fill;
	t.fill_op = op;
	return emit(std::move(t));
}

// registry access for one task (array_registry.cpp:41-67 + planner.cpp:62-70)
void planner::record(int64_t c, int64_t t, bool write, const box& region, bool check_filled, std::vector<int64_t>& out) {
	if(recording_ && std::find(rec_chunks_.begin(), rec_chunks_.end(), c) == rec_chunks_.end()) {
		rec_chunks_.push_back(c);
		rec_before_.push_back(deps_.save(c));
	}
	if(check_filled && !deps_.filled(c))
		throw plan_error("chunk " + std::to_string(c) + " is read before any fill or write; its contents would be undefined");
	if(cfg_.suppress_conflict_deps) {
		static thread_local std::vector<int64_t> discard;
		discard.clear();
		if(write)
			deps_.write(c, t, region, discard);
		else
			deps_.read(c, t, region, discard);
	} else if(write) {
		deps_.write(c, t, region, out);
	} else {
		deps_.read(c, t, region, out);
	}
	if(cfg_.record_accesses) accesses_.push_back({t, c, region, write});
}

// copy within a worker, or a tagged send/recv pair across workers (planner.cpp:72-120)
int64_t planner::transfer(int64_t src, int64_t dst, const box& region, std::vector<int64_t> src_deps, std::vector<int64_t> dst_deps) {
	const chunk_meta sm = chunk(src), dm = chunk(dst);
	if(sm.desc.home.worker == dm.desc.home.worker) {
		const int64_t tid = next_task_;
		std::vector<int64_t> d = std::move(src_deps);
		d.insert(d.end(), dst_deps.begin(), dst_deps.end());
		if(!sm.temp) record(src, tid, false, region, true, d);
		if(!dm.temp) record(dst, tid, true, region, false, d);
		task t;
		t.worker = dm.desc.home.worker;
		t.resource = dm.desc.home;
		t.kind = task_kind::copy;
		t.deps = std::move(d);
		t.src = src;
		t.dst = dst;
		t.src_region = region;
		t.dst_region = region;
		const int64_t id = emit(std::move(t));
		if(sm.temp) touch(src, id);
		if(dm.temp) touch(dst, id);
		return id;
	}
	const int sw = sm.desc.home.worker, dw = dm.desc.home.worker;
	const uint64_t tag = tags_[{sw, dw}]++;
	const int64_t send_tid = next_task_;
	if(!sm.temp) record(src, send_tid, false, region, true, src_deps);
	task s;
	s.worker = sw;
	s.resource = sm.desc.home;
	s.kind = task_kind::send;
	s.deps = std::move(src_deps);
	s.chunk = src;
	s.region = region;
	s.peer = dw;
	s.tag = tag;
	const int64_t send_id = emit(std::move(s));
	if(sm.temp) touch(src, send_id);
	const int64_t recv_tid = next_task_;
	if(!dm.temp) record(dst, recv_tid, true, region, false, dst_deps);
	task r;
	r.worker = dw;
	r.resource = dm.desc.home;
	r.kind = task_kind::recv;
	r.deps = std::move(dst_deps);
	r.chunk = dst;
	r.region = region;
	r.peer = sw;
	r.tag = tag;
	const int64_t recv_id = emit(std::move(r));
	if(dm.temp) touch(dst, recv_id);
	return recv_id;
}

const array_rec& planner::create_array(const box& domain, dtype type, std::vector<chunk_desc> chunks, fill_kind fill) {
	for(auto& c : chunks) {
		if(c.home.worker < 0 || c.home.worker >= cfg_.workers || c.home.device < 0 || c.home.device >= cfg_.devices_per_worker)
			throw validation_error("chunk home " + to_string(c.home) + " is outside the configured system");
		c.id = next_chunk_++;
	}
	if(domain.rank() < 1 || domain.rank() > kMaxRank) throw validation_error("arrays have between one and three dimensions");
	if(domain.is_empty()) throw validation_error("array domain is empty");
	for(const auto& c : chunks)
		if(c.region.rank() != domain.rank()) throw validation_error("axis-count mismatch: chunk vs domain");
	validate_chunks(chunks, domain);
	auto rec = std::make_unique<array_rec>();
	rec->id = next_array_++;
	rec->domain = domain;
	rec->type = type;
	rec->chunks = std::move(chunks);
	rec->index.build(rec->chunks);
	array_rec& a = *rec;
	arrays_.emplace(a.id, std::move(rec));
	for(const auto& c : a.chunks) {
		chunks_[c.id] = chunk_meta{c, type, false};
		deps_.add_chunk(c.id, c.region);
		const int64_t id = emit_create(c.home.worker, c.home, c.id, fill, reduce_op::plus);
		deps_.mark_created(c.id, id, fill != fill_kind::none);
		if(cfg_.record_accesses) accesses_.push_back({id, c.id, c.region, true});
	}
	return a;
}

void planner::delete_array(int64_t id) {
	const std::vector<chunk_desc> chunks = array(id).chunks;
	for(const auto& c : chunks) {
		std::vector<int64_t> d;
		record(c.id, next_task_, true, c.region, false, d);
		task t;
		t.worker = c.home.worker;
		t.resource = c.home;
		t.kind = task_kind::del;
		t.deps = std::move(d);
		t.chunk = c.id;
		emit(std::move(t));
	}
	for(const auto& c : chunks) deps_.drop_chunk(c.id);
	arrays_.erase(id);
}

void planner::mark_filled(int64_t id) {
	for(const auto& c : array(id).chunks) deps_.mark_filled(c.id);
}

namespace {

struct bound_param {
	size_t param = 0;
	int64_t array = -1;
	const access_decl* acc = nullptr;
	size_t access_index = 0;
};

} // namespace

// ---- launch-plan memo ------------------------------------------------------------------------
//
// Planning is a deterministic function of the call (kernel, grid, block, work, arguments,
// annotation), of the conflict state of the chunks the launch touches, of the per-pair message
// tags and of the next task / chunk ids. An iterative loop repeats the same calls (a ping-pong
// heat step is two alternating calls), and once the loop is in steady state every touched chunk
// is in the state it had one period earlier with all task ids moved by the tasks emitted since.
// A repeated call whose chunks pass that test (dep_tracker::matches) replays the recorded tasks
// with ids, dependencies and tags moved, and sets the chunks to the recorded after-state moved
// the same way: exactly the plan a fresh planning pass would emit, at a fraction of its cost.
// Launches that create temporaries, reduce trees or collectives are not recorded.
constexpr size_t kMemoMaxSuperblocks = 256;
constexpr size_t kMemos = 8;

bool planner::same_call(const launch_memo& m, const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
    const std::vector<launch_arg>& args, const annotation& ann) const {
	if(m.ann != &ann || m.kernel != kernel || !(m.grid == grid) || !(m.block == block) || m.work.size() != work.size() || m.args.size() != args.size())
		return false;
	for(size_t i = 0; i < work.size(); ++i)
		if(!(m.work[i].blocks == work[i].blocks) || !(m.work[i].device == work[i].device)) return false;
	for(size_t i = 0; i < args.size(); ++i) {
		const auto& a = m.args[i];
		const auto& b = args[i];
		if(a.kind != b.kind || a.i != b.i || a.array != b.array || std::memcmp(&a.f, &b.f, sizeof(double)) != 0) return false;
	}
	return true;
}

bool planner::replay(const launch_memo& m, std::pair<int64_t, int64_t>& out) {
	const int64_t delta = next_task_ - m.first;
	for(size_t i = 0; i < m.chunks.size(); ++i)
		if(!deps_.matches(m.chunks[i], m.before[i], delta)) return false;
	const int64_t first = next_task_;
	for(const auto& rec : m.tasks) {
		task t = rec;
		for(auto& d : t.deps) d += delta;
		if(t.kind == task_kind::send || t.kind == task_kind::recv) {
			const std::pair<int, int> pair = t.kind == task_kind::send ? std::make_pair(t.worker, t.peer) : std::make_pair(t.peer, t.worker);
			const auto b = m.tags_before.find(pair);
			t.tag = t.tag - (b == m.tags_before.end() ? 0 : b->second) + tags_[pair];
		}
		emit(std::move(t));
	}
	for(const auto& [pair, used] : m.tags_used) tags_[pair] += used;
	for(size_t i = 0; i < m.chunks.size(); ++i) deps_.restore(m.chunks[i], m.after[i], delta);
	if(cfg_.record_accesses)
		for(auto a : m.accesses) {
			a.task += delta;
			accesses_.push_back(a);
		}
	++memo_hits_;
	out = {first, next_task_};
	return true;
}

std::pair<int64_t, int64_t> planner::launch(const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
    const std::vector<launch_arg>& args, const annotation& ann) {
	if(!cfg_.plan_cache) return plan_launch(kernel, grid, block, work, args, ann);
	for(const auto& m : memos_) {
		std::pair<int64_t, int64_t> r;
		if(same_call(m, kernel, grid, block, work, args, ann) && replay(m, r)) return r;
	}
	const bool rec = work.size() <= kMemoMaxSuperblocks;
	const int64_t first = next_task_, chunks0 = next_chunk_;
	const uint64_t coll0 = collectives_;
	const size_t acc0 = accesses_.size();
	const auto tags0 = tags_;
	recording_ = rec;
	rec_chunks_.clear();
	rec_before_.clear();
	std::pair<int64_t, int64_t> r;
	try {
		r = plan_launch(kernel, grid, block, work, args, ann);
	} catch(...) {
		recording_ = false;
		throw;
	}
	recording_ = false;
	if(!rec || next_chunk_ != chunks0 || collectives_ != coll0 || rec_chunks_.empty()) return r;
	launch_memo m;
	m.kernel = kernel;
	m.grid = grid;
	m.block = block;
	m.work = work;
	m.args = args;
	m.ann = &ann;
	m.first = first;
	for(int64_t id = first; id < next_task_; ++id) m.tasks.push_back(plan_[static_cast<size_t>(id - plan_base_)]);
	m.tags_before = tags0;
	for(const auto& [pair, n] : tags_) {
		const auto b = tags0.find(pair);
		const uint64_t used = n - (b == tags0.end() ? 0 : b->second);
		if(used) m.tags_used[pair] = used;
	}
	m.chunks = rec_chunks_;
	m.before = std::move(rec_before_);
	for(const auto c : m.chunks) m.after.push_back(deps_.save(c));
	if(cfg_.record_accesses) m.accesses.assign(accesses_.begin() + static_cast<std::ptrdiff_t>(acc0), accesses_.end());
	rec_before_.clear();
	// several memos per call are kept: a loop that interleaves other requests every few launches
	// repeats its states with a longer period than the call sequence itself
	memos_.push_front(std::move(m));
	if(memos_.size() > kMemos) memos_.pop_back();
	return r;
}

std::pair<int64_t, int64_t> planner::plan_launch(const std::string& kernel, const box& grid, const point& block, const std::vector<superblock>& work,
    const std::vector<launch_arg>& args, const annotation& ann) {
	const int64_t first = next_task_;
	const kernel_entry* kdef = find_kernel(kernel);
	if(!kdef) throw plan_error("unknown kernel \"" + kernel + "\"");
	const kernel_entry& def = *kdef;
	const size_t np = def.params.size();

	// signature checks (planner.cpp:163-213)
	if(args.size() != np)
		throw validation_error("kernel \"" + kernel + "\" takes " + std::to_string(np) + " arguments, got " + std::to_string(args.size()));
	for(int k = 0; k < grid.rank(); ++k)
		if(grid.lo[k] != 0) throw validation_error("launch grids start at the origin");
	if(grid.is_empty()) throw validation_error("launch grid is empty");
	if(block.rank != grid.rank()) throw validation_error("block size and grid axis counts differ");

	std::vector<bound_param> bound(np);
	std::vector<bool> is_array(np, false);
	for(size_t i = 0; i < np; ++i) {
		const auto& p = def.params[i];
		const auto& a = args[i];
		if(!p.is_array) {
			const bool want_int = dtype_integral(p.type);
			if(want_int && a.kind != launch_arg::int_k) throw validation_error("parameter \"" + p.name + "\" expects an integer scalar");
			if(!want_int && a.kind != launch_arg::float_k) throw validation_error("parameter \"" + p.name + "\" expects a float scalar");
			continue;
		}
		if(a.kind != launch_arg::array_k) throw validation_error("parameter \"" + p.name + "\" expects an array");
		const array_rec& h = array(a.array);
		if(h.type != p.type)
			throw validation_error("parameter \"" + p.name + "\" expects element type " + dtype_name(p.type) + ", array has " + dtype_name(h.type));
		if(h.domain.rank() != p.rank) throw validation_error("parameter \"" + p.name + "\" expects rank " + std::to_string(p.rank));
		const access_decl* acc = ann.find(p.name);
		if(!acc) throw validation_error("annotation does not mention array parameter \"" + p.name + "\"");
		bound[i] = bound_param{i, a.array, acc, static_cast<size_t>(acc - ann.accesses.data())};
		is_array[i] = true;
	}
	for(const auto& acc : ann.accesses) {
		bool found = false;
		for(size_t i = 0; i < np && !found; ++i) found = is_array[i] && def.params[i].name == acc.argument;
		if(!found) throw validation_error("annotation mentions \"" + acc.argument + "\" which is not an array parameter");
	}
	for(size_t i = 0; i < np; ++i) {
		if(!is_array[i]) continue;
		for(size_t j = 0; j < np; ++j) {
			if(j == i || !is_array[j] || bound[j].array != bound[i].array) continue;
			const auto& m = bound[i].acc->mode;
			if(m.writes() || m.reduces())
				throw validation_error("one array is bound to several parameters and \"" + def.params[i].name + "\" writes or reduces into it");
		}
	}

	// superblocks in thread space (whole blocks; planner.cpp:216-234)
	point bext = point::zeros(grid.rank());
	for(int k = 0; k < grid.rank(); ++k) {
		if(block[k] <= 0) throw validation_error("block size must be positive");
		bext[k] = (grid.extent(k) + block[k] - 1) / block[k];
	}
	validate_work(work, box::extents(bext));
	const size_t S = work.size();
	std::vector<box> sb_threads(S);
	for(size_t s = 0; s < S; ++s) {
		box t;
		t.lo = point::zeros(grid.rank());
		t.hi = point::zeros(grid.rank());
		for(int k = 0; k < grid.rank(); ++k) {
			t.lo[k] = work[s].blocks.lo[k] * block[k];
			t.hi[k] = work[s].blocks.hi[k] * block[k];
		}
		sb_threads[s] = t;
	}

	// access regions per superblock (annotation.cpp:464-517)
	const size_t A = ann.accesses.size();
	std::vector<const array_rec*> acc_array(A, nullptr);
	for(size_t i = 0; i < np; ++i)
		if(is_array[i]) acc_array[bound[i].access_index] = &array(bound[i].array);
	std::vector<box> regions(S * A);
	std::vector<span> env(ann.vars.size() + 1);
	for(size_t s = 0; s < S; ++s) {
		make_env(ann, sb_threads[s], block, env.data());
		for(size_t a = 0; a < A; ++a) regions[s * A + a] = eval_access(ann.accesses[a], env.data(), acc_array[a]->domain);
	}

	// overlapping plain writes between superblocks are a plan error (annotation.cpp:524-538)
	for(size_t a = 0; a < A; ++a) {
		const auto& m = ann.accesses[a].mode;
		if(!m.writes() || m.reduces()) continue;
		std::vector<size_t> order;
		for(size_t s = 0; s < S; ++s)
			if(!regions[s * A + a].is_empty()) order.push_back(s);
		std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return regions[x * A + a].lo[0] < regions[y * A + a].lo[0]; });
		for(size_t x = 0; x < order.size(); ++x) {
			const box& rx = regions[order[x] * A + a];
			for(size_t y = x + 1; y < order.size() && regions[order[y] * A + a].lo[0] < rx.hi[0]; ++y) {
				const box ov = intersect(rx, regions[order[y] * A + a]);
				if(!ov.is_empty())
					throw plan_error("write conflict: superblocks " + std::to_string(std::min(order[x], order[y])) + " and "
					                 + std::to_string(std::max(order[x], order[y])) + " both write \"" + ann.accesses[a].argument + "\" on " + to_string(ov));
			}
		}
	}

	// launch-wide bounding box per reduce access
	std::vector<box> rbox(A);
	for(size_t a = 0; a < A; ++a) {
		if(!ann.accesses[a].mode.reduces()) continue;
		box b = box::empty(acc_array[a]->domain.rank());
		for(size_t s = 0; s < S; ++s) b = hull(b, regions[s * A + a]);
		rbox[a] = b;
	}

	struct partial {
		int64_t chunk, producer;
	};
	std::vector<std::vector<partial>> partials(A);
	std::vector<int> cand;

	struct rec_t {
		int64_t chunk;
		bool write;
		bool check;
		box region;
	};
	struct write_t {
		size_t access;
		box region;
		int64_t source;
		bool temp;
	};
	// per-superblock scratch, reused
	std::vector<rec_t> recs;
	std::vector<write_t> writes;
	std::vector<int64_t> dead;
	std::vector<std::pair<size_t, int64_t>> sb_partials;
	for(size_t s = 0; s < S; ++s) {
		const device_id dev = work[s].device;
		const int worker = dev.worker;
		std::vector<arg_bind> binds(np);
		std::vector<int64_t> exec_deps;
		exec_deps.reserve(8);
		recs.clear();
		writes.clear();
		dead.clear();
		sb_partials.clear();

		for(size_t i = 0; i < np; ++i) {
			const auto& p = def.params[i];
			if(!p.is_array) {
				binds[i].kind = dtype_integral(p.type) ? arg_kind::scalar_int : arg_kind::scalar_float;
				binds[i].i = args[i].i;
				binds[i].f = args[i].f;
				continue;
			}
			const bound_param& bp = bound[i];
			const access_mode mode = bp.acc->mode;
			const box& region = regions[s * A + bp.access_index];
			const array_rec& h = array(bp.array);

			if(mode.reduces()) {
				const box& b = rbox[bp.access_index];
				if(b.is_empty()) continue;
				const int64_t part = new_temp(b, dev, h.type);
				const int64_t create = emit_create(worker, dev, part, fill_kind::identity, mode.op);
				touch(part, create);
				exec_deps.push_back(create);
				binds[i].kind = arg_kind::chunk;
				binds[i].chunk = part;
				binds[i].region = b;
				binds[i].access = 3;
				sb_partials.emplace_back(bp.access_index, part);
				continue;
			}
			if(region.is_empty()) continue;

			h.index.query(region, cand);
			const int enc = select_enclosing(h.chunks, cand, region, dev);
			if(enc >= 0 && h.chunks[static_cast<size_t>(enc)].home == dev) {
				const int64_t cid = h.chunks[static_cast<size_t>(enc)].id;
				binds[i].kind = arg_kind::chunk;
				binds[i].chunk = cid;
				binds[i].region = region;
				binds[i].access = static_cast<int8_t>((mode.reads() ? 1 : 0) | (mode.writes() ? 2 : 0));
				recs.push_back({cid, mode.writes(), mode.reads(), region});
				if(mode.writes()) writes.push_back({bp.access_index, region, cid, false});
				continue;
			}
			// stage a temporary on the executing device, pulled from the enclosing replica or
			// assembled from every intersecting fragment (planner.cpp:324-347)
			const int64_t temp = new_temp(region, dev, h.type);
			const int64_t create = emit_create(worker, dev, temp, fill_kind::none, reduce_op::plus);
			touch(temp, create);
			exec_deps.push_back(create);
			if(mode.reads()) {
				std::vector<int> sources;
				if(enc >= 0)
					sources.push_back(enc);
				else
					sources = cand;
				for(const int src : sources) {
					const auto& sc = h.chunks[static_cast<size_t>(src)];
					exec_deps.push_back(transfer(sc.id, temp, intersect(sc.region, region), {}, {create}));
				}
			}
			binds[i].kind = arg_kind::chunk;
			binds[i].chunk = temp;
			binds[i].region = region;
			binds[i].access = static_cast<int8_t>((mode.reads() ? 1 : 0) | (mode.writes() ? 2 : 0));
			if(mode.writes())
				writes.push_back({bp.access_index, region, temp, true});
			else
				dead.push_back(temp);
		}

		const int64_t exec_tid = next_task_;
		for(const auto& r : recs) record(r.chunk, exec_tid, r.write, r.region, r.check, exec_deps);
		task e;
		e.worker = worker;
		e.resource = dev;
		e.kind = task_kind::execute;
		e.deps = std::move(exec_deps);
		e.kern = kdef;
		e.device = dev;
		e.sb_blocks = work[s].blocks;
		e.sb_threads = sb_threads[s];
		e.sb_inside_grid = encloses(grid, sb_threads[s]);
		e.block_size = block;
		e.args = std::move(binds);
		const int64_t exec_id = emit(std::move(e));
		for(const auto& b : plan_.back().args)
			if(b.kind == arg_kind::chunk && chunk(b.chunk).temp) touch(b.chunk, exec_id);
		for(const auto& [a, part] : sb_partials) partials[a].push_back({part, exec_id});

		// propagate written regions into every other overlapping replica; scatter temps
		for(const auto& w : writes) {
			const array_rec& h = *acc_array[w.access];
			h.index.query(w.region, cand);
			for(const int t : cand) {
				const auto& target = h.chunks[static_cast<size_t>(t)];
				if(!w.temp && target.id == w.source) continue;
				transfer(w.source, target.id, intersect(target.region, w.region), {exec_id}, {});
			}
			if(w.temp) dead.push_back(w.source);
		}
		for(const int64_t t : dead) emit_delete_temp(worker, dev, t);
	}

	// hierarchical reduction: device -> worker -> root w0d0 -> destination chunks
	for(size_t a = 0; a < A; ++a) {
		const auto& acc = ann.accesses[a];
		if(!acc.mode.reduces() || partials[a].empty()) continue;
		const box b = rbox[a];
		const array_rec& h = *acc_array[a];
		const dtype type = h.type;
		const reduce_op op = acc.mode.op;
		std::vector<int64_t> temps;
		for(const auto& p : partials[a]) temps.push_back(p.chunk);

		const auto emit_reduce = [&](int worker, device_id dev, const std::vector<partial>& in) -> partial {
			const int64_t out = new_temp(b, dev, type);
			temps.push_back(out);
			const int64_t create = emit_create(worker, dev, out, fill_kind::none, reduce_op::plus);
			touch(out, create);
			task r;
			r.worker = worker;
			r.resource = dev;
			r.kind = task_kind::reduce;
			r.op = op;
			r.output = out;
			r.deps.reserve(in.size() + 1);
			r.inputs.reserve(in.size());
			r.deps.push_back(create);
			for(const auto& p : in) {
				r.inputs.push_back(p.chunk);
				r.deps.push_back(p.producer);
			}
			const int64_t rid = emit(std::move(r));
			for(const auto& p : in) touch(p.chunk, rid);
			touch(out, rid);
			return {out, rid};
		};

		std::map<device_id, std::vector<partial>> by_dev;
		for(const auto& p : partials[a]) by_dev[chunk(p.chunk).desc.home].push_back(p);
		std::map<device_id, partial> dev_result;
		for(const auto& [dev, parts] : by_dev) dev_result[dev] = parts.size() == 1 ? parts[0] : emit_reduce(dev.worker, dev, parts);

		std::map<int, std::vector<partial>> by_worker;
		for(const auto& [dev, res] : dev_result) by_worker[dev.worker].push_back(res);
		std::map<int, partial> worker_result;
		for(const auto& [w, res] : by_worker) worker_result[w] = res.size() == 1 ? res[0] : emit_reduce(w, chunk(res[0].chunk).desc.home, res);

		if(cfg_.collective_reduce && cfg_.workers > 1) {
			// every worker joins one allreduce group, in place on its worker result (an
			// identity-filled box for a worker without partials), then copies the total into
			// its own destination chunks; members with data are listed in worker order, the
			// order of the reference's root reduce, so an in-process combine is bit-identical
			std::vector<partial> member(static_cast<size_t>(cfg_.workers));
			std::vector<int64_t> data;
			for(int w = 0; w < cfg_.workers; ++w) {
				const auto it = worker_result.find(w);
				if(it != worker_result.end()) {
					member[static_cast<size_t>(w)] = it->second;
					data.push_back(it->second.chunk);
					continue;
				}
				const device_id home{w, 0};
				const int64_t filler = new_temp(b, home, type);
				temps.push_back(filler);
				const int64_t create = emit_create(w, home, filler, fill_kind::identity, op);
				touch(filler, create);
				member[static_cast<size_t>(w)] = {filler, create};
			}
			const uint64_t group = collectives_++;
			std::vector<int64_t> ar(static_cast<size_t>(cfg_.workers));
			for(int w = 0; w < cfg_.workers; ++w) {
				const partial& m = member[static_cast<size_t>(w)];
				task r;
				r.worker = w;
				r.resource = chunk(m.chunk).desc.home;
				r.kind = task_kind::allreduce;
				r.op = op;
				r.tag = group;
				r.inputs = data;
				r.output = m.chunk;
				r.type = type;
				r.region = b;
				r.deps.push_back(m.producer);
				ar[static_cast<size_t>(w)] = emit(std::move(r));
				touch(m.chunk, ar[static_cast<size_t>(w)]);
			}
			h.index.query(b, cand);
			for(const int t : cand) {
				const auto& target = h.chunks[static_cast<size_t>(t)];
				const int w = target.home.worker;
				transfer(member[static_cast<size_t>(w)].chunk, target.id, intersect(target.region, b), {ar[static_cast<size_t>(w)]}, {});
			}
			for(const int64_t id : temps) {
				const device_id home = chunk(id).desc.home;
				emit_delete_temp(home.worker, home, id);
			}
			continue;
		}

		const device_id root{0, 0};
		std::vector<int64_t> final_inputs, final_deps;
		for(const auto& [w, res] : worker_result) {
			if(w == 0) {
				final_inputs.push_back(res.chunk);
				final_deps.push_back(res.producer);
				continue;
			}
			const int64_t landing = new_temp(b, root, type);
			temps.push_back(landing);
			const int64_t create = emit_create(0, root, landing, fill_kind::none, reduce_op::plus);
			touch(landing, create);
			final_inputs.push_back(landing);
			final_deps.push_back(transfer(res.chunk, landing, b, {res.producer}, {create}));
		}
		const int64_t fin = new_temp(b, root, type);
		temps.push_back(fin);
		const int64_t fin_create = emit_create(0, root, fin, fill_kind::none, reduce_op::plus);
		touch(fin, fin_create);
		final_deps.push_back(fin_create);
		task r;
		r.worker = 0;
		r.resource = root;
		r.kind = task_kind::reduce;
		r.op = op;
		r.inputs = final_inputs;
		r.output = fin;
		r.deps = std::move(final_deps);
		const int64_t fin_id = emit(std::move(r));
		for(const auto in : final_inputs) touch(in, fin_id);
		touch(fin, fin_id);

		h.index.query(b, cand);
		for(const int t : cand) {
			const auto& target = h.chunks[static_cast<size_t>(t)];
			transfer(fin, target.id, intersect(target.region, b), {fin_id}, {});
		}
		for(const int64_t id : temps) {
			const device_id home = chunk(id).desc.home;
			emit_delete_temp(home.worker, home, id);
		}
	}
	return {first, next_task_};
}

namespace {

// a minus b as disjoint boxes (slab by slab along each axis)
void subtract(const box& a, const box& b, std::vector<box>& out) {
	if(!overlaps(a, b)) {
		out.push_back(a);
		return;
	}
	box rest = a;
	for(int k = 0; k < a.rank(); ++k) {
		if(rest.lo[k] < b.lo[k]) {
			box s = rest;
			s.hi[k] = b.lo[k];
			out.push_back(s);
			rest.lo[k] = b.lo[k];
		}
		if(rest.hi[k] > b.hi[k]) {
			box s = rest;
			s.lo[k] = b.hi[k];
			out.push_back(s);
			rest.hi[k] = b.hi[k];
		}
	}
}

} // namespace

std::pair<int64_t, int64_t> planner::host_transfer(int64_t array_id, uint64_t host_addr, bool write, const box* host_box) {
	const array_rec& a = array(array_id);
	// the host array covers `host_box` (default: the whole domain). The tasks do not depend on
	// it, so ranks of a one-process-per-GPU job that each pass their own box and buffer still
	// plan identical task sequences; a task's region must lie inside the box on the rank that
	// executes it (checked by the executor)
	const int64_t first = next_task_;
	std::vector<box> covered;
	for(const auto& c : a.chunks) {
		std::vector<box> parts{c.region};
		if(!write) {
			for(const auto& done : covered) {
				std::vector<box> next;
				for(const auto& part : parts) subtract(part, done, next);
				parts.swap(next);
			}
			covered.push_back(c.region);
		}
		for(const auto& r : parts) {
			if(r.is_empty()) continue;
			const int64_t tid = next_task_;
			std::vector<int64_t> d;
			record(c.id, tid, write, r, !write, d);
			task t;
			t.worker = c.home.worker;
			t.resource = c.home;
			t.kind = write ? task_kind::host_write : task_kind::host_read;
			t.deps = std::move(d);
			t.chunk = c.id;
			t.region = r;
			t.src_region = host_box ? *host_box : a.domain;
			t.type = a.type;
			t.tag = host_addr;
			emit(std::move(t));
		}
	}
	return {first, next_task_};
}

} // namespace mtb
