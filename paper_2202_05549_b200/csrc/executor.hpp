// GPU executor: the B200 replacement for the reference's system_runtime
// (proj/src/runtime.cpp:99-717).
//
// The reference runs one scheduler thread per worker that counts dependencies, stages chunks
// through the memory manager and hands kernel bodies to one CPU thread per device. On B200 the
// dependency DAG is resolved by the hardware instead: tasks arrive in id order (every
// dependency points backwards, planner.cpp:35-40), each task is enqueued immediately on a CUDA
// stream of its device, every dependency on another stream becomes a cudaStreamWaitEvent and
// every task records one event. submit() therefore returns as soon as the work is queued, so
// planning of launch n+1 overlaps execution of launch n with no host scheduler in the loop.
//
// Chunk store: per-GPU stream-ordered pool (cudaMallocFromPoolAsync / cudaFreeAsync), so a
// chunk's allocation, fill, uses and release are all ordered on-device; fill_spec none is
// zero-filled like the reference's std::vector::resize (SURVEY finding 4). Copies are
// cudaMemcpy3D(Peer)Async over NVLink; send/recv pairs go through device message buffers
// matched by (src worker, dst worker, tag); reduce tasks are one combine kernel reading its
// inputs (peer memory where needed) in the reference's input order.
#pragma once

#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <string>
#include <tuple>
#include <cstdlib>
#include <nvtx3/nvtx3.hpp>
#include <unordered_map>
#include <vector>

#include "plan.hpp"
#include "registry.hpp"

namespace mtb {

// NVTX ranges (tracing): planning of each launch, each flush, and the host-side issue
// of every task by kind, in the "manta-b200" domain. Header-only NVTX 3; no cost without a tool.
struct nvtx_domain {
	static constexpr char const* name{"manta-b200"};
};

struct executor_config {
	int workers = 1;
	int devices_per_worker = 1;
	int num_gpus = 0;            // 0: all visible
	int streams_per_device = 4;
	uint64_t device_capacity = 0; // 0: 90% of free memory at start
	uint64_t host_capacity = 0;   // pinned-host spill tier; 0 disables spilling
	int lookahead = 512;          // spill tier: tasks held back so eviction can see future uses
	int first_worker = 0;         // workers [first, first+local) execute here (multi-process)
	int gpu_base = 0;             // first CUDA device ordinal this executor uses
	int local_workers = -1;       // -1: all workers
	uint64_t disk_capacity = 0;   // disk tier below the host tier (0: none)
	uint64_t staging_threshold = 0; // throttle: bytes of chunks in use by in-flight tasks per device (0: off)
	std::string spill_dir;        // spill file directory ("" = system temp directory)
	uint64_t schedule_seed = 0;   // != 0: randomised stream choice + delays (reference ready_seed)
};

struct exec_counters {
	uint64_t tasks = 0;
	uint64_t kernels = 0; // device launches issued by execute/reduce/fill
	uint64_t copies = 0;
	uint64_t bytes_copied = 0;
	uint64_t bytes_sent = 0;
	uint64_t bytes_received = 0;
	uint64_t peak_device_bytes = 0;
	uint64_t evictions = 0;
	uint64_t bytes_device_to_host = 0;
	uint64_t bytes_host_to_device = 0;
	uint64_t dead_drops = 0; // evictions that skipped the write-back (data dead ahead)
	uint64_t dead_skips = 0; // restores that skipped the H2D (data overwritten before read)
	uint64_t host_reclaims = 0; // host copies of resident chunks taken back when the host tier is full
	uint64_t bytes_host_in = 0, bytes_host_out = 0; // host_write / host_read tasks
	uint64_t graph_captures = 0, graph_replays = 0;  // CUDA-graph replay of repeated submissions
	uint64_t bytes_host_to_disk = 0, bytes_disk_to_host = 0; // disk tier
	uint64_t messages = 0;    // inter-process send + recv tasks
	uint64_t message_ops = 0; // stream operations (kernels, copies, allocations) they enqueued
	uint64_t fused_copies = 0, bytes_fused = 0; // copy tasks stored by their producing kernel
};

class executor {
  public:
	explicit executor(const executor_config& cfg);
	~executor();
	executor(const executor&) = delete;
	executor& operator=(const executor&) = delete;

	void submit(const std::vector<task>& tasks);
	// the same one task at a time: submit_one for each (ascending ids), then end_submit
	void submit_one(const task& t);
	void end_submit();
	void sync();
	// host transfers: `host` holds the row-major box `host_box`; `region` is copied. Both
	// synchronise the chunk's GPU first (call after the tasks that produce the data).
	void download(int64_t chunk, void* host, const box& host_box, const box& region);
	void upload(int64_t chunk, const void* host, const box& host_box);
	bool has_chunk(int64_t chunk) const { return bufs_.count(chunk) != 0; }
	std::string report_json(); // waits for traced tasks' end events
	const exec_counters& counters() const { return ctr_; }
	// per worker, the fields of the reference's run_report memory counters (runtime.cpp:613-636)
	struct worker_counters {
		uint64_t evictions = 0, bytes_device_to_host = 0, bytes_host_to_device = 0, bytes_host_to_disk = 0, bytes_disk_to_host = 0;
		uint64_t bytes_sent = 0, bytes_received = 0, staging_checks = 0, staging_violations = 0;
	};
	const worker_counters& worker_stats(int w) const { return wctr_.at(static_cast<size_t>(w)); }

	// stream of the most recent execute on a chunk's device (bench timing hook)
	cudaStream_t last_exec_stream() const { return last_exec_stream_; }
	int gpu_of(device_id d) const;

	// Device-side timing. mark(0)/mark(1) record, on every GPU, an event that completes when
	// all work enqueued so far (every stream) has completed; elapsed_ms() is the max over
	// GPUs of mark(1) - mark(0).
	void mark(int slot);
	double elapsed_ms();
	// Per-kernel event timing on the launching stream (bench roofline): when enabled every
	// execute task's launcher call is bracketed by timing events.
	void set_profile(bool on) { profile_ = on; }
	// per-task device timestamps for report_json (the reference's run_report task records,
	// runtime.cpp:389, :514-525): a timing event after a task's dependency waits and one after
	// its work, both on its stream; times are ns since tracing was switched on
	void set_trace(bool on);
	void kernel_time(const std::string& kernel, int64_t* count, double* total_ms);

	// One process per worker: GPU-driven point-to-point messaging for send/recv tasks whose
	// peer worker runs in another process. Every rank exports one IPC-mapped mailbox (a ring of
	// kSlots x kSlotBytes per source rank, ready flags, consumption counters); after the blobs
	// are exchanged out of band (torch.distributed), each rank maps every peer's mailbox.
	// allreduce tasks between processes run on an NCCL communicator (libnccl loaded at run
	// time: the one already in the process, else `lib`, else the default search path)
	void nccl_unique_id(const char* lib, void* id128);
	void nccl_init(const char* lib, const void* id128, int nranks, int rank);

	std::vector<uint8_t> peer_export();
	void peer_import(const std::vector<std::vector<uint8_t>>& blobs);
	static constexpr int kSlots = 4;
	static constexpr uint64_t kSlotBytes = 16ull << 20;

  private:
	struct buffer {
		void* ptr = nullptr; // device copy (null while evicted)
		uint64_t bytes = 0;
		box region;
		dtype type = dtype::f32;
		device_id home;
		int gpu = 0;
		// spill tier
		void* host = nullptr;     // pinned host copy
		bool host_valid = false;  // host copy equals the device contents
		std::vector<int64_t> users; // tasks that touched the device copy since it became resident
		int64_t disk_off = -1;    // spill-file block holding a copy (disk tier)
		bool disk_valid = false;  // that copy equals the current contents
		cudaEvent_t restored = nullptr; // completes when the last H2D restore has landed
		cudaEvent_t evicted = nullptr;  // completes when the last eviction's D2H has landed
		uint64_t last_use = 0;
	};
	struct ldev {
		int gpu = 0;
		std::vector<cudaStream_t> compute;
		cudaStream_t copy = nullptr;
		cudaStream_t recv = nullptr; // inter-process receives (never queued behind a spinning send)
		cudaStream_t host_in = nullptr, host_out = nullptr; // host_write / host_read tasks (both PCIe directions at once)
		size_t rr = 0;
	};
	struct peer_link {
		char* tx_ring = nullptr;              // my ring inside the peer's mailbox
		uint64_t* tx_ready = nullptr;         // ready flags for my segments (peer memory)
		uint64_t* tx_consumed = nullptr;      // peer's consumption of my segments (my memory)
		uint64_t tx_seq = 0;
		char* rx_ring = nullptr;              // the peer's ring inside my mailbox
		uint64_t* rx_ready = nullptr;         // its ready flags (my memory)
		uint64_t* rx_consumed = nullptr;      // my consumption of its segments (peer memory)
		uint64_t rx_seq = 0;
		cudaStream_t tx = nullptr, rx = nullptr; // per-peer streams: a send waiting for ring space
		                                         // never holds up other copies or other peers
		unsigned* tx_done = nullptr;          // CTA completion counters of the fused kernels (my memory)
		unsigned* rx_done = nullptr;
	};
	unsigned* link_ctr_ = nullptr;
	char* mbox_ = nullptr;
	int world_ = 0;
	int my_rank_ = -1;
	std::vector<peer_link> links_;
	std::vector<void*> opened_;
	bool remote_worker(int w) const { return cfg_.local_workers >= 0 && (w < cfg_.first_worker || w >= cfg_.first_worker + cfg_.local_workers); }
	void remote_send(const task& t);
	void remote_recv(const task& t);
	struct gpu_res {
		int ordinal = 0;
		cudaMemPool_t pool = nullptr;
		uint64_t used = 0;
		uint64_t capacity = 0;
		cudaStream_t service = nullptr; // message-buffer releases
		cudaStream_t timing = nullptr;
		cudaStream_t graph = nullptr; // launches of replayed submissions (CUDA graphs)
		cudaStream_t h2d = nullptr, d2h = nullptr; // spill tier
		std::deque<cudaEvent_t> frees;             // one event per eviction (after its D2H + free), oldest first
		cudaEvent_t marks[2] = {nullptr, nullptr};
	};
	struct kernel_timing {
		std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
		int64_t count = 0;
		double total_ms = 0.0;
	};
	struct done_ev {
		cudaEvent_t ev = nullptr;
		cudaStream_t stream = nullptr;
		int gpu = 0;
	};
	struct message {
		void* ptr = nullptr;
		uint64_t bytes = 0;
		int gpu = 0;
		cudaEvent_t ready = nullptr;
	};

	executor_config cfg_;
	std::vector<gpu_res> gpus_;
	std::vector<worker_counters> wctr_;        // per worker
	std::vector<uint64_t> dev_used_, dev_peak_; // per logical device (worker-major): chunk bytes by home
	worker_counters& wc(int worker) { return wctr_[static_cast<size_t>(worker)]; }
	void charge(const buffer& b, uint64_t bytes, bool add); // device bytes of a chunk (GPU pool + its home device)
	// staging throttle + monitor (memory.cpp:290-295, 371-374): per logical device, the chunks
	// used by issued tasks that have not completed, with their bytes; a task whose chunks would
	// push the union past the threshold waits (on the host) for the oldest in-flight tasks
	struct staged_task {
		int64_t id;
		size_t dev;
		std::vector<std::pair<int64_t, uint64_t>> chunks;
	};
	std::deque<staged_task> staged_;
	std::vector<std::unordered_map<int64_t, int>> pins_;
	std::vector<uint64_t> pinned_bytes_;
	void throttle(const task& t);
	void unpin(const staged_task& s);
	std::vector<ldev> ldevs_; // worker-major
	std::unordered_map<int64_t, buffer> bufs_;
	std::unordered_map<int64_t, done_ev> done_;
	std::unordered_map<cudaStream_t, int64_t> tail_;
	std::map<std::tuple<int, int, uint64_t>, message> mailbox_;
	std::vector<std::vector<cudaEvent_t>> free_events_; // per GPU
	int64_t last_id_ = -1;
	exec_counters ctr_;
	cudaStream_t last_exec_stream_ = nullptr;
	bool profile_ = false;
	struct trace_rec {
		int64_t id;
		int worker;
		task_kind kind;
		int gpu;
		cudaEvent_t t0 = nullptr, t1 = nullptr;
	};
	bool trace_ = false;
	std::vector<trace_rec> trace_recs_;
	std::unordered_map<int64_t, size_t> trace_open_;
	std::vector<cudaEvent_t> trace_base_; // per executor GPU
	std::map<std::string, kernel_timing> ktimes_;

	// ---- CUDA-graph replay of repeated submissions --------------------------------------
	// Iterative programs submit the same task pattern again and again (a heat step a->b, then
	// b->a, ...). When a submission (the tasks of one mt_flush) consists only of execute / copy
	// tasks on one GPU, no spill tier, tracing or kernel profiling is active, and its signature
	// (kinds, kernels, chunk ids, regions, arguments, intra-submission dependencies) has been seen
	// before, its GPU work is captured once into a CUDA graph (stream capture forked over the
	// device's streams, so the graph keeps the DAG's concurrency) and from then on each
	// occurrence is one cudaGraphLaunch after waiting for its external dependencies. All tasks
	// of a replay complete on one event (reference counted in shared_ev_). MTB_NO_GRAPHS=1
	// disables it.
	struct graph_entry {
		cudaGraphExec_t exec = nullptr;
		int gpu = 0;
		int64_t tasks = 0, kernels = 0, copies = 0, fused_copies = 0;
		uint64_t bytes_copied = 0, bytes_fused = 0;
	};
	bool graphs_on_ = std::getenv("MTB_NO_GRAPHS") == nullptr;
	bool capturing_ = false;
	int64_t capture_first_ = -1;
	std::vector<task> gbatch_; // buffered tasks of the current submission (graph mode)
	std::unordered_map<std::string, graph_entry> graphs_;
	std::unordered_map<std::string, int> sig_seen_;
	std::unordered_map<cudaEvent_t, int> shared_ev_;
	bool graph_eligible(const std::vector<task>& b, int* gpu) const;
	std::string signature(const std::vector<task>& b) const;
	bool capture(const std::vector<task>& b, int gpu, graph_entry& out);
	void replay(const graph_entry& g, const std::vector<task>& b);
	void release_done_event(cudaEvent_t ev, int gpu);
	void issue_batch();

	// ---- halo copies fused into the producing kernel ---------------------------------------
	// In a submission, a copy task C whose source region the preceding execute task E writes
	// (C depends on E, E's kernel declares a mirror param, every other dependency of C is older
	// than E, and C's destination chunk lives on E's GPU or a peer-accessible one) is handed to
	// E's launcher as a mirror: the kernel stores those output cells a second time, straight into
	// the destination chunk. E then also waits for C's other dependencies, and C completes with E.
	// A launcher that cannot apply a mirror leaves it, and C is issued as an ordinary copy.
	// Off under spill, tracing, staging throttle or schedule perturbation; MTB_NO_HALO_FUSION=1
	// disables it.
	bool fusion_on_ = std::getenv("MTB_NO_HALO_FUSION") == nullptr || std::atoi(std::getenv("MTB_NO_HALO_FUSION")) == 0;
	std::unordered_map<int64_t, std::vector<const task*>> mirror_plan_; // E id -> copies
	std::unordered_map<int64_t, int> mirrored_;                         // fused copy ids
	std::vector<char> peer_ok_;                                          // [a * ngpus + b]
	void plan_mirrors(const std::vector<task>& b);

	// ---- disk tier (memory.cpp:85-159): host copies of evicted chunks move to a spill file when
	// the pinned-host tier is full, and come back through a pinned block on restore
	int spill_fd_ = -1;
	std::string spill_path_;
	uint64_t disk_end_ = 0;
	std::multimap<uint64_t, uint64_t> disk_free_; // block size -> offset
	uint64_t disk_alloc(uint64_t bytes);
	void disk_release(buffer& b);
	void* spill_host_to_disk(uint64_t bytes, int64_t exclude);
	void disk_read(const buffer& b, void* dst);

	ldev& dev(device_id d);
	int ord(int gpu_index) const { return gpus_[static_cast<size_t>(gpu_index)].ordinal; }
	cudaEvent_t take_event(int gpu);
	void wait_deps(const task& t, cudaStream_t s);
	cudaStream_t pick_compute(const task& t, ldev& L);
	// schedule perturbation (cfg.schedule_seed): a random on-device delay before a task
	uint64_t rng_state_ = 0;
	uint64_t next_random();
	void perturb(cudaStream_t s);
	void finish(const task& t, cudaStream_t s);
	void retire_completed();
	buffer& buf(int64_t chunk);

	// spill tier (active when cfg.host_capacity > 0)
	bool spill_ = false;
	std::deque<task> queue_;
	std::vector<cudaEvent_t> stage_waits_;
	std::multimap<uint64_t, std::pair<void*, cudaEvent_t>> host_free_; // size -> (block, reusable-after event)
	uint64_t host_used_ = 0;
	uint64_t clock_ = 0;
	void issue(const task& t);
	void drain(bool all);
	void used_chunks(const task& t, std::vector<std::pair<int64_t, bool>>& out) const;
	struct access_t {
		int64_t chunk;
		box region;
		bool read;      // may read `region` (anything not a definite overwrite counts)
		bool overwrite; // definitely writes every cell of `region`
		bool kill;      // delete
	};
	void accesses_of(const task& t, std::vector<access_t>& out) const;
	// true when, in `first` (optional) followed by the queued tasks, every cell of the chunk
	// is overwritten (or the chunk deleted) before any of it is read
	bool dead_ahead(int64_t chunk, const task* first) const;
	void stage(const task& t);
	void note_use(const task& t);
	void ensure_room(int gpu, uint64_t bytes, const std::vector<int64_t>& pinned);
	void evict(int64_t chunk);
	void restore(int64_t chunk, const std::vector<int64_t>& pinned, const task& current);
	void* host_alloc(uint64_t bytes, int gpu, int64_t exclude);
	void host_release(void* p, uint64_t bytes, cudaEvent_t after);
	void alloc_wait(int gpu, cudaStream_t s);
	cudaEvent_t alloc_event(int gpu) const;

	void run_create(const task& t);
	void run_delete(const task& t);
	void run_execute(const task& t);
	void run_copy(const task& t);
	void run_send(const task& t);
	void run_recv(const task& t);
	void run_reduce(const task& t);
	void run_allreduce(const task& t);
	void run_host_io(const task& t);
	void finish_id(int64_t id, cudaStream_t s, int gpu);

	// in-process allreduce groups: members issue in worker order, the last one combines
	struct coll_group {
		std::vector<int64_t> tasks;
		std::vector<int64_t> outputs;
		std::vector<std::pair<cudaEvent_t, int>> ready; // (event, gpu index)
	};
	std::map<uint64_t, coll_group> groups_;
	void* nccl_dl_ = nullptr;
	void* nccl_comm_ = nullptr;
	void nccl_load(const char* lib);
};

// region copy helpers (rank <= 3, row-major chunks); enqueue on `s`. A gpu index of -1 marks
// a host buffer.
void copy_box(const void* src_base, const box& src_chunk, int src_gpu, void* dst_base, const box& dst_chunk, int dst_gpu, const box& region,
    size_t elem, cudaStream_t s);

// device fill of `count` elements with the fill value of (kind, op) for `type`
void device_fill(void* ptr, uint64_t count, dtype type, fill_kind kind, reduce_op op, cudaStream_t s);

// out = in[0]; out = op(out, in[k]) for k >= 1 (runtime.cpp:463-504 semantics)
void device_reduce(void* out, const void* const* inputs, int n, uint64_t count, dtype type, reduce_op op, cudaStream_t s);

void check_cuda(cudaError_t e, const char* what);

} // namespace mtb
