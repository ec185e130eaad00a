/*
 * manta_b200.h — C-ABI of the B200-native distributed-launch runtime.
 *
 * This is the drop-in boundary for the reference's hot path (Lightning / "manta",
 * /root/reference/proj). The reference exposes three C++ interfaces on this path and
 * no FFI; each block below replaces one of them with plain C types (no torch, no STL):
 *
 *   driver (planner)      proj/include/manta/planner.hpp:51-78
 *       mt_ctx_create / mt_array_create / mt_array_delete / mt_launch / mt_plan_export
 *   system_runtime        proj/include/manta/runtime.hpp:70-98
 *       mt_exec_create / mt_exec_submit / mt_exec_sync / mt_exec_read_chunk / mt_exec_report_json
 *   distributions         proj/include/manta/distribution.hpp:62-92
 *       mt_dist_tile / mt_dist_replicated / mt_dist_single / mt_work_block
 *   kernel plugin API     proj/include/manta/kernels.hpp:75-105
 *       mt_kernel_register / mt_kernel_count / mt_kernel_info
 *   errors                proj/include/manta/errors.hpp:9-35
 *       every call returns MT_OK or one of the MT_E* codes; mt_last_error() returns the
 *       message of the calling thread's last failure (parse errors carry line:col).
 *
 * The oracle shim (oracle/ref_shim.cpp) exports the same entry points with the prefix
 * `mr_` over the unmodified reference, so tests drive both through one binding.
 */
#ifndef MANTA_B200_H
#define MANTA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MT_MAX_RANK 3
#define MT_KERNEL_NAME_MAX 64

/* ---- error codes (errors.hpp:9-35) ---------------------------------------------------- */
enum mt_status {
	MT_OK = 0,
	MT_EPARSE = 1,      /* manta::parse_error      */
	MT_EVALIDATION = 2, /* manta::validation_error */
	MT_EPLAN = 3,       /* manta::plan_error       */
	MT_EEXEC = 4,       /* manta::execution_error  */
	MT_EINTERNAL = 5,   /* anything else (CUDA failure, bad handle) */
};

/* ---- element types (dtype.hpp:13; bf16 is a B200 extension for the tcgen05 matmul) --- */
enum mt_dtype { MT_I32 = 0, MT_I64 = 1, MT_F32 = 2, MT_F64 = 3, MT_BF16 = 4 };

/* ---- task IR (task.hpp:19-95) --------------------------------------------------------- */
enum mt_task_kind {
	MT_TASK_CREATE = 0,
	MT_TASK_DELETE = 1,
	MT_TASK_EXECUTE = 2,
	MT_TASK_COPY = 3,
	MT_TASK_SEND = 4,
	MT_TASK_RECV = 5,
	MT_TASK_REDUCE = 6,
	/* B200 extension (cfg.collective_reduce): one per worker, in place on `output`; the
	 * group is `tag`, its data-carrying members are `inputs` in worker order (a worker
	 * without a partial joins with an identity-filled buffer and is not in `inputs`) */
	MT_TASK_ALLREDUCE = 7,
	/* B200 extension (mt_array_write_async / mt_array_read_async): copy `region` of chunk
	 * `chunk` from / to the host array at address `tag` (row-major over `src_region`) */
	MT_TASK_HOST_WRITE = 8,
	MT_TASK_HOST_READ = 9,
};
enum mt_fill_kind { MT_FILL_NONE = 0, MT_FILL_ZERO = 1, MT_FILL_ONE = 2, MT_FILL_IDENTITY = 3 };
enum mt_reduce_op { MT_RED_PLUS = 0, MT_RED_TIMES = 1, MT_RED_MIN = 2, MT_RED_MAX = 3 };
enum mt_arg_kind { MT_ARG_INT = 0, MT_ARG_FLOAT = 1, MT_ARG_CHUNK = 2, MT_ARG_NONE = 3 };

/* Half-open box [lo, hi) (geometry.hpp:45-70). Also used for points (hi unused). */
typedef struct mt_rect {
	int32_t rank;
	int32_t pad_;
	int64_t lo[MT_MAX_RANK];
	int64_t hi[MT_MAX_RANK];
} mt_rect;

typedef struct mt_device {
	int32_t worker;
	int32_t device;
} mt_device;

typedef struct mt_chunk_desc {
	int64_t id;
	mt_rect region;
	mt_device home;
} mt_chunk_desc;

typedef struct mt_superblock {
	mt_rect blocks; /* thread-block index space */
	mt_device device;
} mt_superblock;

/* arg_binding (task.hpp:44-50) */
typedef struct mt_arg_binding {
	int32_t kind; /* mt_arg_kind */
	int32_t pad_;
	int64_t i;
	double f;
	int64_t chunk;
} mt_arg_binding;

/*
 * One task, flattened. Variable-length parts (deps, reduce inputs, execute args) live in
 * side pools and are referenced by (offset, count). Field use per kind:
 *   create : chunk, region, home, dtype, fill, fill_op
 *   delete : chunk
 *   execute: kernel, device, sb_blocks, sb_threads, block_size(.lo), args
 *   copy   : src, dst, src_region, dst_region
 *   send   : chunk, region, peer, tag          recv: chunk, region, peer, tag
 *   reduce : op, inputs, output
 *   allreduce: op, inputs (group members with data), output (this worker's member), tag (group)
 *   host_write / host_read: chunk, region (copied box), src_region (host array box),
 *            dtype, tag (host address)
 */
typedef struct mt_task {
	int64_t id;
	int32_t worker;
	int32_t kind; /* mt_task_kind */
	mt_device resource;
	int64_t deps_off;
	int64_t ndeps;
	int64_t chunk;
	mt_rect region;
	mt_device home;
	int32_t dtype;
	int32_t fill;
	int32_t fill_op;
	int32_t op;
	char kernel[MT_KERNEL_NAME_MAX];
	mt_device device;
	mt_rect sb_blocks;
	mt_rect sb_threads;
	mt_rect block_size;
	int64_t args_off;
	int64_t nargs;
	int64_t src;
	int64_t dst;
	mt_rect src_region;
	mt_rect dst_region;
	int32_t peer;
	int32_t pad_;
	uint64_t tag;
	int64_t inputs_off;
	int64_t ninputs;
	int64_t output;
} mt_task;

/* ---- launch arguments (planner.hpp:25-35) ------------------------------------------- */
enum mt_launch_arg_kind { MT_LARG_INT = 0, MT_LARG_FLOAT = 1, MT_LARG_ARRAY = 2 };
typedef struct mt_launch_arg {
	int32_t kind;
	int32_t pad_;
	int64_t i;
	double f;
	int64_t array;
} mt_launch_arg;

/* ---- configuration (planner.hpp:17-23, runtime.hpp:24-33, memory.hpp:43-55) -------- */
typedef struct mt_config {
	int32_t workers;
	int32_t devices_per_worker;
	int32_t suppress_conflict_deps; /* fault-injection hook (planner.hpp:20-22) */
	int32_t compat_deps;            /* 1: whole-chunk edges exactly as the reference */
	int32_t execute;                /* 0: plan only (no GPU needed); 1: run on GPUs    */
	int32_t num_gpus;               /* physical GPUs to map devices onto (0 = all)     */
	int32_t streams_per_device;     /* compute streams per logical device (0 = 4)      */
	int32_t single_worker;          /* 0: this process executes every worker; 1: only worker_rank
	                                   (one process per GPU; every rank plans the full plan) */
	uint64_t device_capacity;       /* bytes per device the chunk store may use (0 = 90% of free HBM) */
	uint64_t host_capacity;         /* pinned-host spill tier bytes (0 = no spill tier)  */
	uint64_t staging_threshold;     /* staging throttle (memory.cpp:290-295): per device, the bytes of chunks in use by
	                                   issued-but-unfinished tasks stay within it (the issuing thread waits for the
	                                   oldest in-flight tasks); a task above it alone is an execution error;
	                                   0 = off (no waiting, graph replay allowed) */
	int32_t record_accesses;        /* keep (task, chunk, region, write) records for mt_plan_accesses */
	int32_t lookahead_tasks;        /* spill tier: tasks buffered ahead for Belady eviction (0 = 512) */
	int32_t worker_rank;            /* with single_worker: the worker this process executes */
	int32_t gpu_base;               /* with single_worker: CUDA ordinal of this process's first GPU */
	int32_t collective_reduce;      /* 1: cross-worker reduce trees become one allreduce per worker
	                                   (NCCL between processes, a peer-memory combine in one process)
	                                   instead of send-to-root / root reduce / send-back
	                                   (planner.cpp:389-517); 0: the reference's tree */
	int32_t drop_executed_tasks;    /* 1: forget tasks once handed to the executor (long runs; mt_plan_export
	                                   then sees only tasks not yet flushed, and a launch's temporaries are
	                                   unknown to mt_chunk_meta once their delete task is planned);
	                                   0: retain the whole plan */
	uint64_t disk_capacity;         /* disk tier below the pinned-host tier (memory.cpp:113-159): host copies
	                                   of evicted chunks move to a spill file when the host tier is full;
	                                   0 = no disk tier */
	const char* spill_dir;          /* directory of the spill file (NULL: the system temp directory) */
	uint64_t schedule_seed;         /* 0: deterministic stream choice; else every task goes to a compute stream
	                                   drawn from a generator seeded with it, behind a random on-device delay,
	                                   and graph replay is off: the GPU analogue of the reference's seeded
	                                   ready-task choice (runtime.cpp:313-319, run_overrides::ready_seed) */
	int32_t plan_cache_off;         /* 1: plan every launch from scratch; 0: a repeated identical launch whose
	                                   chunks are in the earlier launch's conflict state (task ids moved)
	                                   replays that plan (identical tasks, a fraction of the cost) */
	int32_t pad_;
} mt_config;

/* One planned chunk access (a create counts as a write of the whole chunk). */
typedef struct mt_access {
	int64_t task;
	int64_t chunk;
	mt_rect region;
	int32_t write;
	int32_t pad_;
} mt_access;

typedef struct mt_ctx mt_ctx;
typedef struct mt_exec mt_exec;

const char* mt_last_error(void);
const char* mt_version(void);

/* ---- distributions (distribution.cpp:110-220) -------------------------------------- */
/* Tiles `domain` into chunks of `extents` grown by `halo` and clipped; homes round-robin.
 * Writes at most `cap` descriptors; *n_out receives the total. row/col/tile/stencil
 * distributions are all this call with the matching extents/halo. */
int mt_dist_tile(const mt_rect* domain, const int64_t* extents, const int64_t* halo, const mt_device* devices, int32_t ndev, int64_t first_id,
    mt_chunk_desc* out, int64_t cap, int64_t* n_out);
int mt_dist_replicated(const mt_rect* domain, const mt_device* devices, int32_t ndev, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out);
int mt_dist_single(const mt_rect* domain, mt_device home, int64_t first_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out);
/* block_work_dist: superblocks of `threads_per_superblock` over `grid`, round-robin devices */
int mt_work_block(const mt_rect* grid, const int64_t* block, const int64_t* threads_per_superblock, const mt_device* devices, int32_t ndev,
    mt_superblock* out, int64_t cap, int64_t* n_out);

/* ---- driver: planning + (optionally) execution ---------------------------------------- */
int mt_ctx_create(const mt_config* cfg, mt_ctx** out);
int mt_ctx_destroy(mt_ctx* ctx);
/* devices() in worker-major order */
int mt_ctx_devices(mt_ctx* ctx, mt_device* out, int32_t cap, int32_t* n_out);
/* create_array (planner.cpp:122-140): chunk ids are rebased onto the global id space */
int mt_array_create(mt_ctx* ctx, const mt_rect* domain, int32_t dtype, const mt_chunk_desc* chunks, int64_t nchunks, int32_t fill, int64_t* out_id);
int mt_array_delete(mt_ctx* ctx, int64_t array_id);
/* the array's (rebased) chunk descriptors */
int mt_array_chunks(mt_ctx* ctx, int64_t array_id, mt_chunk_desc* out, int64_t cap, int64_t* n_out);
int mt_launch(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* annotation, int64_t* first_task, int64_t* past_last_task);
/* The repeat loop of apply_scenario (scenario.cpp:407-441) in one call: `repeat` launches of the
 * same request; after each one every array argument equal to swap_a becomes swap_b and vice
 * versa (the scenario's name swap; pass -1 for no swap); the new tasks are handed to the executor
 * after every `flush_every` launches (0: only at the end, negative: never). *first_task / *past_last_task cover
 * all launches. */
int mt_launch_repeat(mt_ctx* ctx, const char* kernel, const mt_rect* grid, const int64_t* block, const mt_superblock* work, int64_t nwork,
    const mt_launch_arg* args, int32_t nargs, const char* annotation, int32_t repeat, int64_t swap_a, int64_t swap_b, int32_t flush_every,
    int64_t* first_task, int64_t* past_last_task);
/* Hands every task emitted since the previous call to the executor (take_pending+submit). */
int mt_flush(mt_ctx* ctx);
int mt_sync(mt_ctx* ctx);
/* Reads a whole array (row-major over its domain) into host memory; assembles chunks in
 * ascending id order like the reference's gather (scenario.cpp:471-484). */
int mt_array_read(mt_ctx* ctx, int64_t array_id, void* host, uint64_t bytes);
/* Uploads host data into every chunk of an array (B200 extension: e2e input path). */
int mt_array_write(mt_ctx* ctx, int64_t array_id, const void* host, uint64_t bytes);
/* B200 extension: asynchronous host transfers, planned as tasks and therefore ordered against
 * launches by the dependency tracking (a write overwrites every chunk; a read copies each
 * cell once, from the lowest-id chunk holding it). They return once queued; the host buffer
 * (row-major over the domain; pinned memory for DMA overlap) must stay valid and untouched
 * until mt_sync. Replaces the synchronous round trip of mt_array_write / mt_array_read
 * (runtime.cpp:697-712 read_chunk) in pipelines that stream inputs and results. */
int mt_array_write_async(mt_ctx* ctx, int64_t id, const void* host, uint64_t bytes);
int mt_array_read_async(mt_ctx* ctx, int64_t id, void* host, uint64_t bytes);
/* The same with a host array that covers only `host_box` (row-major over it). Task planning
 * does not depend on the box, so in a one-process-per-GPU job every rank calls it collectively
 * with its own box and buffer (e.g. its chunks' rows) and the ranks' plans stay identical;
 * every transfer a rank executes must lie inside that rank's box (MT_EEXEC otherwise). */
int mt_array_write_box_async(mt_ctx* ctx, int64_t id, const mt_rect* host_box, const void* host, uint64_t bytes);
int mt_array_read_box_async(mt_ctx* ctx, int64_t id, const mt_rect* host_box, void* host, uint64_t bytes);
/* Byte-compares every overlapping chunk pair (check_replicas, scenario.cpp:486-509);
 * *coherent = 1 when all agree. */
int mt_array_check_replicas(mt_ctx* ctx, int64_t array_id, int32_t* coherent);
/* Plan export: tasks with id in [first, last) plus side pools. Pass caps of 0 to size. */
int mt_plan_export(mt_ctx* ctx, int64_t first, int64_t last, mt_task* tasks, int64_t task_cap, int64_t* ntasks, int64_t* pool, int64_t pool_cap,
    int64_t* npool, mt_arg_binding* args, int64_t args_cap, int64_t* nargs);
int64_t mt_plan_size(mt_ctx* ctx);
/* launches planned by replaying an earlier identical launch's plan (mt_config.plan_cache_off) */
uint64_t mt_plan_cache_hits(mt_ctx* ctx);
/* access records of non-temporary chunks in emission order (needs cfg.record_accesses);
 * used to check that the dependency DAG orders every pair of conflicting accesses */
int mt_plan_accesses(mt_ctx* ctx, mt_access* out, int64_t cap, int64_t* n_out);
/* parse_annotation (annotation.cpp:105-391) as canonical text: {"bindings": [[space, [vars]]...],
 * "accesses": [[argument, mode, op, [["single", E] | ["slice", E|null, E|null]...]]...]} with
 * E = [constant, [[variable, coefficient]...]] (folded terms, first-occurrence order). Parse errors
 * return MT_EPARSE. *len = text length; written with its terminator when cap > *len. */
int mt_annotation_describe(const char* text, char* out, int64_t cap, int64_t* len);
/* chunk_meta (planner.hpp:41-45): temp flag, dtype, descriptor */
int mt_chunk_meta(mt_ctx* ctx, int64_t chunk, mt_chunk_desc* desc, int32_t* dtype, int32_t* temp);
/* executor attached to a context (NULL when cfg.execute == 0) */
mt_exec* mt_ctx_exec(mt_ctx* ctx);

/* ---- one process per worker (cfg.single_worker) -------------------------------------- */
/* Every rank exports its IPC mailbox blob, the blobs are exchanged out of band (any
 * all-gather, e.g. torch.distributed), then every rank imports all of them (rank order,
 * equal sizes). Send/recv tasks between workers of different processes then move through
 * GPU-driven NVLink rings with no host involvement. Barrier before destroying contexts. */
int mt_ctx_peer_export(mt_ctx* ctx, void* buf, int64_t cap, int64_t* len);
int mt_ctx_peer_import(mt_ctx* ctx, const void* blobs, int64_t blob_len, int32_t nblobs);
/* NCCL communicator for allreduce tasks between processes (cfg.collective_reduce with
 * cfg.single_worker; the reduce tree as ncclAllReduce over the partial box).
 * Rank 0 creates the 128-byte unique id, it is broadcast out of band, then every rank calls
 * mt_ctx_nccl_init collectively (rank = worker_rank, nranks = workers). `nccl_lib` is the
 * libnccl.so.2 to load when none is loaded in the process yet (NULL: the default search). */
int mt_ctx_nccl_unique_id(mt_ctx* ctx, const char* nccl_lib, void* id128);
int mt_ctx_nccl_init(mt_ctx* ctx, const char* nccl_lib, const void* id128);

/* ---- executor alone: drop-in for manta::system_runtime ------------------------------ */
int mt_exec_create(const mt_config* cfg, mt_exec** out);
int mt_exec_destroy(mt_exec* ex);
/* tasks must arrive in ascending id order across calls (take_pending order) */
int mt_exec_submit(mt_exec* ex, const mt_task* tasks, int64_t ntasks, const int64_t* pool, const mt_arg_binding* args);
int mt_exec_sync(mt_exec* ex);
int mt_exec_read_chunk(mt_exec* ex, int64_t chunk, void* dst, uint64_t bytes);
int mt_exec_write_chunk(mt_exec* ex, int64_t chunk, const void* src, uint64_t bytes);
/* run_report::to_json field names (runtime.cpp:613-636); returns required size in *len */
int mt_exec_report_json(mt_exec* ex, char* buf, int64_t cap, int64_t* len);

/* counters: tasks, device launches, copies, bytes copied, bytes sent, bytes received, peak
 * device bytes, evictions, spill bytes D2H, spill bytes H2D, dead drops (evictions without
 * write-back), dead skips (restores without H2D), host reclaims, host_write bytes, host_read
 * bytes, CUDA-graph captures, CUDA-graph replays, disk bytes out / in, inter-process messages,
 * their stream operations, copy tasks fused into their producing kernel (halo mirrors) and their
 * bytes (first n of them) */
int mt_exec_stats(mt_exec* ex, uint64_t* out, int32_t n);
/* cudaStream_t of the most recent execute task (for event timing on the launching stream) */
void* mt_exec_last_stream(mt_exec* ex);
/* device timing: mark(0) / mark(1) complete when all work enqueued before them has
 * completed on every GPU; elapsed = max over GPUs of mark1 - mark0 */
int mt_exec_mark(mt_exec* ex, int32_t slot);
int mt_exec_elapsed_ms(mt_exec* ex, double* ms);
/* per-kernel CUDA-event timing on the launching stream (count, total ms since enabled) */
int mt_exec_profile(mt_exec* ex, int32_t on);
int mt_exec_kernel_time(mt_exec* ex, const char* kernel, int64_t* count, double* total_ms);
/* per-task tracing (the reference's run_report task records, runtime.cpp:389, :514-525): while
 * on, every task gets device timestamps (after its dependency waits, after its work, on its
 * stream) and mt_exec_report_json lists {id, kind, start_ns, end_ns} per worker, ns since
 * tracing was switched on */
int mt_exec_trace(mt_exec* ex, int32_t on);

/* ---- kernel plugin API (kernels.hpp:56-105) ------------------------------------------ */
/* View of one chunk as seen by a kernel: element (g0,g1,g2) lives at
 * base[sum_k (g_k - offset_k) * stride_k] (array_view, kernels.hpp:18-42). `base` is a
 * device pointer on the executing GPU. */
typedef struct mt_view {
	void* base;
	int32_t dtype;
	int32_t rank;
	int64_t offset[MT_MAX_RANK];
	int64_t stride[MT_MAX_RANK];
	int64_t extent[MT_MAX_RANK];
} mt_view;

/* Everything one superblock launch sees (the AOT form of the paper's wrapper,
 * PAPER.md:491-511 / kernels.cpp:538-596). Threads to run: every global thread index g with
 * threads.lo <= g < threads.hi (whole blocks, planner.cpp:225-234). */
typedef struct mt_launch_ctx {
	int32_t rank;
	int32_t nparams;
	int64_t block_offset[MT_MAX_RANK]; /* superblock_blocks.lo */
	int64_t block_count[MT_MAX_RANK];  /* superblock block extents */
	int64_t block_size[MT_MAX_RANK];
	int64_t threads_lo[MT_MAX_RANK];
	int64_t threads_hi[MT_MAX_RANK];
	const int64_t* scalars_int;  /* per param index */
	const double* scalars_float; /* per param index */
	const mt_view* views;        /* per param index (base NULL when unbound) */
	const void* user;            /* the `user` pointer given at registration */
	/* Fused halo copies (B200 extension; launchers that ignore them leave mirror_applied at 0 and
	 * the executor issues the copies itself). Each mirror asks the kernel to store the cells it
	 * writes into param `param` inside the global box [lo, hi) a second time, into `dst` (another
	 * chunk: the halo of a neighbouring chunk on this GPU or, over NVLink, on a peer GPU). The
	 * launcher sets mirror_applied[i] = 1 for each mirror it wrote completely. */
	int32_t nmirrors;
	const struct mt_mirror* mirrors;
	int32_t* mirror_applied;
} mt_launch_ctx;

typedef struct mt_mirror {
	int32_t param;
	int32_t pad_;
	int64_t lo[MT_MAX_RANK];
	int64_t hi[MT_MAX_RANK];
	mt_view dst;
} mt_mirror;

/* Launcher: enqueue the superblock's work on `stream` (a cudaStream_t) and return 0. */
typedef int (*mt_launcher_fn)(const mt_launch_ctx* ctx, void* stream);

enum mt_param_kind { MT_PARAM_SCALAR = 0, MT_PARAM_ARRAY = 1 };
typedef struct mt_param_spec {
	char name[32];
	int32_t kind;
	int32_t dtype;
	int32_t rank;
	int32_t writable;
} mt_param_spec;

/* register_kernel (kernels.cpp:81-91): rejects duplicates and unsupported ranks. The
 * registry is process-global and shared by all contexts. */
int mt_kernel_register(const char* id, const mt_param_spec* params, int32_t nparams, mt_launcher_fn launcher);
int mt_kernel_count(void);
/* context-local kernel (shadows the global registry for this context's launches); the
 * launcher may be NULL for plan-only contexts */
int mt_ctx_kernel_register(mt_ctx* ctx, const char* id, const mt_param_spec* params, int32_t nparams, mt_launcher_fn launcher, const void* user);
/* context-local synthesized `gather` kernel for an annotation (scenario.cpp:276-389): one
 * array parameter per access (element type + domain given in access order) and a device
 * body that folds the thread's read regions into its write/reduce regions */
int mt_ctx_gather_register(mt_ctx* ctx, const char* id, const char* annotation_text, int32_t naccess, const int32_t* dtypes, const mt_rect* domains);
int mt_kernel_info(int32_t index, char* id, int32_t id_cap, mt_param_spec* params, int32_t cap, int32_t* nparams);
/* Runtime compilation, the paper's user model (wrapper kernels.cpp:522-596).
 * `source` defines  __device__ void <id>(dim3 virtBlockIdx, <params in order>)  with scalars
 * as int32_t/int64_t/float/double and arrays as manta::Vector<T> / Matrix<T> / Tensor<T>
 * (const for read-only parameters; operator[] chains and operator() take GLOBAL indices).
 * Per superblock the generated wrapper bakes the block offset and view offsets/strides as
 * constants and NVRTC compiles it for sm_100a on first use (cached per device and instance).
 * The source is compiled once here; compiler errors return MT_EVALIDATION with the log. */
int mt_ctx_kernel_compile(mt_ctx* ctx, const char* id, const mt_param_spec* params, int32_t nparams, const char* source);
/* the wrapper text for one instance (generate_wrapper_source, kernels.hpp:109-121):
 * offsets/strides concatenated over the array parameters in signature order */
int mt_wrapper_source(const char* id, const mt_param_spec* params, int32_t nparams, const int64_t* block_offset, int32_t rank, const int64_t* offsets,
    const int64_t* strides, char* out, int64_t cap, int64_t* len);

/* ---- scenario fuzzing (make_fuzz_scenario, proj/src/scenario.cpp:653-807) ------------- */
/* The reference's random scenario for `seed` as scenario-file JSON (scenario.cpp:131-167):
 * same draws (std::mt19937_64, uniform_int_distribution) in the same order. Writes at most
 * `cap` bytes including the NUL; *len receives the text length. */
int mt_fuzz_scenario_json(uint64_t seed, char* buf, int64_t cap, int64_t* len);

/* ---- direct contraction entry points (the kernels behind matmul_nt_bf16 / _tf32) ------- */
/* C (f32, m x n, row pitch ldc) = A (m x k) x Bt^T (Bt: n x k), all row-major DEVICE pointers,
 * enqueued on `stream` (a cudaStream_t, NULL = legacy default). bf16: A and Bt are bf16 bit
 * patterns (kind::f16); tf32: f32 operands read as TF32 (kind::tf32). Row pitches in elements
 * must make 16-byte multiples. Returns 0, or 5 (k <= 0), 6 (misaligned operands), 7 (tensor
 * map encode failed), 1 (launch error). The reference's `matmul` (kernels.cpp:167-193) is the
 * scalar form; these are the C3 tensor-core forms. */
int mt_gemm_bf16_nt(const void* a, const void* bt, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream);
int mt_gemm_tf32_nt(const float* a, const float* bt, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream);
/* tf32 operands are first rounded to nearest-even TF32 into stream-ordered scratch (so the
 * contraction is unbiased; MTB_TF32_TRUNCATE=1 skips it, return 8 = scratch allocation failed).
 * _nn: B is row-major K x N (pitch ldb), the layout of the reference's `matmul`
 * (kernels.cpp:167-193), transposed to K-major in the same pass; the builtin `matmul` takes this
 * path for superblocks with m*n*k >= 2^30 (MTB_MATMUL_EXACT=1: always the scalar kernel). */
int mt_gemm_tf32_nn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc, void* stream);
/* number of tcgen05 contraction launches issued by this process so far (evidence of which path
 * a `matmul` launch took) */
uint64_t mt_tensor_core_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* MANTA_B200_H */
