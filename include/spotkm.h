/*
 * spotkm.h -- C ABI of the B200 (sm_100a) device-mapping / context-migration
 * hot path of SpotServe (arXiv 2311.15566).
 *
 * The reference (`spotsim`, pure Python) exposes this path as Python
 * functions; this ABI is what a Python/ctypes (or any FFI) binding calls in
 * their place.  Each entry point below names the reference interface it
 * replaces (file:line under /root/reference/pkg/src/spotsim/).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Pointers prefixed `d_` are DEVICE
 *     pointers (caller-owned, e.g. torch tensors' data_ptr()); `h_` pointers
 *     are host memory.  `stream` is a cudaStream_t passed as void*.
 *   - All calls are asynchronous on `stream` and keep no global state; they
 *     are re-entrant across distinct streams / buffers.
 *   - Return value is an sk_status; sk_last_error() gives thread-local text.
 *     Status -> reference exception: SK_EINVAL/SK_EGROUP -> MappingError,
 *     SK_ENOSOURCE -> MigrationError, SK_ERANGE -> MappingError (inputs out
 *     of the exact-arithmetic range), SK_ECUDA -> RuntimeError.
 *
 * Exactness contract: every edge weight is an exact integer
 * numerator N over a per-plan denominator K (lcm of the tensor-shard counts),
 * converted once with a correctly rounded division -- bit-identical to the
 * reference's float(Fraction) (domain.py:299-320).  The matcher replays the
 * reference's `_hungarian_max` (mapping.py:71-122) in IEEE double with the
 * same operation order and tie-break, so assignments and total_weight are
 * bit-identical.
 */
#ifndef SPOTKM_H
#define SPOTKM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPOTKM_ABI_VERSION 3

typedef enum {
  SK_OK = 0,
  SK_EINVAL = 1,    /* malformed arguments                       -> MappingError   */
  SK_EGROUP = 2,    /* fused group does not divide G and M        -> MappingError   */
  SK_ERANGE = 3,    /* numerator bound >= 2^127 / K >= 2^62       -> MappingError   */
  SK_ENOSOURCE = 4, /* a required shard has no live holder        -> MigrationError */
  SK_ECUDA = 5,     /* CUDA runtime error                         -> RuntimeError   */
  SK_ENOPEER = 6    /* peer access unavailable for the executor   -> RuntimeError   */
} sk_status;

/* plan flags */
#define SK_PLAN_FUSED_SUM 1 /* fused edge weight = Python builtin sum() of the inner match (else max) */
#define SK_PLAN_DENSE 2     /* the F buffer holds a caller-given dense W (km_match); no segments      */
#define SK_PLAN_GENERIC 4   /* general-range plan: wide segments (sk_segment_wide), 128-bit
                               numerators, 64-bit K, any fused group 1..32 (see sk_map_fuse)     */

/*
 * One context segment of an old GPU's inventory: layers [l0, l1) x the
 * tensor-shard interval [a, b) / K.  pipe == 0: model parameters, `unit` =
 * bytes_per_layer x multiplicity.  pipe >= 1: KV cache that counts only
 * toward positions of NEW pipeline `pipe`; `unit` = kv_bytes_per_token_per_layer
 * x sum over the segment's requests of min(tokens held, tokens needed).
 * Shared bytes with position v = sum_seg |[l0,l1) & stage(v)| * |[a,b) & I(v)| * unit / K
 * (the closed form of overlap_bytes, domain.py:299-320, on
 * required_context_with_cache, mapping.py:155-169).
 */
typedef struct sk_segment {
  int32_t l0, l1;
  int32_t a, b;
  int32_t pipe;
  int32_t reserved;
  int64_t unit;
} sk_segment; /* 32 bytes */

/*
 * The same segment for SK_PLAN_GENERIC plans, whose endpoints may exceed
 * int32 (K up to 2^62) and whose numerators may exceed 2^53 (accumulated in
 * 128 bits; every plan's sum_seg (l1-l0)(b-a)unit < 2^127, checked on the
 * host).  It occupies TWO sk_segment slots; row_ptr counts slots.
 */
typedef struct sk_segment_wide {
  int32_t l0, l1;
  int32_t pipe;
  int32_t reserved;
  int64_t a, b;
  int64_t unit;
  int64_t reserved2[3];
} sk_segment_wide; /* 64 bytes = 2 x sk_segment */

/*
 * One mapping problem (one build_graph / map_devices call).
 * Rows are the candidate GPUs in the reference row order (instances by
 * natural_key, then local index; mapping.py:193-198); columns are the target
 * positions in lexicographic (d, p, m) order (domain.py:92-99).
 */
typedef struct sk_plan {
  int32_t rows;     /* R = candidate GPUs                                       */
  int32_t D, P, M;  /* target configuration                                     */
  int32_t L;        /* model layers                                             */
  int32_t K;        /* common denominator of every interval (multiple of M), <= 2^31-1;
                       0 for SK_PLAN_GENERIC plans, which carry it in Kw        */
  int32_t group;    /* fused group size g = min(G, M) (1 = flat km_match)       */
  int32_t flags;    /* SK_PLAN_*                                                */
  int32_t row_base; /* row r's segments: seg[row_ptr[row_base+r] .. row_ptr[row_base+r+1]) */
  int32_t reserved;
  int64_t f_off;    /* element offset of the plan's fused matrix (nA x nB) and perm block;
                       SK_PLAN_GENERIC plans use sk_fused_elems() doubles there  */
  int64_t out_off;  /* element offset of the plan's R assignment entries        */
  int64_t Kw;       /* SK_PLAN_GENERIC: the common denominator, < 2^62          */
} sk_plan; /* 64 bytes */

/* Elements of the fused buffer one plan occupies at f_off: nA*nB for the
 * regular path; for SK_PLAN_GENERIC plans the fused matrix is followed by
 * the g matched weights and the g inner-permutation bytes of every fused
 * pair: nA*nB*(1+g) doubles + ceil(nA*nB*g / 8). */
int64_t sk_fused_elems(int32_t nA, int32_t nB, int32_t group, int32_t flags);

/* Library / ABI identification. */
int sk_abi_version(void);
const char* sk_last_error(void);

/*
 * K1 -- build_graph (mapping.py:184-216): dense W[R][C] in float64, one plan
 * per call row block.  d_W receives, for plan q, R*C doubles at d_W + f_off.
 */
int sk_build_weights(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                     const sk_segment* d_segs, double* d_W, int max_rows, int max_cols,
                     void* stream);
/* (SK_PLAN_GENERIC plans: 128-bit numerators, one correctly rounded
 * conversion each -- the same float(Fraction) value for any size.) */

/*
 * K2 -- map_devices (mapping.py:222-283) for a batch of plans: per fused pair
 * an inner KM on the g x g block (weights built on the fly, never stored),
 * fused weight max|sum, then one warp per plan runs the outer KM on the
 * zero-padded fused matrix and expands the assignment.  Also serves km_match
 * (mapping.py:125-149) with group = 1.
 *   d_fused : >= sum over plans of nA*nB doubles   (scratch, at f_off)
 *   d_perm  : >= sum over plans of nA*nB uint32    (scratch, at f_off)
 *   d_assign: per plan R int32 at out_off: column index or -1 (unassigned)
 *   d_total : per plan total_weight (accumulated in the reference order)
 *   max_na / max_nb = max fused rows / slots (R/g, C/g), max_rows = max R over the batch.
 *   group_mask: bit g set when some plan has group g (1..8), bit 0 when some
 *               plan is SK_PLAN_GENERIC (0 = launch everything).
 *   SK_PLAN_GENERIC plans (any group 1..32, 128-bit numerators): one warp per
 *   fused pair runs the inner KM on the g x g block in shared memory.
 *   fused_elems: elements of d_fused / d_perm in use (cleared first).
 */
int sk_map_batched(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                   const sk_segment* d_segs, double* d_fused, uint32_t* d_perm,
                   int32_t* d_assign, double* d_total, int max_na, int max_nb,
                   int max_rows, int group_mask, int64_t fused_elems, void* stream);

/* The two halves of sk_map_batched, for callers that time or pipeline them:
 * K2a (inner KMs + fused weights) and K2b (outer KM + expansion).  K2a
 * writes every element of each plan's fused matrix (zero rows first, then
 * only the fused pairs that can be non-zero); [clear_begin, clear_begin +
 * clear_count) of d_fused / d_perm is additionally memset to zero first --
 * not needed, pass clear_count = 0.  d_steps
 * (optional, may be NULL) receives per plan {Dijkstra steps, cost-row element
 * loads from L2 (0 for dictionary-coded plans)} (2 x int64) -- the
 * algorithmic work of the outer KM. */
int sk_map_fuse(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                const sk_segment* d_segs, double* d_fused, uint32_t* d_perm, int max_na, int max_nb,
                int group_mask, int64_t clear_begin, int64_t clear_count, void* stream);
int sk_map_outer(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                 const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                 int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                 void* stream);

/* sk_map_outer with a global code scratch: big size classes (few plans per
 * SM with shared-memory codes) keep their dictionary codes in d_codes
 * (L2-resident) instead of shared memory, so more plans run per SM.
 * sk_outer_codes_bytes returns the bytes a launch of (n_plans, max_n,
 * max_rows) would use, 0 when it keeps the codes in shared memory; pass
 * NULL / 0 to disable. */
int sk_map_outer_codes(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                       const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                       int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                       uint8_t* d_codes, int64_t codes_bytes, void* stream);
int64_t sk_outer_codes_bytes(int n_plans, int max_n, int max_rows);

/* K2 with the fused matrix dictionary-coded by K2a itself: sk_map_fuse_coded
 * writes each plan's fused weights as one-byte codes into the outer KM's code
 * layout (d_codes, sk_precoded_bytes of them) and its distinct values into a
 * 256-slot dictionary per plan (d_dict, *dict_bytes of them) instead of
 * doubles into d_fused; sk_map_outer_coded reads them (no double matrix, no
 * dictionary build).  A plan with more than 255 distinct non-zero fused
 * values (and every general-range plan) still gets its double matrix in
 * d_fused and takes the uncoded path -- same results either way.
 * sk_precoded_bytes returns 0 when the class cannot be coded (max_n > 4095:
 * use sk_map_fuse + sk_map_outer).  Both calls must see the same (n_plans,
 * max_n) and buffers. */
int64_t sk_precoded_bytes(int n_plans, int max_n, int64_t* dict_bytes);
int sk_map_fuse_coded(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                      const sk_segment* d_segs, double* d_fused, uint32_t* d_perm, int max_na,
                      int max_nb, int group_mask, uint8_t* d_codes, int64_t codes_bytes,
                      uint64_t* d_dict, int64_t dict_bytes, void* stream);
int sk_map_outer_coded(const sk_plan* d_plans, int n_plans, const int32_t* d_row_ptr,
                       const sk_segment* d_segs, const double* d_fused, const uint32_t* d_perm,
                       int32_t* d_assign, double* d_total, int64_t* d_steps, int max_n, int max_rows,
                       uint8_t* d_codes, int64_t codes_bytes, const uint64_t* d_dict, void* stream);
/* Outer problems with n > 4095 (any size) run one 1024-thread CTA per plan
 * with the column state in device scratch that the call allocates
 * stream-ordered (cudaMallocAsync) and frees on the same stream. */

/*
 * km_match on caller-given dense weights (mapping.py:125-149): plans with
 * SK_PLAN_DENSE, group 1, W (R x C, row-major doubles) at d_W + f_off.
 */
int sk_km_dense(const sk_plan* d_plans, int n_plans, const double* d_W, int32_t* d_assign,
                double* d_total, int max_n, int max_rows, void* stream);

/*
 * Sweep expansion: compact preemption-sweep descriptors -> sk_plan rows and
 * segments on device (positional old layout on instances i-0..i-(n-1), alive
 * subset, B cached requests per old pipeline with identity inheritance;
 * SURVEY.md 8(d)).  Host precomputes offsets; the kernel writes row_ptr/segs.
 */
typedef struct sk_sweep_desc {
  int32_t oD, oP, oM;    /* old configuration                        */
  int32_t G;             /* GPUs per instance                        */
  int32_t n_inst;        /* pool instances before preemption         */
  int32_t alive_off;     /* word offset of the alive bitmask         */
  int32_t tok_off;       /* offset of oD per-old-pipeline token sums */
  int32_t plan;          /* index of the sk_plan this fills          */
  int64_t bpl, kv;       /* model bytes per layer / kv per token per layer */
} sk_sweep_desc; /* 48 bytes */

int sk_sweep_expand(const sk_sweep_desc* d_desc, int n_desc, const uint32_t* d_alive,
                    const int64_t* d_tok, const sk_plan* d_plans, int32_t* d_row_ptr,
                    sk_segment* d_segs, int max_rows, void* stream);

/*
 * K3 -- migration executor (the paper's batched send/recv, PAPER.md:491-497;
 * the reference only plans it: migration.py:311-384).  One byte-range copy
 * per Transfer, pulled by the destination GPU from a peer-mapped source over
 * NVLink.  Copies of one plan round run concurrently; `round_ptr` delimits
 * rounds; copies are grouped per destination device.
 */
typedef struct sk_copy {
  uint64_t src;   /* device address readable from the launching device (peer or local) */
  uint64_t dst;   /* device address on the launching device                            */
  uint64_t bytes;
} sk_copy;

int sk_copy_batched(const sk_copy* d_copies, int n_copies, int n_ctas, void* stream);

/*
 * K3, plan-ordered: ONE persistent launch per rank executes the rank's share
 * of a MigrationPlan round by round (migration.py:311-384).  CTA 0 monitors
 * progress; workers copy 1 MiB chunks in plan order.  A chunk whose
 * destination reuses arena space released at the end of round `wait_round`
 * (the plan's `releases`, recycled by the host's arena allocator) waits until
 * every rank has completed rounds 0..wait_round (their progress words,
 * peer-mapped); no other cross-rank wait.  Stage-ready flags (start_stage,
 * migration.py:352-371) are raised on the device as soon as global progress
 * passes the round each marker follows, stamped with %globaltimer.
 *   d_ctl: sk_exec_ctl_bytes(n_rounds, n_stages) bytes of device memory:
 *     u32 [0] work_next [1] progress (rounds complete, read by peers)
 *     [2] error (0 ok, 1 worker timeout, 2 monitor timeout) [3] reserved,
 *     [4, 4+n_rounds) chunks done per round, then n_stages stage flags, then
 *     (8-byte aligned) u64 stamps: launch start, each stage's ready time (ns).
 *   d_peer_progress: device array of n_peers device pointers to the other
 *     ranks' progress words (CUDA IPC mappings of their d_ctl + 1).
 * The call resets d_ctl on `stream` first; ranks must not launch a new run
 * before every peer has reset (a barrier between runs).
 */
typedef struct sk_exec_chunk {
  uint64_t src, dst, bytes;
  int32_t round;       /* plan round (non-start_stage action index) it belongs to */
  int32_t wait_round;  /* -1, or: wait until every rank completed rounds 0..wait_round */
} sk_exec_chunk; /* 32 bytes */

int64_t sk_exec_ctl_bytes(int n_rounds, int n_stages);
/* Zero a control block (flags down) ahead of a run, e.g. before handing its
 * IPC handle to a consumer that will wait on the stage flags. */
int sk_exec_reset(uint32_t* d_ctl, int n_rounds, int n_stages, void* stream);
int sk_exec_plan(const sk_exec_chunk* d_chunks, int n_chunks, const uint32_t* d_round_total, int n_rounds,
                 const int32_t* d_stage_round, int n_stages, uint32_t* d_ctl,
                 const uint32_t* const* d_peer_progress, int n_peers, uint32_t* d_flag_mirror, int n_ctas,
                 double timeout_s, void* stream);
/* d_flag_mirror (optional): the device address of host memory (e.g. a POSIX
 * shared-memory segment registered with sk_host_register) that receives a
 * copy of each stage flag as it is raised -- how a consumer in ANOTHER
 * process learns readiness without a GPU-side wait (contexts of two processes
 * time-slice on one GPU, so a waiting consumer kernel or stream can hold off
 * the producer). */
int sk_host_register(void* h_ptr, uint64_t bytes, void** d_ptr);
int sk_host_unregister(void* h_ptr);

/* Consumer side of the stage-ready flags (e.g. a serving process that maps
 * a context daemon's control block with CUDA IPC): work queued on `stream`
 * after this call runs only once *d_flag >= value.  d_status (optional)
 * receives 0, or 1 if timeout_s passed first. */
int sk_wait_flag(const uint32_t* d_flag, uint32_t value, double timeout_s, uint32_t* d_status, void* stream);
/* The same wait as a stream memory operation (cuStreamWaitValue32, GEQ):
 * executed by the stream's front end, no SM held -- use it when the flag's
 * producer is a kernel of another process on the same GPU. */
int sk_stream_wait_flag(const uint32_t* d_flag, uint32_t value, void* stream);

/* Copy-engine comparison path: one cudaMemcpyAsync per (HOST array) entry,
 * in order, on `stream`.  sk_d2h: blocking device -> host copy (control
 * block readback). */
int sk_memcpy_batched(const sk_copy* h_copies, int n, void* stream);
int sk_d2h(void* h_dst, const void* d_src, uint64_t bytes);

/* Peer-access helper: enable access from `device` to each of `peers`. */
int sk_enable_peer_access(int device, const int* peers, int n_peers);

/* Executor memory: cudaMalloc'd slabs (exportable with CUDA IPC so peer ranks
 * of the same box can map them and pull over NVLink). */
int sk_dev_alloc(uint64_t bytes, void** d_ptr);
int sk_dev_free(void* d_ptr);
int sk_ipc_get_handle(const void* d_ptr, void* handle64);   /* 64-byte cudaIpcMemHandle_t */
int sk_ipc_open_handle(const void* handle64, void** d_ptr);
int sk_ipc_close_handle(void* d_ptr);

/* Byte-pattern fill / verify of context regions: the 8-byte word at global
 * byte offset x of a context object holds splitmix64(key ^ x/8).  `base` is
 * the region's global offset inside its object (8-byte aligned). */
typedef struct sk_region {
  uint64_t ptr, bytes, key, base;
} sk_region;
int sk_fill_regions(const sk_region* d_regions, int n, void* stream);
int sk_verify_regions(const sk_region* d_regions, int n, unsigned long long* d_bad, void* stream);
const char* sk_reshard_error(void);

/* ------------------------------------------------------------------------
 * Migration planner (host, native, bit-exact) -- replaces plan_migration
 * (migration.py:311-384) incl. derive_transfers (201-305), _cover_from_holders
 * (149-194), memopt_layer_order (89-143) and simulate_buffer_usage (387-401).
 * Interval endpoints are integer numerators over K (lcm of every interval
 * denominator and M); GPUs are given in the reference's sorted order
 * (natural_key(instance), local index); instances carry their natural-key
 * rank, plain string rank (release sorting) and departing flag.
 */
typedef struct sk_mig_input {
  int32_t n_inst, n_gpus;
  const int32_t* inst_natrank;
  const int32_t* inst_strrank;
  const uint8_t* inst_departing;
  const int32_t* gpu_inst;
  const int32_t* gpu_local;
  const int32_t* gpu_pos;       /* flat target position ((d-1)*P+(p-1))*M+(m-1), or -1 */
  const int32_t* model_ptr;     /* [n_gpus+1] */
  const int64_t* model_shards;  /* (layer, lo, hi) triples, inventory order */
  const int32_t* cache_ptr;     /* [n_gpus+1] */
  const int64_t* cache_shards;  /* (rid, layer, lo, hi, tokens), inventory order */
  int32_t D, P, M, L;
  int64_t bpl, kv, K;
  const int32_t* inh_ptr;       /* [D+2] CSR over new pipelines 1..D, or NULL */
  const int64_t* inh_items;     /* (rid, tokens) pairs in inherited order */
  int32_t has_umax, reserved;
  double u_max;
} sk_mig_input;

typedef struct sk_mig_transfer {
  int32_t kind, layer; /* kind 0 model, 1 cache */
  int64_t lo, hi;      /* numerators over K */
  int32_t src, dst;    /* gpu indices (input order) */
  double bytes;
  int64_t rid, tokens; /* rid -1 for model transfers */
} sk_mig_transfer;

typedef struct sk_mig_action {
  int32_t kind; /* 0 migrate_cache, 1 migrate_layer, 2 start_stage */
  int32_t layer, stage;
  int32_t tr_begin, tr_end, rel_begin, rel_end;
  int32_t reserved;
} sk_mig_action;

typedef struct sk_mig_release {
  int32_t inst, layer;
  double bytes;
} sk_mig_release;

typedef struct sk_mig_result sk_mig_result; /* opaque, library-owned */

/* derive_only != 0: stop after derive_transfers; the result then holds the
 * model transfers (first) and cache transfers, cache releases in `releases`
 * and per-layer releases in `layer_releases`, all in the reference's order.
 * SK_ENOSOURCE: sk_planner_error() holds "<lo> <hi>" numerators of the
 * uncovered piece. */
int sk_plan_migration(const sk_mig_input* in, int derive_only, sk_mig_result** out);
/* Many independent plans on a pool of n_threads host threads (0 = all
 * cores): per plan status[i], outs[i] (free each with sk_mig_free), and for
 * SK_ENOSOURCE the uncovered piece's numerators in err_range[2i..2i+1]. */
int sk_plan_migration_many(const sk_mig_input* ins, int n, int derive_only, int n_threads,
                           sk_mig_result** outs, int32_t* status, int64_t* err_range);
/* counts[7] = {transfers, actions, action_transfers, releases, peak entries,
 *              layer_releases, model transfers} */
int sk_mig_counts(const sk_mig_result* r, int64_t* counts);
int sk_mig_export(const sk_mig_result* r, sk_mig_transfer* transfers, sk_mig_action* actions,
                  int32_t* action_transfers, sk_mig_release* releases, double* peak,
                  sk_mig_release* layer_releases);
void sk_mig_free(sk_mig_result* r);
const char* sk_planner_error(void);

/* plan_timeline (costmodel.py:189-228): per-action completion times under
 * per-instance full-duplex link serialisation; migration_cost (231-260) is
 * the caller's scalar reduction of these. */
typedef struct sk_timeline_input {
  int32_t n_inst, n_actions;
  const int32_t* action_ptr; /* [n_actions+1] into the transfer arrays */
  const int32_t* src_inst;
  const int32_t* dst_inst;
  const double* bytes;
  double bandwidth, latency, start;
  const uint8_t* has_release; /* per instance, or NULL */
  const double* release;
} sk_timeline_input;

int sk_plan_timeline(const sk_timeline_input* t, double* ends);

/* migration_cost (costmodel.py:231-260) on the host: the timeline above, then
 * the full duration, or with progressive != 0 the worst stage-ready
 * constraint; act_stage[a] = stage of a start_stage action, else -1;
 * step = t_dec(config) / P (0 without a config). */
int sk_migration_cost(const sk_timeline_input* t, const int32_t* act_stage, double step,
                      int32_t progressive, double* cost);

/* simulate_buffer_usage (migration.py:387-401): per-instance peak bytes of a
 * plan replay.  Instances 0..n_seed-1 are the old layout's, in its order;
 * per action a: received transfers tr_ptr[a]..tr_ptr[a+1] (dst instance,
 * bytes) then end-of-round releases rel_ptr[a]..; name_rank orders
 * instances by id string.  order[0..*n_order) = the result's key order. */
int sk_simulate_buffer_usage(int32_t n_inst, int32_t n_seed, int32_t n_actions, const int32_t* tr_ptr,
                             const int32_t* tr_dst, const double* tr_bytes, const int32_t* rel_ptr,
                             const int32_t* rel_inst, const double* rel_bytes, const int32_t* name_rank,
                             double* peaks, int32_t* order, int32_t* n_order);

/* Batched migration_cost (costmodel.py:231-260 over plan_timeline 189-228)
 * for many candidate plans on the device, one thread per plan.  Per plan:
 * actions [act_begin, act_end) (CSR act_ptr into the transfer arrays;
 * act_stage = stage of a start_stage action, else -1), instances are
 * plan-local ids with release floors at inst_base + i, scratch holds
 * 2 * sum(n_inst) doubles and flags as many bytes. */
typedef struct sk_tl_plan {
  int32_t act_begin, act_end;
  int32_t inst_base, n_inst;
  double start, step; /* step = t_dec(config) / P, or 0 */
  int32_t progressive, reserved;
} sk_tl_plan; /* 40 bytes */

int sk_migration_cost_batched(const sk_tl_plan* d_plans, int n_plans, const int32_t* d_act_ptr,
                              const int32_t* d_act_stage, const int32_t* d_src_inst,
                              const int32_t* d_dst_inst, const double* d_bytes,
                              const uint8_t* d_has_release, const double* d_release,
                              double* d_scratch, uint8_t* d_flags, double bandwidth,
                              double latency, double* d_cost, void* stream);

/* ------------------------------------------------------------------------
 * Candidate scoring (estimator.cu): exec_latency / throughput
 * (costmodel.py:121-183) for many (config, workload) queries and the
 * controller's choice optimize_config (controller.py:79-117) for many
 * (n_available, obtainable, rate) scenarios, on the device, bit-identical.
 * Profile tables: per profiled (P,M,B) shape s: decode[s] seconds; prefill
 * points pre_s/pre_v[pre_ptr[s] .. pre_ptr[s+1]) with s_in ascending.
 */
typedef struct sk_est_query {
  int32_t shape;  /* profiled (P,M,B) shape index */
  int32_t D, P, B;
  int64_t s_in, s_out;
} sk_est_query; /* 32 bytes */

/* d_latency[i] = exec_latency(query i); d_phi (optional) = D*B / (latency /
 * (P * eta)) -- throughput() when s_in/s_out are the profile's nominal ones. */
int sk_score_configs(const sk_est_query* d_q, int n, const double* d_decode, const int32_t* d_pre_ptr,
                     const int64_t* d_pre_s, const double* d_pre_v, double eta, double* d_latency,
                     double* d_phi, void* stream);
/* Candidates in ascending (D,P,M,B) order with instance count, nominal phi
 * and latency; per scenario the chosen candidate index, or -1 (nothing fits).
 * band = 1 + LATENCY_SIMILARITY as the reference computes it. */
int sk_select_configs(const int32_t* d_n_inst, const double* d_phi, const double* d_latency, int n_cfg,
                      const int32_t* d_n_available, const int32_t* d_obtainable, const double* d_rate,
                      int n_queries, double band, int32_t* d_choice, void* stream);
const char* sk_estimator_error(void);

/* memopt_layer_order (migration.py:114-143) on per-layer traffic given as CSR
 * lists of (instance, bytes): incoming[l] and freed[l] for l in 0..L-1.
 * order receives L layer indices. */
int sk_memopt_order(int32_t n_layers, int32_t n_inst, const int32_t* in_ptr, const int32_t* in_inst,
                    const double* in_bytes, const int32_t* fr_ptr, const int32_t* fr_inst,
                    const double* fr_bytes, int32_t has_umax, double u_max, int32_t* order);

/* Correctly rounded (num_hi * 2^64 + num_lo) / den as a double, num >= 0,
 * den > 0: the conversion float(Fraction) performs (utility, exposed for tests). */
double sk_rat_to_double(int64_t num_hi, uint64_t num_lo, int64_t den);

#ifdef __cplusplus
}
#endif

#endif /* SPOTKM_H */
