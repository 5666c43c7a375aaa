/*
 * mk.h -- C ABI of the B200 hierarchical task megakernel (libmk.so).
 *
 * This is the drop-in boundary below the Python task-graph API.  In the
 * reference (/root/reference/pkg/src/chipletsim) the call that executes a
 * task graph is
 *
 *     simulate(g, machine, h=None, *, traversal, distribution, window,
 *              dispatch_overhead_s, fence_seconds_per_line, keep_event_log)
 *         -> SimTrace                                   (runtime.py:253-264)
 *
 * Here the host graph compiler (paper_2604_15379_b200/lowering.py) flattens a
 * TaskGraph into the descriptor arrays below and one decode step is one
 * cooperative launch of a persistent sm_100a kernel:
 *
 *   mk_probe      <- MachineConfig num_xcds / cus_per_xcd (machine.py:43-52):
 *                    the die map is measured, not configured.
 *   mk_create     <- the TaskGraph that simulate() consumes (taskgraph.py:135)
 *   mk_step       <- simulate() main loop (runtime.py:350-487): per-die
 *                    scheduler CTAs dispatch to worker CTAs, two-level
 *                    completion counting, event polling.
 *   mk_counters   <- SimTrace counters fences / global_atomics /
 *                    local_atomics / dispatches / polls (runtime.py:92-113)
 *   mk_event_log  <- SimTrace.event_log (step, actor, action, id)
 *                    (runtime.py:326, 366, 394, 416, 456, 477)
 *   status codes  <- exit codes 0 / 2 / 3 of the CLI (cli.py:20-22):
 *                    ConfigError/GraphError -> MK_ERR_CONFIG,
 *                    DeadlockError (runtime.py:482-486) -> MK_ERR_DEADLOCK.
 *
 * All pointers in descriptors are device pointers owned by the caller
 * (weights, activations, KV cache).  The handle owns the event counters, the
 * die counters, the worker mailboxes and the statistics.  A handle is bound
 * to one device and one stream at a time and is not re-entrant.
 */
#ifndef MK_H
#define MK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define MK_OK 0
#define MK_ERR_CONFIG 2   /* bad descriptor / graph (GraphError, ConfigError) */
#define MK_ERR_DEADLOCK 3 /* device watchdog fired: an event never completed  */
#define MK_ERR_CUDA 4     /* CUDA runtime error                                */

/* ---- task levels (taskgraph.py:34-38) and device opcodes --------------- */
#define MK_LEVEL_WAVEFRONT 0
#define MK_LEVEL_CU 1
#define MK_LEVEL_CHIPLET 2

#define MK_OP_NOP 0
#define MK_OP_RMSNORM 1      /* OpKind.RMS_NORM (+ embedding gather at L0)   */
#define MK_OP_GEMM 2         /* the four LINEAR_OPS and the LM head          */
#define MK_OP_ATTN_PARTIAL 3 /* OpKind.ATTN_PARTIAL: QK-norm, RoPE, KV append,
                                split-KV partial softmax                     */
#define MK_OP_ATTN_REDUCE 4  /* OpKind.ATTN_REDUCE: merge split partials     */
#define MK_OP_SILU 5         /* OpKind.SILU (standard mode only)             */
#define MK_OP_ARGMAX 6       /* appended: greedy token from LM-head partials */
#define MK_OP_TP_ALLREDUCE 7 /* tensor parallel: flags + rank-ordered sum of the
                                fp32 partials every rank pushed into this rank's
                                exchange region, + residual -> bf16 (not in the
                                reference: SURVEY.md 8(e))  */
#define MK_OP_TP_ARGMAX 8    /* tensor parallel: (max, index) of the local vocab
                                shard pushed to every rank, global greedy token */

#define MK_EPI_NONE 0
#define MK_EPI_RESIDUAL 1 /* o_proj / down: y = x W^T + residual            */
#define MK_EPI_SILU 2     /* fused gate/up halves: y = silu(g) * u           */
#define MK_EPI_LOGITS 3   /* LM head: fp32 logits + per-worker argmax        */
#define MK_EPI_PARTIAL 4  /* TP row-parallel o_proj / down: the fp32 partial
                             product is stored straight into every rank's
                             exchange region (y = byte offset of this rank's
                             slot, identical on all ranks)                   */

#define MK_BODY_GEMV 0   /* CUDA cores, 128-bit weight streaming (batch <= 16)  */
#define MK_BODY_UMMA 1   /* tcgen05.mma: 128 weight rows x batch, TMEM accum.   */

#define MK_TRAV_N_MAJOR 0
#define MK_TRAV_M_MAJOR 1
#define MK_DIST_M_TILE 0
#define MK_DIST_M_SPLIT 1

#define MK_SCHED_PER_DIE 0 /* one scheduler CTA per die (chiplet-aware)    */
#define MK_SCHED_FLAT 1    /* one scheduler for the GPU (die-unaware)      */

#define MK_MAX_SMS 256
#define MK_MAX_DIES 8
#define MK_MAX_TP 8        /* tensor-parallel ranks                              */

typedef struct mk_topology {
  int32_t num_sms;
  int32_t num_dies;
  int32_t sms_per_die[MK_MAX_DIES];
  int32_t die_of_sm[MK_MAX_SMS]; /* indexed by %smid                       */
  float separation;              /* far-near L2 latency gap / spread; <1 =
                                    the die split is not trustworthy       */
  float near_cycles;             /* mean same-die L2 hit latency            */
  float far_cycles;              /* mean cross-die L2 hit latency           */
} mk_topology;

/* One task descriptor (64 bytes).  graph tasks keep graph order. */
typedef struct mk_task {
  int32_t op;         /* MK_OP_*                                              */
  int32_t level;      /* MK_LEVEL_*                                           */
  int32_t die;        /* chiplet binding, -1 otherwise                        */
  int32_t wait0;      /* event ids, -1 = none                                 */
  int32_t wait1;
  int32_t signal;     /* event id, -1 = none                                  */
  int32_t n_items;    /* work items of a CU task (fan-out); 0 for chiplet     */
  int32_t n_units;    /* dispatch units the items are grouped into            */
  int32_t sub_ctr;    /* sub-counter for multi-unit CU tasks, -1 otherwise    */
  int32_t param_off;  /* byte offset of the op parameter block (8-aligned)    */
  int32_t layer;
  int32_t graph_index;/* index in TaskGraph.tasks, -1 for appended tasks     */
  int32_t pad[4];
} mk_task;

/* One dispatch unit: a chiplet task, or a contiguous item range of a CU task */
typedef struct mk_unit {
  int32_t task;
  int32_t item_begin;
  int32_t item_end;
  int32_t pad;
} mk_unit;

/* Op parameter blocks (all 8-byte aligned, pointers first). */
typedef struct mk_gemm_params {
  const void* w;      /* packed bf16 weights of this task (slab / tile set)   */
  const void* x;      /* activations, bf16 [M][ldx]                           */
  void* y;            /* output: bf16 [M][ldy] (fp32 for LOGITS)              */
  const void* res;    /* residual bf16 [M][ldres] or NULL                     */
  float* amax_val;    /* LOGITS: per-(worker,row) running max                 */
  int32_t* amax_idx;  /* LOGITS: per-(worker,row) argmax                      */
  const void* norm_gamma; /* fused RMSNorm of x while staging (NULL = none)  */
  int32_t M, K, N;    /* N = weight rows of this task (N_local)               */
  int32_t T_M, T_N, T_K;
  int32_t ldx, ldy, ldres;
  int32_t y_col0;     /* first output column written by this task           */
  int32_t epilogue;   /* MK_EPI_*                                            */
  int32_t traversal;  /* MK_TRAV_*                                            */
  int32_t distribution;/* MK_DIST_*                                          */
  int32_t xcd;        /* die binding (M_SPLIT row rotation)                   */
  int32_t tile_m;     /* CU tile task: its tile; -1 for a die task          */
  int32_t tile_n;
  int32_t amax_base;  /* LOGITS: first worker slot of this task             */
  int32_t amax_stride;/* LOGITS: rows per worker slot                       */
  int32_t stage_x;    /* 1: stage x rows in shared memory per m-tile          */
  float norm_eps;
  int32_t body;       /* MK_BODY_*: CUDA-core warp-row GEMV or tcgen05 UMMA   */
  int32_t y_cols;     /* valid output columns of y (masks padded LM-head rows) */
  int32_t ksplit;     /* 1: die-task K-split -- worker w owns K-chunk slots
                         [w*S/W, (w+1)*S/W) of the traversal order
                         (PAPER.md:569-573); 0: whole tiles per
                         schedule() (traversal.py:125-202)             */
  int32_t tile_ctr0;  /* K-split: first per-tile arrival sub-counter      */
  int32_t piece_floats;/* K-split: floats per partial piece               */
  int32_t ss_nparts;  /* tcgen05 folded RMSNorm: partial sums per row in ss_in */
  float* kpart;       /* K-split: partial pieces [W][2][piece_floats] fp32 */
  float* ss_out;      /* tcgen05 residual epilogue: per (128-col tile, TMEM
                         quadrant) sums of squares of the bf16 output,
                         [d/128*4][M] -- the next RMSNorm's statistics     */
  const float* ss_in; /* tcgen05 GEMM after an RMSNorm folded into its
                         weights (W * gamma): [ss_nparts][M] partials; the
                         epilogue scales row b by rsqrt(sum/K + eps)       */
} mk_gemm_params;

typedef struct mk_norm_params {
  const void* x;       /* bf16 [M][d] (ignored when embed != NULL)           */
  const void* gamma;   /* bf16 [d]                                           */
  void* y;             /* bf16 [M][d]                                        */
  const void* embed;   /* L0 only: bf16 [vocab][d]                           */
  const int32_t* tokens;/* L0 only: [M]                                      */
  void* x_store;       /* L0 only: gathered rows -> residual stream          */
  int32_t M, d;
  float eps;
  int32_t fused;       /* 1: the consuming GEMM normalises; only gather here */
  float* ss_out;       /* fused + L0 gather: each row's sum of squares [M]   */
} mk_norm_params;

typedef struct mk_attn_params {
  const void* qkv;     /* bf16 [M][ldqkv]: q | k | v                          */
  const void* q_gamma; /* bf16 [head_dim]                                    */
  const void* k_gamma;
  void* k_cache;       /* bf16 [M][kv_heads][t_max][head_dim] (this layer)   */
  void* v_cache;
  const float* rope_cos; /* fp32 [t_max][head_dim/2]                          */
  const float* rope_sin;
  const int32_t* positions; /* [M]: index of the token being decoded        */
  float* partial;      /* fp32 [M][kv_heads][n_splits][group][head_dim+4]   */
  void* out;           /* ATTN_REDUCE: bf16 [M][q_heads*head_dim]            */
  int32_t M, ldqkv;
  int32_t q_heads, kv_heads, head_dim, group;
  int32_t kv_head;     /* which kv head this task covers                     */
  int32_t split;       /* tokens per split (S)                                */
  int32_t n_splits;    /* splits per row allocated (t_max / S)                */
  int32_t t_max;
  float eps, scale;
  int32_t sub_splits;  /* warps sharing one (item, head) -- or, on the
                          tensor-core path, warps per item (1, 2, 4)        */
  int32_t mma;         /* 1: tensor-core path (head_dim 128, 64-token splits,
                          group <= 4; K/V rows chunk-swizzled)             */
  int32_t fuse_reduce; /* 1: ATTN_PARTIAL: the last split of a row merges all
                          splits into `out` (per-row arrival counters at
                          red_ctr0); ATTN_REDUCE: no-op                    */
  int32_t red_ctr0;    /* first per-row arrival sub-counter                 */
  const int32_t* page_table; /* paged KV (NULL = contiguous rows): [M][max_pages]
                          physical page of every `split`-token block of a row;
                          k_cache / v_cache are then page pools
                          [n_pages][kv_heads][split][head_dim]            */
  int32_t max_pages;   /* pages per row (t_max / split)                     */
  int32_t prefill;     /* 1: chunked prefill -- the M rows are consecutive
                          tokens of ONE sequence (positions p0..p0+M-1, the
                          same pages): every item also folds the chunk's
                          earlier tokens into its K/V slots (tensor-core
                          path, M <= 64)                                   */
} mk_attn_params;

typedef struct mk_silu_params {
  const void* gu;      /* bf16 [M][2F]: gate | up                            */
  void* y;             /* bf16 [M][F]                                         */
  int32_t F, row0, rows, col0, cols, pad;
} mk_silu_params;

typedef struct mk_argmax_params {
  const float* amax_val;   /* [n_slots][M]                                    */
  const int32_t* amax_idx;
  int32_t* out_tokens;     /* [M] this step's greedy tokens                   */
  int32_t* next_tokens;    /* [M] input of the next step (may alias)          */
  int32_t* positions;      /* [M] advanced by one                             */
  int32_t M, n_slots;
} mk_argmax_params;

/* MK_OP_TP_ALLREDUCE (units split the d/8 column chunks) and
 * MK_OP_TP_ARGMAX (one unit, all rows).  Offsets are bytes into the
 * exchange region, identical on every rank (mk_tp_init). */
typedef struct mk_tp_params {
  int64_t recv_off;    /* ALLREDUCE: fp32 [world][M][d] partials of this point  */
  int64_t flag_off;    /* uint32 [world]: epoch each rank announced this point  */
  int64_t gather_off;  /* ARGMAX: {float val, int32 idx} [world][M]              */
  const void* res;     /* ALLREDUCE: bf16 residual [M][d]                       */
  void* y;             /* ALLREDUCE: bf16 [M][d] = res + sum_rank partial       */
  const float* amax_val;   /* ARGMAX: local LM-head shard slots [n_slots][M]    */
  const int32_t* amax_idx;
  int32_t* out_tokens;
  int32_t* next_tokens;
  int32_t* positions;
  int32_t M, d, n_slots, vocab0;  /* vocab0: first global row of this shard  */
} mk_tp_params;

typedef struct mk_graph_desc {
  int32_t n_tasks;
  int32_t n_events;
  int32_t n_units;
  int32_t n_sub_ctrs;
  int32_t n_schedulers;      /* = num dies (PER_DIE) or 1 (FLAT)              */
  int32_t sched_mode;        /* MK_SCHED_*                                    */
  int32_t workers_per_sched; /* W: workers each scheduler drives              */
  int32_t param_bytes;
  const mk_task* tasks;      /* host arrays, copied by mk_create              */
  const int32_t* event_required; /* [n_events]                                */
  const mk_unit* units;      /* units grouped per scheduler, topological order */
  const int32_t* sched_begin;/* [n_schedulers+1] offsets into units           */
  const void* params;        /* param blob                                    */
  const int32_t* positions;  /* device [n_rows]: decode position of every row,
                                read once per launch (borrowed)               */
  int32_t n_rows;
  int32_t pad;
  int32_t* tokens;           /* device [n_rows]: token ids this step decodes
                                (borrowed; written by mk_step_tokens)        */
  const int32_t* out_tokens; /* device [n_rows]: greedy ids the step emits     */
} mk_graph_desc;

typedef struct mk_counters {
  uint64_t dispatches;      /* units dispatched (one per chiplet broadcast)   */
  uint64_t mailbox_writes;  /* worker mailbox entries written                 */
  uint64_t global_atomics;  /* event-counter increments                       */
  uint64_t local_atomics;   /* die-local completion increments                */
  uint64_t fences;          /* gpu-scope fences before a global increment     */
  uint64_t fanout_atomics;  /* sub-counter increments of multi-unit CU tasks  */
  uint64_t polls;           /* acquire loads spent waiting on events          */
  uint64_t tiles;           /* GEMM tiles computed                            */
  uint64_t executions;      /* (unit, worker) executions                      */
  uint64_t steps;
  /* diagnostics (mk_set_debug bit 2): SM cycles spent waiting, summed */
  uint64_t wait_ring_empty; /* fetch warp: ring slot not yet released          */
  uint64_t wait_mma_full;   /* MMA lane: weight slot not yet landed            */
  uint64_t wait_mma_x;      /* MMA lane: activation chunk not yet landed       */
  uint64_t wait_mma_tmem;   /* MMA lane: accumulator buffer not yet drained    */
  uint64_t wait_epi_done;   /* epilogue: accumulator not yet complete          */
  uint64_t mma_chunks;      /* K-chunks issued by MMA lanes                    */
} mk_counters;

/* Event-log record (one per executed unit per worker, plus scheduler
 * dispatch records).  kind: 0 = dispatch, 1 = execute. */
typedef struct mk_log_rec {
  int32_t kind;
  int32_t task;
  int32_t item_begin;
  int32_t worker;      /* global worker id, or -1-scheduler for dispatches */
  int32_t smid;
  int32_t die;
  uint64_t t_start;    /* %globaltimer ns                                   */
  uint64_t t_end;
} mk_log_rec;

typedef struct mk_handle mk_handle;

int mk_probe(int device, mk_topology* out);
/* Raw probe data: L2-hit latency (cycles) [MK_MAX_SMS][n_lines] by %smid. */
int mk_probe_raw(int device, uint32_t* lat_out, int32_t* n_lines_out);
int mk_create(int device, const mk_graph_desc* g, const mk_topology* topo,
              mk_handle** out);
/* One decode step (one cooperative launch) on `stream` (cudaStream_t, may be
 * NULL).  Asynchronous: check mk_sync() for the watchdog verdict. */
int mk_step(mk_handle* h, void* stream);
/* One decode step with host token buffers: copies
 * `tokens_in` [n_rows] host->device, launches, copies the greedy ids
 * device->host into `tokens_out`, all on `stream`; completes at mk_sync /
 * stream synchronisation (pinned host memory for true asynchrony). */
int mk_step_tokens(mk_handle* h, void* stream, const int32_t* tokens_in, int32_t* tokens_out);
int mk_sync(mk_handle* h);
int mk_counters_get(mk_handle* h, mk_counters* out);
int mk_counters_reset(mk_handle* h);
/* Enable the device event log with room for `capacity` records (0 = off). */
int mk_log_enable(mk_handle* h, int64_t capacity);
int64_t mk_log_read(mk_handle* h, mk_log_rec* out, int64_t max_records);
/* Optional tile log: (task, worker, m, n) per GEMM tile (0 = off). */
int mk_tile_log_enable(mk_handle* h, int64_t capacity);
int64_t mk_tile_log_read(mk_handle* h, int32_t* out4, int64_t max_records);
/* Per-unit phase stamps (diagnostics; 0 = off): for every unit a worker
 * executes, 8 uint64 words {task | item_begin << 32, poll start, dependency
 * acquired, body start (GEMM operands staged), consumer 0 done, all
 * consumers done, completion signalled, sequence number}, %globaltimer ns,
 * laid out [scheduler][worker][units_per_worker][8].  mk_trace_read returns
 * the total word count. */
int mk_trace_enable(mk_handle* h, int32_t units_per_worker);
int64_t mk_trace_read(mk_handle* h, uint64_t* out, int64_t max_words);
int mk_set_watchdog(mk_handle* h, double seconds);
/* L2 prefetch run-ahead of each worker (CUDA-core kernel instance), in
 * 16 KiB ring slots beyond the fetch warp (0 = off): weight slots of queued
 * GEMM units are prefetched into L2 while the worker waits on dependencies. */
int mk_set_prefetch(mk_handle* h, int slots);
/* Diagnostics only: bit0 = consumers skip GEMM math, bit1 = no TMA copies,
 * bit2 = count wait cycles (mk_counters wait_*). */
int mk_set_debug(mk_handle* h, int flags);
/* Tensor parallelism: `peer_bases[q]` is rank q's
 * exchange region as addressable from this device (peer-mapped /
 * IPC-opened; peer_bases[rank] = own region).  Call before the first step. */
int mk_tp_init(mk_handle* h, int rank, int world, void* const* peer_bases);
/* Exchange regions: plain cudaMalloc (IPC-exportable), zero-filled. */
int mk_tp_alloc(int device, size_t bytes, void** out);
int mk_tp_free(void* ptr);
/* CUDA IPC handle (64 bytes) of an mk_tp_alloc region / open a peer's. */
int mk_ipc_export(void* ptr, uint8_t* handle64);
int mk_ipc_import(int device, const uint8_t* handle64, void** out);
int mk_ipc_close(void* ptr);
/* Launch geometry override (before the first step): `ctas` CTAs (flat
 * scheduler only: workers <= ctas - 1) and cooperative (1) or plain (0)
 * launches -- several ranks of a TP group can then share one GPU, each on
 * its own subset of SMs (single-GPU test of the device TP path). */
int mk_set_grid(mk_handle* h, int ctas, int cooperative);
int mk_destroy(mk_handle* h);
const char* mk_last_error(void);
int mk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MK_H */
