// mk_kernel.cu -- the persistent hierarchical-task megakernel (sm_100a).
//
// One cooperative launch = one decode step.  grid = #SMs, one CTA per SM
// (dynamic shared memory forces it).  Each CTA reads %smid, looks up its die
// in the probed table and takes a role:
//
//   rank 0 of a die  -> scheduler CTA of that die (PER_DIE) -- or rank 0 of
//                       the GPU in FLAT mode (die-unaware baseline)
//   rank 1..W        -> worker w = rank-1 of that scheduler
//
// Scheduler (one warp): walks its die's dispatch list (topological order,
// host-lowered from the TaskGraph) and writes worker mailboxes: a die task
// (reference CHIPLET level) is broadcast to all W workers of its die, a CU
// task unit goes to the next worker round-robin (ref runtime.py:301-307,
// 373-417).  It does not wait for dependencies: dispatch runs ahead so the
// workers can stream weights early; dependencies are resolved by the worker
// with gpu-scope acquire loads on the event counters.
//
// Worker: warp 0 is the fetch warp -- it reads the mailbox, forwards units to
// the consumer warps through a shared-memory queue, and streams every weight
// tile (and every cached K/V block) the unit will need into a 12-slot shared
// memory ring with TMA bulk copies (L2 evict_first), ignoring dependencies
// (weights and past KV are immutable during the step).  Warps 1..8 are the
// consumers: wait on the unit's events, run the op body, signal completion
// with two-level counting (ref runtime.py:432-480):
//   die task : atom.acq_rel on the die-local counter; the W-th arrival on
//              the die issues fence.acq_rel.gpu + red.release.gpu on the
//              event counter (one fence + one global atomic per die per event)
//   CU task  : red.release.gpu on the event counter (fanned-out CU tasks count
//              their units on a sub-counter first).
//
// Counters are monotone across launches: the event fires in step e (epoch,
// 1-based) when counter >= required * e, so no per-step reset is needed.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <string>
#include <algorithm>
#include <type_traits>

#include "mk.h"
#include "mk_ptx.cuh"

namespace mk {

constexpr int kConsWarps = 8;
constexpr int kCons = kConsWarps * 32;          // consumer threads
constexpr int kProdThreads = 128;              // producer warpgroup (warp 0 fetches)
constexpr int kThreads = kCons + kProdThreads;  // 12 warps = 3 warpgroups
constexpr int kProdRegs = 88;                   // setmaxnreg budget: 128*88 + 256*200
constexpr int kConsRegs = 200;                  //   = 62464 <= 65536
constexpr int kProdRegsUmma = 104;              // tcgen05 instance: 128*104 + 256*200
constexpr int kConsRegsUmma = 200;              //   = 64512 = the 168 x 384 the launch holds
constexpr int kSlotBytes = 16384;
constexpr int kSlots = 10;
constexpr int kXsBytes = 49152;                 // staged activations per task / x ring
constexpr int kMaxSplits = 128;                 // split-KV splits per row
constexpr int kMaxPieces = 512;                 // splits x token subsets
constexpr int kXStagesMax = 16;                 // UMMA activation ring: up to 16 stages of
                                                //   NT rows x 64 bf16 (128B-swizzled), TMA-fed
// TMEM: 2 accumulator buffers (segments double-buffered) x 4 independent
// accumulators x 64 columns.  The 4 MMAs of a K-chunk go to 4 different
// accumulators: back-to-back skinny MMAs (N <= 64) into ONE accumulator are
// bound by the dependent-accumulate latency (measured ~900 cycles per
// chunk at N = 16 and N = 64 alike), not by the tensor pipe.
constexpr int kAccs = 4;
constexpr int kAccCols = 64;
constexpr int kBufCols = kAccs * kAccCols;
constexpr int kTmemCols = 2 * kBufCols;
constexpr int kTQ = 32;                         // smem unit queue depth
constexpr int kPBytes = 192;                    // param block bytes cached per queued unit
constexpr int kPosRows = 256;                   // decode positions cached per CTA
constexpr int kMailbox = 64;                    // mailbox depth per worker
constexpr uint32_t kEnd = 0xFFFFFFu;
constexpr int kMaxNB = 16;
// Kernel instances: feature bits select the op bodies compiled into one
// instance, so a small-batch graph runs a kernel without the tcgen05 and
// K-split code (smaller code, same register allocation as the plain GEMV).
constexpr int kFeatUmma = 1;      // tcgen05 GEMM body, MMA warp, TMEM
constexpr int kFeatKsplit = 2;    // K-split die tasks (partial pieces)
// Lean instances: only the op bodies a batch-1 GEMV graph (F = Lean|Ksplit)
// or an all-tcgen05 graph (F = Lean|Umma|Ksplit) executes.  The general
// instances carry every batch width's unrolled GEMV body (0.1-0.24 M SASS
// instructions, 1.7-3.9 MB of code); each op switch of a decode step then
// refetches its code through the instruction caches from L2 while HBM
// streams.
constexpr int kFeatLean = 4;
constexpr int kAmaxRows = 64;

enum StatIdx {
  S_DISPATCH = 0, S_MAILBOX, S_GLOBAL, S_LOCAL, S_FENCE, S_FANOUT, S_POLL,
  S_TILES, S_EXEC, S_STEPS,
  // debug bit 2: cycles spent waiting, per role (diagnostics)
  S_W_RING_EMPTY, S_W_MMA_FULL, S_W_MMA_X, S_W_MMA_TMEM, S_W_EPI_DONE, S_MMA_CHUNKS, S_N
};

struct KArgs {
  const mk_task* tasks;
  const mk_unit* units;
  const int32_t* sched_begin;
  const uint8_t* params;
  uint32_t* ev_ctr;
  const int32_t* ev_req;
  const int32_t* ev_dmask; // per event: bit g = signalled by one die task of group g (and
                           // by nothing else): waiters poll those die counters directly
  uint32_t* die_ctr;       // [n_events][n_sched]
  uint32_t* sub_ctr;
  uint64_t* mailbox;       // [n_sched*W][kMailbox]
  uint64_t* mb_head;       // consumer progress per worker (persistent)
  uint64_t* mb_tail;       // scheduler progress per worker (persistent)
  const int8_t* die_of_sm;
  uint32_t* role_ctr;      // [n_groups]
  const int32_t* group_size;
  unsigned long long* stats;
  mk_log_rec* log;
  unsigned long long* log_cursor;
  long long log_cap;
  int32_t* tile_log;
  unsigned long long* tile_cursor;
  long long tile_cap;
  int* err;
  int* err_info;
  unsigned long long watchdog_ns;
  int n_events;
  int n_sched;
  int sched_mode;
  int W;
  uint32_t epoch;
  int debug;               // bit0: consumers skip GEMM math, bit1: fetch issues no TMA
  int use_umma;            // graph has tcgen05 GEMM tasks: allocate TMEM, run the MMA warp
  const CUtensorMap* tmaps; // [n_tasks]: activation (x) tensor map of each tcgen05 GEMM task
  int x_stages;            // x ring stages of two chunks (kXsBytes / (2 x_stage_bytes))
  int x_stage_bytes;       // one chunk: 128 * max NT over the graph's tcgen05 tasks
  int pf_slots;            // L2 prefetch run-ahead of the prefetch warp (16 KiB slots)
  const int32_t* positions; // decode position per row (read once per launch into smem)
  int n_rows;
  uint64_t* trace;         // per-unit phase stamps [worker][trace_cap][8] (mk_trace_enable)
  int trace_cap;
  // tensor parallelism (mk_tp_init): exchange region of every rank as
  // addressable from this device; tp_peer[tp_rank] is this rank's own
  int tp_world, tp_rank;
  uint8_t* tp_peer[MK_MAX_TP];
};

struct AttnScratch {
  float xch[8][132];                // sub-warp partial state exchange
};

struct Smem {
  uint64_t full[kSlots];
  uint64_t empty[kSlots];
  uint32_t slot_tag[kSlots];        // ring position last loaded into each slot
  uint64_t tq_full[kTQ];
  uint64_t tq_empty[kTQ];
  int4 tq[kTQ];
  float amx_val[kConsWarps][kAmaxRows];   // LM head: per-warp running max per row
  int amx_idx[kConsWarps][kAmaxRows];
  float bred[32];
  int ibred[32];
  float rsum[kConsWarps][kMaxNB];   // x-staging: per-warp sums of squares
  float rs[kMaxNB];                 // x-staging: 1/rms per staged row
  float rsn[kAmaxRows];             // tcgen05 folded RMSNorm: 1/rms per batch row
  int4 cur;                         // consumer broadcast: current unit
  int abort_flag;
  int piece_last;                   // K-split: this CTA summed the tile's pieces (GEMV)
  int epi_last;                     // K-split: same, tcgen05 epilogue warps
  uint32_t ring_pos;                // slots the fetch warp has issued (prefetch warp's bound)
  // tcgen05 path
  uint64_t xfull[kXStagesMax], xempty[kXStagesMax];
  uint64_t tile_done[2], tmem_free[2];
  uint64_t job_full;
  int4 job;                         // {task, worker-in-task, first ring slot, 0}
  uint64_t tr[8];                   // phase stamps of the current unit (trace)
  uint64_t xs_bar;                  // hoisted x / gamma staging (TMA bulk copies)
  int xs_hoist;                     // the current unit's x rows (+ gamma) are in flight to u.xs
  uint32_t xs_parity;               //   ... on this phase of xs_bar
  uint32_t tmem_base;
  // Descriptor cache: the mailbox warp copies every queued unit's task
  // descriptor and parameter block here, so no role reads them from global
  // memory on the critical path (an acquire poll invalidates L1, and an L2
  // round trip costs 1-3 us while HBM streams).  pad[0..1] of the cached
  // task hold ev_req of its wait events.
  int32_t pos[kPosRows];            // positions[] at launch (advanced only by the last task)
  int32_t n_pos;                    // rows cached in pos[]
  alignas(16) mk_task tcache[kTQ];
  uint64_t pcache[kTQ][kPBytes / 8];
  union __align__(1024) {            // 1024: 128B-swizzle atoms of the x ring
    AttnScratch at;
    uint16_t xs[kXsBytes / 2];      // GEMM: staged (normalised) activations
  } u;
};

// Scheduler CTAs never use the ring: their mailbox cursors live there.
struct SchedSmem {
  uint64_t tail[MK_MAX_SMS];
  uint64_t head[MK_MAX_SMS];
};

constexpr size_t kRingOffset = (sizeof(Smem) + 1023) / 1024 * 1024;

// Tensor-core split-KV attention (attn_mma_pass) applies to head_dim 128
// with 64-token splits and up to 4 query heads per kv head.
constexpr int kAttnHD = 128;
constexpr int kAttnSplit = 64;
constexpr int kAttnMaxG = 4;                   // query heads per kv head on this path
constexpr int kChunkRows = 64;                  // chunked prefill: tokens per launch

__host__ __device__ __forceinline__ bool attn_mma_path(const mk_attn_params& p) {
  return p.mma != 0 && p.head_dim == kAttnHD && p.split == kAttnSplit && p.group <= kAttnMaxG;
}


constexpr size_t kSmemBytes = kRingOffset + size_t(kSlots) * kSlotBytes;
static_assert(kSmemBytes <= 232448, "megakernel shared memory exceeds the 227 KB per-CTA limit");
static_assert(kPBytes == 24 * 8, "the mailbox warp copies 24 param words (lanes 8..31)");

// Build split (see __graft_entry__.build): the device code below is compiled
// once per kernel instance (-DMK_INSTANCE=F, explicit instantiation at the
// end of the file), the host ABI once (-DMK_HOST_TU) against a declaration.
#ifndef MK_HOST_TU
namespace {   // device helpers: internal linkage (compiled into every instance TU)

// Phase stamp of the current unit (mk_trace_enable): consumer thread 0 only.
#define MK_TRACE(a, s, ct, i) \
  do { if ((a).trace && (ct) == 0) (s).tr[i] = globaltimer(); } while (0)

__device__ __forceinline__ bool aborted(const KArgs& a) {
  return *reinterpret_cast<volatile int*>(a.err) != 0;
}

__device__ __noinline__ void raise_error(const KArgs& a, int code, int info) {
  if (atomicCAS(a.err, 0, code) == 0) *a.err_info = info;
}
__device__ __forceinline__ void raise_deadlock(const KArgs& a, int info) {
  raise_error(a, MK_ERR_DEADLOCK, info);
}
// A decode position outside the allocated KV rows: reported as a config
// error (info = -100 - row) instead of indexing past the cache / RoPE table.
__device__ __forceinline__ bool pos_ok(const KArgs& a, int pos, int t_max, int row) {
  if (pos >= 0 && pos < t_max) return true;
  raise_error(a, MK_ERR_CONFIG, -100 - row);
  return false;
}

// Has event e fired in this launch?  req = ev_req[e] (n_units in sub-counter
// mode), dmask = ev_dmask[e]: > 0 die counters, < 0 the sub-counter -1-dmask
// (both cached in the task descriptor by the mailbox warp).  ACQ: acquire
// loads; otherwise relaxed (the caller fences once).
template <bool ACQ>
__device__ __forceinline__ bool ev_done(const KArgs& a, int e, int32_t req, int32_t dmask) {
  if (dmask > 0) {
    const uint32_t target = uint32_t(a.W) * a.epoch;
    for (int g = 0; g < a.n_sched; ++g) {
      if (!((dmask >> g) & 1)) continue;
      const uint32_t* c = &a.die_ctr[size_t(e) * a.n_sched + g];
      if ((int32_t)((ACQ ? ld_acquire(c) : ld_relaxed(c)) - target) < 0) return false;
    }
    return true;
  }
  const uint32_t target = uint32_t(req) * a.epoch;
  const uint32_t* c = dmask < 0 ? &a.sub_ctr[-1 - dmask] : &a.ev_ctr[e];
  return (int32_t)((ACQ ? ld_acquire(c) : ld_relaxed(c)) - target) >= 0;
}

// Spin helper: returns false if the watchdog fired / the launch aborted.
struct Spin {
  uint64_t t0 = 0;
  uint32_t n = 0;
  __device__ __forceinline__ bool ok(const KArgs& a, int info) {
    if ((++n & 255u) == 0) {
      if (aborted(a)) return false;
      uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > a.watchdog_ns) { raise_deadlock(a, info); return false; }
    }
    return true;
  }
};

__device__ __forceinline__ bool mbar_wait(const KArgs& a, uint64_t* bar, uint32_t parity, int info) {
  Spin sp;
  while (!mbar_try_wait(bar, parity)) {
    if (!sp.ok(a, info)) return false;
  }
  return true;
}

// Latency-critical single-role waits (fetch warp, MMA warp): spin on the
// non-suspending test_wait -- a suspended try_wait is only woken after a
// delay, which paces a ring handshake at the wake-up latency.
__device__ __forceinline__ bool mbar_spin(const KArgs& a, uint64_t* bar, uint32_t parity, int info) {
  Spin sp;
  while (!mbar_test_wait(bar, parity)) {
    if (!sp.ok(a, info)) return false;
  }
  return true;
}

// Long waits of whole warps: lane 0 polls with a nanosleep backoff, the warp
// then reconverges -- 32 spinning lanes per warp would flood the SM's
// mbarrier unit and slow the latency-critical single-lane roles.
__device__ __forceinline__ void mbar_wait_warp(const KArgs& a, uint64_t* bar, uint32_t parity, int info) {
  if ((threadIdx.x & 31) == 0) {
    Spin sp;
    uint32_t ns = 32;
    while (!mbar_try_wait(bar, parity)) {
      if (!sp.ok(a, info)) break;
      __nanosleep(ns);
      ns = ns < 512 ? ns * 2 : 512;
    }
  }
  __syncwarp();
  mbar_try_wait(bar, parity);   // every lane observes the completed phase
}

// mbar_wait that adds the cycles it spent to `acc` when debug bit 2 is set
__device__ __forceinline__ bool mbar_wait_p(const KArgs& a, uint64_t* bar, uint32_t parity, int info,
                                            unsigned long long& acc) {
  if (!(a.debug & 4)) return mbar_spin(a, bar, parity, info);
  const long long t0 = clock64();
  const bool ok = mbar_spin(a, bar, parity, info);
  acc += (unsigned long long)(clock64() - t0);
  return ok;
}

// Decode position of row b: the launch-time smem copy (positions change only
// in the step's final ARGMAX task), global memory beyond kPosRows rows.
__device__ __forceinline__ int row_pos(const int32_t* gpos, int b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem& s = *reinterpret_cast<const Smem*>(smem_raw);
  return b < s.n_pos ? s.pos[b] : gpos[b];
}

// Parameter block of a task descriptor from the smem cache (t must be one of
// Smem::tcache: the block sits in the matching pcache entry).
template <typename T>
__device__ __forceinline__ const T* P(const KArgs& a, const mk_task& t) {
  static_assert(sizeof(T) <= size_t(kPBytes), "param block exceeds the descriptor cache");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Smem& s = *reinterpret_cast<const Smem*>(smem_raw);
  (void)a;
  return reinterpret_cast<const T*>(s.pcache[&t - s.tcache]);
}

// Element offset of token `tok`'s row (kv head p.kv_head, sequence b) in the
// KV cache: contiguous [M][kv_heads][t_max][hd], or -- paged KV -- the
// row's page of `split` tokens in the pool [n_pages][kv_heads][split][hd].
__device__ __forceinline__ size_t kv_off(const mk_attn_params& p, int b, int tok) {
  if (p.page_table) {
    const int pg = p.page_table[size_t(b) * p.max_pages + tok / p.split];
    return ((size_t(pg) * p.kv_heads + p.kv_head) * p.split + tok % p.split) * p.head_dim;
  }
  return ((size_t(b) * p.kv_heads + p.kv_head) * p.t_max + tok) * p.head_dim;
}

// MK_EPI_PARTIAL: one fp32 partial-product element pushed into every rank's
// exchange region (this rank's slot: byte offset p.y, row-major [M][ldy]).
// Remote stores are posted over NVLink; the unit fences at system scope
// before it signals (tp_partial_done), so the TP_ALLREDUCE announcement that
// follows the local event orders them for the peers.
__device__ __forceinline__ void tp_store(const KArgs& a, const mk_gemm_params& p, int row, int col,
                                         float v) {
  const size_t off = reinterpret_cast<size_t>(p.y) + (size_t(row) * p.ldy + col) * 4;
  for (int q = 0; q < a.tp_world; ++q)
    __stcg(reinterpret_cast<float*>(a.tp_peer[q] + off), v);
}

// ---------------------------------------------------------------------------
// Tile iteration shared by the fetch warp and the consumers (ref
// traversal.py:125-202 restated as an owner-inverse loop).
// ---------------------------------------------------------------------------
struct TileIter {
  int mt, nt, W, w, trav, dist, xcd;
  int idx, row, n, fixed_m, fixed_n, done;
  __device__ __forceinline__ void init(const mk_gemm_params& p, int workers, int worker) {
    const int rows_per_out = (p.epilogue == MK_EPI_SILU) ? 2 : 1;
    mt = (p.M + p.T_M - 1) / p.T_M;
    nt = p.N / (p.T_N * rows_per_out);
    W = workers; w = worker; trav = p.traversal; dist = p.distribution;
    xcd = p.xcd; fixed_m = p.tile_m; fixed_n = p.tile_n; done = 0;
    idx = w; row = 0; n = w;
  }
  __device__ __forceinline__ bool next(int& m_out, int& n_out) {
    if (fixed_m >= 0) {              // standard-mode CU tile task
      if (done) return false;
      done = 1; m_out = fixed_m; n_out = fixed_n; return true;
    }
    if (dist == MK_DIST_M_SPLIT) {
      while (row < mt) {
        if (n < nt) {
          m_out = (xcd % mt + row) % mt; n_out = n; n += W; return true;
        }
        ++row; n = w;
      }
      return false;
    }
    if (idx >= mt * nt) return false;
    if (trav == MK_TRAV_M_MAJOR) { m_out = idx % mt; n_out = idx / mt; }
    else { m_out = idx / nt; n_out = idx % nt; }
    idx += W;
    return true;
  }
};

__device__ __forceinline__ int gemm_rows(const mk_gemm_params& p) {
  return p.T_N * (p.epilogue == MK_EPI_SILU ? 2 : 1);
}

// ---------------------------------------------------------------------------
// K-split range partition of a die task ("K-split", done on
// B200 across the die's worker CTAs).  The traversal's tile order (the same
// (m, n) sequence schedule() walks, traversal.py:125-202) is refined into its
// K-chunks -- one 16 KiB ring slot each -- and worker w owns the contiguous
// slot range [w*S/W, (w+1)*S/W).  Every worker streams the same number of
// weight bytes whatever the tile count; consecutive workers still share
// weight columns in M-major order.  A tile cut by a range boundary is
// computed as partial pieces (fp32, per worker) and the last-arriving piece
// sums them in piece order (deterministic) and runs the epilogue.
// ---------------------------------------------------------------------------
struct Seg {
  int tile, m, n, c0, c1;
  bool first;          // the worker's first segment (its piece slot 0)
};

__device__ __forceinline__ void tile_mn(const mk_gemm_params& p, int mt, int nt, int idx,
                                        int& m, int& n) {
  if (p.distribution == MK_DIST_M_SPLIT) { m = (p.xcd % mt + idx / nt) % mt; n = idx % nt; }
  else if (p.traversal == MK_TRAV_M_MAJOR) { m = idx % mt; n = idx / mt; }
  else { m = idx / nt; n = idx % nt; }
}

struct RangeIter {
  int mt, nt, chunks;
  long long s0, s1, s;
  const mk_gemm_params* p;
  __device__ __forceinline__ void init(const mk_gemm_params& pp, int W, int w) {
    p = &pp;
    mt = (pp.M + pp.T_M - 1) / pp.T_M;
    nt = pp.N / gemm_rows(pp);
    chunks = pp.K / pp.T_K;
    const long long S = (long long)mt * nt * chunks;
    s0 = S * w / W; s1 = S * (w + 1) / W; s = s0;
  }
  __device__ __forceinline__ bool next(Seg& g) {
    if (s >= s1) return false;
    g.tile = int(s / chunks);
    g.c0 = int(s % chunks);
    g.c1 = int(min((long long)chunks, g.c0 + (s1 - s)));
    g.first = s == s0;
    tile_mn(*p, mt, nt, g.tile, g.m, g.n);
    s += g.c1 - g.c0;
    return true;
  }
  __device__ long long slots() const { return s1 - s0; }
};

// Uniform segment walk: K-split ranges, or the reference's whole-tile
// ownership (TileIter) as single full-K segments.
struct SegIter {
  bool ks;
  RangeIter ri;
  TileIter ti;
  int chunks;
  __device__ __forceinline__ void init(const mk_gemm_params& p, int W, int w) {
    ks = p.ksplit != 0;
    chunks = p.K / p.T_K;
    if (ks) ri.init(p, W, w); else ti.init(p, W, w);
  }
  __device__ __forceinline__ bool next(Seg& g) {
    if (ks) return ri.next(g);
    if (!ti.next(g.m, g.n)) return false;
    g.tile = -1; g.c0 = 0; g.c1 = chunks; g.first = true;
    return true;
  }
};

// Which worker owns slot s (inverse of w*S/W).
__device__ __forceinline__ int range_owner(long long s, long long S, int W) {
  return int(((s + 1) * W + S - 1) / S) - 1;
}

// The pieces of a cut tile: the non-empty worker ranges between the owners
// of its first and last slot (with more workers than slots some ranges in
// between are empty and contribute nothing).
struct PieceInfo {
  int first_w, last_w, n, slot0;   // owners, piece count, piece-slot of first_w
  long long S;
  int W;
  __device__ __forceinline__ bool empty(int w) const {
    return S * w / W == S * (w + 1) / W;
  }
};

__device__ __forceinline__ PieceInfo tile_pieces(const mk_gemm_params& p, int W, int tile) {
  const int mt = (p.M + p.T_M - 1) / p.T_M, nt = p.N / gemm_rows(p), chunks = p.K / p.T_K;
  PieceInfo pi;
  pi.S = (long long)mt * nt * chunks;
  pi.W = W;
  const long long a = (long long)tile * chunks, b = a + chunks - 1;
  pi.first_w = range_owner(a, pi.S, W);
  pi.last_w = range_owner(b, pi.S, W);
  pi.n = 0;
  for (int w = pi.first_w; w <= pi.last_w; ++w) pi.n += pi.empty(w) ? 0 : 1;
  pi.slot0 = (pi.S * pi.first_w / W) < a ? 1 : 0;   // tile is not its first segment
  return pi;
}

__device__ __forceinline__ float* piece_ptr(const mk_gemm_params& p, int worker, int slot) {
  return p.kpart + (size_t(worker) * 2 + slot) * p.piece_floats;
}

// ---------------------------------------------------------------------------
// Fetch warp: stream the unit's immutable operands into the ring.
// ---------------------------------------------------------------------------
struct Ring {
  uint32_t k = 0;   // slots issued / consumed so far this launch
};

// The sequence of ring slots one unit streams, in consumption order: for a
// GEMM every K-chunk of every tile this worker owns; for an attention unit
// the cached K and V block of every item.  Walked twice by the fetch warp:
// once to prefetch into L2, once to copy into the shared-memory ring.
template <int F>
struct SlotIter {
  const mk_task* t;
  int op, worker, ib, ie;
  // gemm
  typename std::conditional<(F & kFeatKsplit) != 0, SegIter, TileIter>::type it;
  const __nv_bfloat16* w;
  int chunks, R, tk, c, c_end, cur_n;
  // attention
  int item, kv;                 // kv: 0 = K next, 1 = V next
  const __nv_bfloat16* src_k;
  uint32_t bytes_kv;
  bool active;

  __device__ __forceinline__ void init(const KArgs& a, const mk_task& task, int ib_, int ie_, int worker_) {
    t = &task; op = task.op; worker = worker_; ib = ib_; ie = ie_; active = true;
    if (op == MK_OP_GEMM) {
      const mk_gemm_params& p = *P<mk_gemm_params>(a, task);
      it.init(p, a.W, task.level == MK_LEVEL_CHIPLET ? worker : 0);
      w = reinterpret_cast<const __nv_bfloat16*>(p.w);
      R = gemm_rows(p); tk = p.T_K; chunks = p.K / p.T_K; c = c_end = 0; cur_n = 0;
    } else if (op == MK_OP_ATTN_PARTIAL) {
      item = ib; kv = 0; bytes_kv = 0; src_k = nullptr;
    } else {
      active = false;
    }
  }
  // next slot: (src, bytes); false when the unit has no more slots
  __device__ __forceinline__ bool next(const KArgs& a, const void*& src, uint32_t& bytes) {
    if (!active) return false;
    if (op == MK_OP_GEMM) {
      if (c >= c_end) {
        if constexpr ((F & kFeatKsplit) != 0) {
          Seg g;
          if (!it.next(g)) { active = false; return false; }
          cur_n = g.n; c = g.c0; c_end = g.c1;
        } else {
          int m, n;
          if (!it.next(m, n)) { active = false; return false; }
          cur_n = n; c = 0; c_end = chunks;
        }
      }
      src = w + (size_t(cur_n) * chunks + c) * R * tk;
      bytes = uint32_t(R) * tk * 2;
      ++c;
      return true;
    }
    const mk_attn_params& p = *P<mk_attn_params>(a, *t);
    if (kv == 1) {   // V block of the current item
      src = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) +
            (reinterpret_cast<const __nv_bfloat16*>(src_k) - reinterpret_cast<const __nv_bfloat16*>(p.k_cache));
      bytes = bytes_kv; kv = 0; ++item;
      return true;
    }
    const bool full = attn_mma_path(p);   // tensor-core path: whole 64-token blocks
    for (; item < ie; ++item) {
      const int b = item / p.n_splits, sp = item % p.n_splits;
      const int pos = row_pos(p.positions, b);
      const int t0 = sp * p.split;
      if (t0 > pos) continue;
      const int nc = full ? p.split : min(p.split, pos - t0);
      if (nc <= 0) continue;
      src_k = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + kv_off(p, b, t0);
      bytes_kv = uint32_t(nc) * p.head_dim * 2;
      src = src_k; bytes = bytes_kv; kv = 1;
      return true;
    }
    active = false;
    return false;
  }
};

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}

// Consumer-side slot handshake.  After an abort the wait just stops (the
// data is garbage, the launch result is discarded) so that every consumer
// thread keeps the same control flow and no named barrier can hang.
__device__ __forceinline__ void cons_wait_slot(const KArgs& a, Smem& s, const Ring& r) {
  const int i = r.k % kSlots;
  mbar_wait(a, &s.full[i], (r.k / kSlots) & 1, -3);
}
__device__ __forceinline__ void cons_release_slot(Smem& s, Ring& r) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&s.empty[r.k % kSlots]);
  ++r.k;
}

// ---------------------------------------------------------------------------
// GEMM tile body: y[m0:m0+rows, cols] = x[m0:.., :] . W_tile^T  (CUDA cores,
// 128-bit weight streaming; weights come from the smem ring).
// Slot layout: [R rows][T_K] bf16, thread ct owns 16-byte segments
// ct, ct+256, ... -- all in one column (x reuse across rows).  Activations
// come from the per-task staged copy in shared memory (XS) or, when the
// rows do not fit, from global memory one slot ahead of use.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dot8_acc(const float (&w)[8], const float (&x)[8], float& acc) {
#pragma unroll
  for (int e = 0; e < 8; ++e) acc = fmaf(w[e], x[e], acc);
}

// Stage rows [m0, m0+rows) of x (K wide) into s.u.xs, optionally applying
// Qwen3RMSNorm (fp32 statistics, cast, gamma) -- the rms task fused into its
// consumer GEMM.  Bit-identical to run_rmsnorm's output.
__device__ void stage_x(const KArgs& a, Smem& s, const mk_gemm_params& p, int m0, int rows, int ct,
                        bool trace) {
  const uint16_t* x = reinterpret_cast<const uint16_t*>(p.x);
  const int K = p.K;
  const bool norm = p.norm_gamma != nullptr;
  const uint16_t* gam = reinterpret_cast<const uint16_t*>(p.norm_gamma);
  constexpr int kSeg = 6;                  // K <= 6 * 2048 per thread pass
  float ss[kMaxNB];
#pragma unroll
  for (int b = 0; b < kMaxNB; ++b) ss[b] = 0.f;
  uint4 gv[kSeg];
  if (s.xs_hoist) {
    // consumer 0 bulk-copied the rows (and gamma, behind them) right after
    // the dependency poll: only the wait and the sums of squares remain
    mbar_wait(a, &s.xs_bar, s.xs_parity, -17);
    const uint16_t* gs = s.u.xs + rows * K;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) {
      const int k = ct * 8 + q * kCons * 8;
      gv[q] = (norm && k < K) ? *reinterpret_cast<const uint4*>(gs + k) : make_uint4(0, 0, 0, 0);
    }
    if (norm) {
      // RMSNorm as a post-scale: stage gamma * x (one pass, no statistics
      // barrier before it) and the per-warp sums of squares; the GEMV
      // epilogue multiplies each row's dot products by its 1/rms
      // (post_rs) -- y = rs * W (gamma . x), the model's math without the
      // intermediate bf16 rounding of x * rs.
      const int warp = ct >> 5, lane = ct & 31;
#pragma unroll
      for (int b = 0; b < kMaxNB; ++b) {
        if (b < rows) {
#pragma unroll
          for (int q = 0; q < kSeg; ++q) {
            const int k = ct * 8 + q * kCons * 8;
            if (k >= K) continue;
            float f[8], g[8];
            unpack8(*reinterpret_cast<const uint4*>(&s.u.xs[b * K + k]), f);
            unpack8(gv[q], g);
            uint16_t o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) { ss[b] = fmaf(f[e], f[e], ss[b]); o[e] = f2bf(g[e] * f[e]); }
            *reinterpret_cast<uint4*>(&s.u.xs[b * K + k]) = *reinterpret_cast<uint4*>(o);
          }
          float v = ss[b];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
          if (lane == 0) s.rsum[warp][b] = v;
        }
      }
      if (trace && ct == 0 && s.tr[7] == 0) s.tr[7] = globaltimer();
      bar_sync(1, kCons);
      return;
    }
  } else {
    // gamma is static: issue its loads together with x's (one round trip)
#pragma unroll
    for (int q = 0; q < kSeg; ++q) {
      const int k = ct * 8 + q * kCons * 8;
      gv[q] = (norm && k < K) ? *reinterpret_cast<const uint4*>(gam + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int b = 0; b < kMaxNB; ++b) {
      if (b < rows) {
#pragma unroll 4
        for (int k = ct * 8; k < K; k += kCons * 8) {
          const uint4 v = ldg128_cg(x + size_t(m0 + b) * p.ldx + k);
          *reinterpret_cast<uint4*>(&s.u.xs[b * K + k]) = v;
          if (norm) {
            float f[8];
            unpack8(v, f);
#pragma unroll
            for (int e = 0; e < 8; ++e) ss[b] = fmaf(f[e], f[e], ss[b]);
          }
        }
      }
    }
  }
  if (trace && ct == 0 && s.tr[7] == 0) s.tr[7] = globaltimer();
  if (norm) {
    const int warp = ct >> 5, lane = ct & 31;
#pragma unroll
    for (int b = 0; b < kMaxNB; ++b) {
      if (b < rows) {
        float v = ss[b];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) s.rsum[warp][b] = v;
      }
    }
    bar_sync(1, kCons);
    if (ct < rows) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < kConsWarps; ++w) t += s.rsum[w][ct];
      s.rs[ct] = rsqrtf(t / float(K) + p.norm_eps);
    }
    bar_sync(1, kCons);
    for (int b = 0; b < rows; ++b) {
      const float rs = s.rs[b];
#pragma unroll
      for (int q = 0; q < kSeg; ++q) {
        const int k = ct * 8 + q * kCons * 8;
        if (k >= K) continue;
        float f[8], g[8];
        unpack8(*reinterpret_cast<const uint4*>(&s.u.xs[b * K + k]), f);
        unpack8(gv[q], g);
        uint16_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = f2bf(g[e] * bf2f(f2bf(f[e] * rs)));
        *reinterpret_cast<uint4*>(&s.u.xs[b * K + k]) = *reinterpret_cast<uint4*>(o);
      }
    }
  }
  bar_sync(1, kCons);
}

// 1/rms of staged row b when stage_x normalised by post-scale (hoisted
// staging with a norm), else 1 (rows pre-normalised or no norm).  The
// per-warp sums of squares were written before stage_x's final barrier.
__device__ __forceinline__ float post_rs(const Smem& s, const mk_gemm_params& p, int b) {
  if (!p.norm_gamma || !s.xs_hoist) return 1.f;
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < kConsWarps; ++w) t += s.rsum[w][b];
  return rsqrtf(t / float(p.K) + p.norm_eps);
}

// K-split piece handling for the CUDA-core body.  Called by all consumer
// threads after the warp reduction (every lane holds tot[j][b] of rows
// warp + 8j).  Returns true when this CTA runs the epilogue: the tile was
// whole, or this was its last piece -- then tot holds the piece sum (lane b,
// batch row b), summed in piece order so the result does not depend on
// arrival order.
template <int NB, int RPW>
__device__ __forceinline__ bool gemv_piece(const KArgs& a, Smem& s, const mk_gemm_params& p, const Seg& g,
                           int worker, int rows_m, int rpw, int ct, float (&tot)[RPW][NB]) {
  if (g.c0 == 0 && g.c1 == p.K / p.T_K) return true;
  const int warp = ct >> 5, lane = ct & 31;
  float* mine = piece_ptr(p, worker, g.first ? 0 : 1);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane != b || b >= rows_m) continue;
#pragma unroll
    for (int j = 0; j < RPW; ++j)
      if (j < rpw) __stcg(mine + (warp + kConsWarps * j) * p.T_M + b, tot[j][b]);
  }
  const PieceInfo pi = tile_pieces(p, a.W, g.tile);
  __threadfence();
  bar_sync(1, kCons);
  if (ct == 0) {
    const uint32_t old = atom_acq_rel_add(&a.sub_ctr[p.tile_ctr0 + g.tile], 1u);
    s.piece_last = (old + 1 == uint32_t(pi.n) * a.epoch) ? 1 : 0;
  }
  bar_sync(1, kCons);
  if (!s.piece_last) return false;
  __threadfence();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane != b || b >= rows_m) continue;
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      if (j >= rpw) continue;
      float v = 0.f;
      for (int w = pi.first_w; w <= pi.last_w; ++w) {
        if (pi.empty(w)) continue;
        v += __ldcg(piece_ptr(p, w, w == pi.first_w ? pi.slot0 : 0) +
                    (warp + kConsWarps * j) * p.T_M + b);
      }
      tot[j][b] = v;
    }
  }
  return true;
}

// Warp-owned rows: slot [R rows][KC] bf16, warp w owns rows w, w+8, w+16,
// w+24 (< R); lane l covers columns l*8 + 256*p of each row.  Partial dot
// products stay in registers across the tile's K-chunks and are reduced
// with warp shuffles only -- no CTA barrier per tile; each warp releases
// ring slots on its own.  Fused gate/up: R = 2*T_N = 16, so warp w owns
// gate row w and up row w+8 and applies SiLU itself.
template <int NB, bool XS>
__device__ void gemm_tile(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                          const mk_gemm_params& p, int m, int n, int ct,
                          float (&amv)[NB], int (&ami)[NB]) {
  const int warp = ct >> 5, lane = ct & 31;
  const int R = gemm_rows(p);
  const int rpw = R / kConsWarps;          // rows per warp (1, 2 or 4)
  const int KC = p.T_K;
  const int npass = KC >= 256 ? KC / 256 : 1;
  const bool lane_on = lane * 8 < KC;      // KC < 256: upper lanes idle
  const int chunks = p.K / KC;
  const int m0 = m * p.T_M;
  const int rows_m = min(p.T_M, p.M - m0);
  const int out_col0 = p.y_col0 + n * p.T_N;
  const bool silu = p.epilogue == MK_EPI_SILU;
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(p.x);

  // epilogue operands fetched before the stream: lane b holds row b
  float resv[4] = {0.f, 0.f, 0.f, 0.f};
  if (p.epilogue == MK_EPI_RESIDUAL && lane < rows_m) {
    const uint16_t* res = reinterpret_cast<const uint16_t*>(p.res) + size_t(m0 + lane) * p.ldres;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < rpw) resv[j] = bf2f(ldg16_cg(res + out_col0 + warp + kConsWarps * j));
  }

  float acc[4][NB];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[j][b] = 0.f;

  for (int c = 0; c < chunks; ++c) {
    cons_wait_slot(a, s, r);
    if (!(a.debug & 1)) {
      const uint8_t* slot = ring + size_t(r.k % kSlots) * kSlotBytes;
      for (int ps = 0; ps < npass; ++ps) {
        const int kin = ps * 256 + lane * 8;            // column inside the chunk
        const int kg = c * KC + kin;                    // column in K
        float wf[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < rpw && lane_on)
            unpack8(lds128(slot + (size_t(warp + kConsWarps * j) * KC + kin) * 2), wf[j]);
          else {
#pragma unroll
            for (int e = 0; e < 8; ++e) wf[j][e] = 0.f;
          }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b < rows_m && lane_on) {
            uint4 xv;
            if constexpr (XS) xv = *reinterpret_cast<const uint4*>(&s.u.xs[b * p.K + kg]);
            else xv = ldg128_cg(x + size_t(m0 + b) * p.ldx + kg);
            float xf[8];
            unpack8(xv, xf);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < rpw) dot8_acc(wf[j], xf, acc[j][b]);
          }
        }
      }
    }
    cons_release_slot(s, r);
  }

  // warp reduction: after the xor butterfly every lane holds every sum
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= rpw) continue;            // warp-uniform
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float v = acc[j][b];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      acc[j][b] = v;
    }
  }
  // lane b writes batch row b (register-array reads use constant indices)
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane != b || b >= rows_m) continue;
    if (p.norm_gamma) {                 // post-scale RMSNorm (stage_x)
      const float r = post_rs(s, p, b);
#pragma unroll
      for (int j = 0; j < 4; ++j) if (j < rpw) acc[j][b] *= r;
    }
    if (p.epilogue == MK_EPI_LOGITS) {
      float* y = reinterpret_cast<float*>(p.y);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= rpw) continue;
        const int col = out_col0 + warp + kConsWarps * j;
        const float v = acc[j][b];
        if (y) y[size_t(m0 + b) * p.ldy + col] = v;
        if (v > amv[b] || (v == amv[b] && col < ami[b])) { amv[b] = v; ami[b] = col; }
      }
    } else {
      if (p.epilogue == MK_EPI_PARTIAL) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < rpw) tp_store(a, p, m0 + b, out_col0 + warp + kConsWarps * j, acc[j][b]);
        continue;
      }
      uint16_t* y = reinterpret_cast<uint16_t*>(p.y) + size_t(m0 + b) * p.ldy;
      if (silu) {              // gate rows j < rpw/2, up rows j + rpw/2
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j >= rpw / 2) continue;
          const float g = acc[j][b];
          const float u = rpw == 2 ? acc[1][b] : (j == 0 ? acc[2][b] : acc[3][b]);
          st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(g / (1.f + __expf(-g)) * u));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= rpw) continue;
          st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(acc[j][b] + resv[j]));
        }
      }
    }
  }
}

// Fast path: rows per warp RPW in {1,2,4}, K-chunk KC = 1024/RPW (so one
// slot = 8*RPW rows x KC = 16 KiB and every lane covers NP = 4/RPW 16-byte
// segments per row).  All slot loads are issued before any math, the slot is
// released as soon as the weights sit in registers, and independent
// accumulator chains keep the FMA pipe busy.
template <int NB, int RPW, bool XS>
__device__ void gemm_tile_fast(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                               const mk_gemm_params& p, int m, int n, int ct,
                               float (&amv)[NB], int (&ami)[NB]) {
  constexpr int NP = 4 / RPW;
  constexpr int KC = 256 * NP;
  constexpr int CH = (RPW * NB > 4) ? 1 : NP;    // extra chains when few (row, b) pairs
  const int warp = ct >> 5, lane = ct & 31;
  const int chunks = p.K / KC;
  const int m0 = m * p.T_M;
  const int rows_m = min(p.T_M, p.M - m0);
  const int out_col0 = p.y_col0 + n * p.T_N;
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(p.x);

  float resv[RPW];
#pragma unroll
  for (int j = 0; j < RPW; ++j) resv[j] = 0.f;
  if (p.epilogue == MK_EPI_RESIDUAL && lane < rows_m) {
    const uint16_t* res = reinterpret_cast<const uint16_t*>(p.res) + size_t(m0 + lane) * p.ldres;
#pragma unroll
    for (int j = 0; j < RPW; ++j) resv[j] = bf2f(ldg16_cg(res + out_col0 + warp + kConsWarps * j));
  }

  float acc[CH][RPW][NB];
#pragma unroll
  for (int q = 0; q < CH; ++q)
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[q][j][b] = 0.f;

  const uint32_t ring_s = smem_u32(ring);
  const uint32_t xs_s = smem_u32(s.u.xs);
  for (int c = 0; c < chunks; ++c) {
    cons_wait_slot(a, s, r);
    const uint32_t slot = ring_s + uint32_t(r.k % kSlots) * kSlotBytes;
    uint4 wv[NP][RPW];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
#pragma unroll
      for (int j = 0; j < RPW; ++j)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(wv[ps][j].x), "=r"(wv[ps][j].y), "=r"(wv[ps][j].z), "=r"(wv[ps][j].w)
                     : "r"(slot + uint32_t(((warp + kConsWarps * j) * KC + ps * 256 + lane * 8) * 2)));
    uint4 xv[NP][NB];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int kg = c * KC + ps * 256 + lane * 8;
        if constexpr (XS) {
          if (b < rows_m)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(xv[ps][b].x), "=r"(xv[ps][b].y), "=r"(xv[ps][b].z), "=r"(xv[ps][b].w)
                         : "r"(xs_s + uint32_t((b * p.K + kg) * 2)));
          else xv[ps][b] = make_uint4(0, 0, 0, 0);
        } else {
          xv[ps][b] = (b < rows_m) ? ldg128_cg(x + size_t(m0 + b) * p.ldx + kg) : make_uint4(0, 0, 0, 0);
        }
      }
    cons_release_slot(s, r);          // weights now live in registers
    if (a.debug & 1) continue;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      float wf[RPW][8];
#pragma unroll
      for (int j = 0; j < RPW; ++j) unpack8(wv[ps][j], wf[j]);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float xf[8];
        unpack8(xv[ps][b], xf);
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          float& t = acc[CH == 1 ? 0 : ps][j][b];
#pragma unroll
          for (int e = 0; e < 8; ++e) t = fmaf(wf[j][e], xf[e], t);
        }
      }
    }
  }

  float tot[RPW][NB];
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float v = acc[0][j][b];
#pragma unroll
      for (int q = 1; q < CH; ++q) v += acc[q][j][b];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[j][b] = v;
    }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane != b || b >= rows_m) continue;
    if (p.norm_gamma) {                 // post-scale RMSNorm (stage_x)
      const float r = post_rs(s, p, b);
#pragma unroll
      for (int j = 0; j < RPW; ++j) tot[j][b] *= r;
    }
    if (p.epilogue == MK_EPI_LOGITS) {
      float* y = reinterpret_cast<float*>(p.y);
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const int col = out_col0 + warp + kConsWarps * j;
        const float v = tot[j][b];
        if (y) y[size_t(m0 + b) * p.ldy + col] = v;
        if (v > amv[b] || (v == amv[b] && col < ami[b])) { amv[b] = v; ami[b] = col; }
      }
    } else if (p.epilogue == MK_EPI_PARTIAL) {
#pragma unroll
      for (int j = 0; j < RPW; ++j) tp_store(a, p, m0 + b, out_col0 + warp + kConsWarps * j, tot[j][b]);
    } else {
      uint16_t* y = reinterpret_cast<uint16_t*>(p.y) + size_t(m0 + b) * p.ldy;
      if (p.epilogue == MK_EPI_SILU) {
        if constexpr (RPW >= 2) {
#pragma unroll
          for (int j = 0; j < RPW / 2; ++j) {
            const float g = tot[j][b], u = tot[j + RPW / 2][b];
            st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(g / (1.f + __expf(-g)) * u));
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < RPW; ++j) st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(tot[j][b] + resv[j]));
      }
    }
  }
}

// K-split variant of the fast path: K-chunks [c0, c1) of the tile, partial
// pieces summed by the last piece (gemv_piece).  Rows per warp RPW in {1,2,4}, K-chunk KC = 1024/RPW (so one
// slot = 8*RPW rows x KC = 16 KiB and every lane covers NP = 4/RPW 16-byte
// segments per row).  All slot loads are issued before any math, the slot is
// released as soon as the weights sit in registers, and independent
// accumulator chains keep the FMA pipe busy.
template <int NB, int RPW, bool XS>
__device__ __forceinline__ void gemm_tile_fast_ks(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                                  const mk_gemm_params& p, const Seg& sg, int worker, int ct,
                                  float (&amv)[NB], int (&ami)[NB]) {
  const int m = sg.m, n = sg.n, c_begin = sg.c0, c_end = sg.c1;
  Ring rl = r;                             // keep the ring cursor in a register
  constexpr int NP = 4 / RPW;
  constexpr int KC = 256 * NP;
  constexpr int CH = (RPW * NB > 4) ? 1 : NP;    // extra chains when few (row, b) pairs
  const int warp = ct >> 5, lane = ct & 31;
  const int chunks = p.K / KC;
  const int m0 = m * p.T_M;
  const int rows_m = min(p.T_M, p.M - m0);
  const int out_col0 = p.y_col0 + n * p.T_N;
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(p.x);

  float resv[RPW];
#pragma unroll
  for (int j = 0; j < RPW; ++j) resv[j] = 0.f;
  if (p.epilogue == MK_EPI_RESIDUAL && lane < rows_m) {
    const uint16_t* res = reinterpret_cast<const uint16_t*>(p.res) + size_t(m0 + lane) * p.ldres;
#pragma unroll
    for (int j = 0; j < RPW; ++j) resv[j] = bf2f(ldg16_cg(res + out_col0 + warp + kConsWarps * j));
  }

  float acc[CH][RPW][NB];
#pragma unroll
  for (int q = 0; q < CH; ++q)
#pragma unroll
    for (int j = 0; j < RPW; ++j)
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[q][j][b] = 0.f;

  const uint32_t ring_s = smem_u32(ring);
  const uint32_t xs_s = smem_u32(s.u.xs);
  (void)chunks;
  for (int c = c_begin; c < c_end; ++c) {
    cons_wait_slot(a, s, rl);
    const uint32_t slot = ring_s + uint32_t(rl.k % kSlots) * kSlotBytes;
    uint4 wv[NP][RPW];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
#pragma unroll
      for (int j = 0; j < RPW; ++j)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(wv[ps][j].x), "=r"(wv[ps][j].y), "=r"(wv[ps][j].z), "=r"(wv[ps][j].w)
                     : "r"(slot + uint32_t(((warp + kConsWarps * j) * KC + ps * 256 + lane * 8) * 2)));
    uint4 xv[NP][NB];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int kg = c * KC + ps * 256 + lane * 8;
        if constexpr (XS) {
          if (b < rows_m)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(xv[ps][b].x), "=r"(xv[ps][b].y), "=r"(xv[ps][b].z), "=r"(xv[ps][b].w)
                         : "r"(xs_s + uint32_t((b * p.K + kg) * 2)));
          else xv[ps][b] = make_uint4(0, 0, 0, 0);
        } else {
          xv[ps][b] = (b < rows_m) ? ldg128_cg(x + size_t(m0 + b) * p.ldx + kg) : make_uint4(0, 0, 0, 0);
        }
      }
    cons_release_slot(s, rl);         // weights now live in registers
    if (a.debug & 1) continue;
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {
      float wf[RPW][8];
#pragma unroll
      for (int j = 0; j < RPW; ++j) unpack8(wv[ps][j], wf[j]);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float xf[8];
        unpack8(xv[ps][b], xf);
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          float& t = acc[CH == 1 ? 0 : ps][j][b];
#pragma unroll
          for (int e = 0; e < 8; ++e) t = fmaf(wf[j][e], xf[e], t);
        }
      }
    }
  }

  r = rl;
  float tot[RPW][NB];
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float v = acc[0][j][b];
#pragma unroll
      for (int q = 1; q < CH; ++q) v += acc[q][j][b];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      tot[j][b] = v;
    }
  if (!gemv_piece<NB, RPW>(a, s, p, sg, worker, rows_m, RPW, ct, tot)) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (lane != b || b >= rows_m) continue;
    if (p.norm_gamma) {                 // post-scale RMSNorm (stage_x)
      const float r = post_rs(s, p, b);
#pragma unroll
      for (int j = 0; j < RPW; ++j) tot[j][b] *= r;
    }
    if (p.epilogue == MK_EPI_LOGITS) {
      float* y = reinterpret_cast<float*>(p.y);
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const int col = out_col0 + warp + kConsWarps * j;
        const float v = tot[j][b];
        if (y) y[size_t(m0 + b) * p.ldy + col] = v;
        if (v > amv[b] || (v == amv[b] && col < ami[b])) { amv[b] = v; ami[b] = col; }
      }
    } else if (p.epilogue == MK_EPI_PARTIAL) {
#pragma unroll
      for (int j = 0; j < RPW; ++j) tp_store(a, p, m0 + b, out_col0 + warp + kConsWarps * j, tot[j][b]);
    } else {
      uint16_t* y = reinterpret_cast<uint16_t*>(p.y) + size_t(m0 + b) * p.ldy;
      if (p.epilogue == MK_EPI_SILU) {
        if constexpr (RPW >= 2) {
#pragma unroll
          for (int j = 0; j < RPW / 2; ++j) {
            const float g = tot[j][b], u = tot[j + RPW / 2][b];
            st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(g / (1.f + __expf(-g)) * u));
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < RPW; ++j) st_out(&y[out_col0 + warp + kConsWarps * j], f2bf(tot[j][b] + resv[j]));
      }
    }
  }
}

template <int NB, bool XS>
__device__ void gemm_task(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                          const mk_gemm_params& p, int w_in_task, int gw, int tix, int ct,
                          unsigned long long& tiles) {
  const int warp = ct >> 5, lane = ct & 31;
  float amv[NB];
  int ami[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) { amv[b] = -INFINITY; ami[b] = 0x7fffffff; }
  TileIter it;
  it.init(p, a.W, w_in_task);
  int m, n, staged_m = -1;
  int cur_m = -1;
  while (it.next(m, n)) {
    if (p.epilogue == MK_EPI_LOGITS && m != cur_m) {
      // switch the lanes' running argmax to the rows of the new m-tile
      // (lane b always owns row m0 + b, so no cross-lane hazard)
      const int mo = cur_m * p.T_M, mn = m * p.T_M;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (lane != b) continue;
        if (cur_m >= 0 && mo + b < p.M) { s.amx_val[warp][mo + b] = amv[b]; s.amx_idx[warp][mo + b] = ami[b]; }
        if (mn + b < p.M) { amv[b] = s.amx_val[warp][mn + b]; ami[b] = s.amx_idx[warp][mn + b]; }
      }
    }
    cur_m = m;
    if constexpr (XS) {
      if (m != staged_m) {
        stage_x(a, s, p, m * p.T_M, min(p.T_M, p.M - m * p.T_M), ct, a.trace != nullptr);
        staged_m = m;
      }
    }
    if (ct == 0 && a.trace && s.tr[3] == 0) s.tr[3] = globaltimer();
    // fast path for the register-feasible (rows-per-warp, batch) pairs
    const int R = gemm_rows(p);
    bool done = false;
    if constexpr (NB == 1) {
      if (R == 8 && p.T_K == 1024) { gemm_tile_fast<NB, 1, XS>(a, s, ring, r, p, m, n, ct, amv, ami); done = true; }
    }
    if constexpr (NB <= 4) {
      if (!done && R == 16 && p.T_K == 512) { gemm_tile_fast<NB, 2, XS>(a, s, ring, r, p, m, n, ct, amv, ami); done = true; }
    }
    if constexpr (NB <= 8) {
      if (!done && R == 32 && p.T_K == 256) { gemm_tile_fast<NB, 4, XS>(a, s, ring, r, p, m, n, ct, amv, ami); done = true; }
    }
    if (!done) gemm_tile<NB, XS>(a, s, ring, r, p, m, n, ct, amv, ami);
    if (ct == 0) {
      ++tiles;
      if (a.tile_log) {
        unsigned long long at = atomicAdd(a.tile_cursor, 1ull);
        if ((long long)at < a.tile_cap) {
          int32_t* rec = a.tile_log + at * 4;
          rec[0] = tix; rec[1] = gw; rec[2] = m; rec[3] = n;
        }
      }
    }
  }
  if (p.epilogue == MK_EPI_LOGITS) {
    if (cur_m >= 0) {
      const int m0 = cur_m * p.T_M;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (lane == b && m0 + b < p.M) { s.amx_val[warp][m0 + b] = amv[b]; s.amx_idx[warp][m0 + b] = ami[b]; }
    }
    bar_sync(1, kCons);
    const int slot = p.amax_base + w_in_task;
    // a CU tile task owns only its m-tile's rows of the shared slot
    const int b_lo = p.tile_m >= 0 ? p.tile_m * p.T_M : 0;
    const int b_hi = p.tile_m >= 0 ? min(p.M, b_lo + p.T_M) : p.M;
    for (int b = b_lo + ct; b < b_hi && b < kAmaxRows; b += kCons) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
      for (int w = 0; w < kConsWarps; ++w) {
        const float v = s.amx_val[w][b];
        const int i = s.amx_idx[w][b];
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      p.amax_val[size_t(slot) * p.amax_stride + b] = best;
      p.amax_idx[size_t(slot) * p.amax_stride + b] = bi;
    }
  }
  bar_sync(1, kCons);   // staged rows / amx[] reusable by the next unit
}

// K-split die task (lowering only K-splits the fast-path shapes).
template <int NB, bool XS>
__device__ void gemm_task_ks(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                          const mk_gemm_params& p, int w_in_task, int gw, int tix, int ct,
                          unsigned long long& tiles) {
  const int warp = ct >> 5, lane = ct & 31;
  float amv[NB];
  int ami[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) { amv[b] = -INFINITY; ami[b] = 0x7fffffff; }
  int staged_m = -1;
  int cur_m = -1;
  RangeIter rit;
  rit.init(p, a.W, w_in_task);
  int m, n;
  Seg sg;
  for (;;) {
    if (!rit.next(sg)) break;
    m = sg.m; n = sg.n;
    if (p.epilogue == MK_EPI_LOGITS && m != cur_m) {
      // switch the lanes' running argmax to the rows of the new m-tile
      // (lane b always owns row m0 + b, so no cross-lane hazard)
      const int mo = cur_m * p.T_M, mn = m * p.T_M;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (lane != b) continue;
        if (cur_m >= 0 && mo + b < p.M) { s.amx_val[warp][mo + b] = amv[b]; s.amx_idx[warp][mo + b] = ami[b]; }
        if (mn + b < p.M) { amv[b] = s.amx_val[warp][mn + b]; ami[b] = s.amx_idx[warp][mn + b]; }
      }
    }
    cur_m = m;
    if constexpr (XS) {
      if (m != staged_m) {
        stage_x(a, s, p, m * p.T_M, min(p.T_M, p.M - m * p.T_M), ct, a.trace != nullptr);
        staged_m = m;
      }
    }
    if (ct == 0 && a.trace && s.tr[3] == 0) s.tr[3] = globaltimer();
    // fast path for the register-feasible (rows-per-warp, batch) pairs
    const int R = gemm_rows(p);
    bool done = false;
    if constexpr (NB == 1) {
      if (R == 8 && p.T_K == 1024) { gemm_tile_fast_ks<NB, 1, XS>(a, s, ring, r, p, sg, w_in_task, ct, amv, ami); done = true; }
    }
    if constexpr (NB <= 4) {
      if (!done && R == 16 && p.T_K == 512) { gemm_tile_fast_ks<NB, 2, XS>(a, s, ring, r, p, sg, w_in_task, ct, amv, ami); done = true; }
    }
    if constexpr (NB <= 8) {
      if (!done && R == 32 && p.T_K == 256) { gemm_tile_fast_ks<NB, 4, XS>(a, s, ring, r, p, sg, w_in_task, ct, amv, ami); done = true; }
    }
    if (ct == 0) {
      ++tiles;
      if (a.tile_log) {
        unsigned long long at = atomicAdd(a.tile_cursor, 1ull);
        if ((long long)at < a.tile_cap) {
          int32_t* rec = a.tile_log + at * 4;
          rec[0] = tix; rec[1] = gw; rec[2] = m; rec[3] = n;
        }
      }
    }
  }
  if (p.epilogue == MK_EPI_LOGITS) {
    if (cur_m >= 0) {
      const int m0 = cur_m * p.T_M;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (lane == b && m0 + b < p.M) { s.amx_val[warp][m0 + b] = amv[b]; s.amx_idx[warp][m0 + b] = ami[b]; }
    }
    bar_sync(1, kCons);
    const int slot = p.amax_base + w_in_task;
    // a CU tile task owns only its m-tile's rows of the shared slot
    const int b_lo = p.tile_m >= 0 ? p.tile_m * p.T_M : 0;
    const int b_hi = p.tile_m >= 0 ? min(p.M, b_lo + p.T_M) : p.M;
    for (int b = b_lo + ct; b < b_hi && b < kAmaxRows; b += kCons) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
      for (int w = 0; w < kConsWarps; ++w) {
        const float v = s.amx_val[w][b];
        const int i = s.amx_idx[w][b];
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      p.amax_val[size_t(slot) * p.amax_stride + b] = best;
      p.amax_idx[size_t(slot) * p.amax_stride + b] = bi;
    }
  }
  bar_sync(1, kCons);   // staged rows / amx[] reusable by the next unit
}

// ---------------------------------------------------------------------------
// tcgen05 skinny GEMM (batch >= 16): D[128 weight rows x NT batch rows] in
// TMEM += W_tile[128 x 64] (ring slot, pre-swizzled in HBM) . X[NT x 64]^T
// (x ring, staged + swizzled by consumer warps 0-3).  One lane of producer
// warp 2 issues the MMAs (mma_warp), consumer warps 4-7 drain the
// double-buffered accumulator (tcgen05.ld) into the epilogue.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int umma_nt(const mk_gemm_params& p) {
  const int rows = min(p.T_M, p.M);
  return (rows + 15) / 16 * 16;
}

// The tcgen05 path runs on two producer warps with warp-uniform control flow
// (a single diverged lane would leave the other 31 parked at a convergence
// barrier); lane 0 of each issues.  The per-chunk paths are kept short --
// they pace the whole die task: ring / x-stage indices and phases advance
// incrementally (stage index + phase bit), smem descriptors are offsets
// of per-ring base descriptors.
//
// x-load warp (warp 3): for each job, TMA-loads the activation chunk of every
// K-chunk the MMAs will consume into the x ring (x_stages deep), gated only
// by the stage being released by the MMA that read it.
__device__ void xload_warp(const KArgs& a, Smem& s) {
  const bool leader = (threadIdx.x & 31) == 0;
  const int XS = a.x_stages;                 // x ring stages
  const uint32_t XB = uint32_t(a.x_stage_bytes);
  uint32_t jq = 0;
  int xl = 0;                                // x stage index / phase (any stage count)
  uint32_t xph = 0;
  const bool no_tma = (a.debug & 16) != 0;
  for (;;) {
    if (!mbar_wait(a, &s.job_full, jq & 1, -15)) break;
    ++jq;
    const int4 job = s.job;
    if (job.x < 0) break;
    const mk_gemm_params& p = *P<mk_gemm_params>(a, s.tcache[job.w]);
    const void* tmap = a.tmaps + job.x;
    const uint32_t x_bytes = uint32_t(umma_nt(p)) * 128u;
    // the job arrives before its dependency resolved: acquire the unit's
    // input events here (relaxed polls + one acquire fence), then order the
    // producers' generic writes before the async-proxy (TMA) reads of x
    {
      const mk_task& t = s.tcache[job.w];
      bool ok = true;
      if (leader) {
        for (int k = 0; k < 2 && ok; ++k) {
          const int e = k ? t.wait1 : t.wait0;
          if (e < 0) continue;
          Spin sp;
          while (!ev_done<false>(a, e, t.pad[k], t.pad[2 + k]))
            if (!sp.ok(a, -15)) { ok = false; break; }
        }
        fence_acq_rel_gpu();
        fence_proxy_async_global();
      }
      if (!__shfl_sync(0xffffffffu, ok ? 1 : 0, 0)) return;
    }
    SegIter lt;
    lt.init(p, a.W, job.y);
    Seg g;
    while (lt.next(g)) {
      const int row = g.m * p.T_M;
      // one stage = the activation chunks of one MMA chunk pair (the MMA
      // warp pairs c0, c0+1, ... of each segment; a last odd chunk alone)
      for (int c = g.c0; c < g.c1; c += 2) {
        const int n = min(2, g.c1 - c);
        if (!mbar_spin(a, &s.xempty[xl], xph ^ 1, -13)) return;
        if (leader) {
          if (no_tma) {                // diagnostics: no activation TMA
            mbar_arrive(&s.xfull[xl]);
          } else {
            uint8_t* dst = reinterpret_cast<uint8_t*>(s.u.xs) + size_t(xl) * 2 * XB;
            mbar_arrive_expect_tx(&s.xfull[xl], uint32_t(n) * x_bytes);
            tma_load_2d(dst, tmap, c * 64, row, &s.xfull[xl]);
            if (n == 2) tma_load_2d(dst + XB, tmap, (c + 1) * 64, row, &s.xfull[xl]);
          }
        }
        __syncwarp();
        if (++xl == XS) { xl = 0; xph ^= 1; }
      }
    }
  }
}

// MMA warp (warp 2): per K-chunk wait for the weight slot and the activation
// stage, issue the four UMMA_K=16 MMAs into the segment's TMEM accumulator,
// release both through tcgen05.commit; one commit per segment to tile_done.
__device__ void mma_warp(const KArgs& a, Smem& s, uint8_t* ring) {
  const bool leader = (threadIdx.x & 31) == 0;
  const int XS = a.x_stages;                 // x ring stages
  const uint32_t XB = uint32_t(a.x_stage_bytes);
  int ri = 0; uint32_t rph = 0;              // ring slot index / phase
  int xi = 0; uint32_t xph = 0;              // x stage index / phase
  uint32_t tb_k = 0, jq = 0;
  unsigned long long w_full = 0, w_x = 0, w_tmem = 0, n_chunks = 0;
  // diagnostics flags read once: the per-chunk path paces the die task
  const bool prof = (a.debug & 4) != 0, no_mma = (a.debug & 8) != 0;
  // trace diagnostics (debug bit 5): stamps 6/7 = first operands ready / last commit
  const bool stamp = a.trace != nullptr && (a.debug & 32) != 0;
  const int dbg_mode = (a.debug & 64) ? 1 : (a.debug & 128) ? 2 : 0;   // umma_chunk8_dbg
  const uint64_t adesc0 = umma_desc_sw128(smem_u32(ring));
  const uint64_t bdesc0 = umma_desc_sw128(smem_u32(s.u.xs));
  for (;;) {
    if (!mbar_wait(a, &s.job_full, jq & 1, -9)) break;
    ++jq;
    const int4 job = s.job;
    if (job.x < 0) break;
    const mk_gemm_params& p = *P<mk_gemm_params>(a, s.tcache[job.w]);
    // Everything the UMMA issue path reads is made provably warp-uniform
    // (values broadcast from lane 0 by shfl): the descriptors then live in
    // uniform registers, instead of a per-instruction ELECT / R2UR
    // waterfall around every UTCHMMA (measured ~120 cycles per MMA).
    const uint32_t idesc = __shfl_sync(0xffffffffu, umma_idesc_bf16(128, umma_nt(p)), 0);
    const uint32_t tmem0 = __shfl_sync(0xffffffffu, s.tmem_base, 0);
    // the job starts at the consumers' ring cursor (job.z)
    ri = __shfl_sync(0xffffffffu, int(uint32_t(job.z) % kSlots), 0);
    rph = __shfl_sync(0xffffffffu, (uint32_t(job.z) / kSlots) & 1, 0);
    SegIter it;
    it.init(p, a.W, job.y);
    Seg sg;
    bool first_pair = true;
    for (;;) {
      if (!__shfl_sync(0xffffffffu, it.next(sg) ? 1 : 0, 0)) break;
      sg.c0 = __shfl_sync(0xffffffffu, sg.c0, 0);
      sg.c1 = __shfl_sync(0xffffffffu, sg.c1, 0);
      const int buf = tb_k & 1;
      bool ok = prof ? mbar_wait_p(a, &s.tmem_free[buf], ((tb_k >> 1) & 1) ^ 1, -10, w_tmem)
                     : mbar_spin(a, &s.tmem_free[buf], ((tb_k >> 1) & 1) ^ 1, -10);
      if (!__all_sync(0xffffffffu, ok)) return;
      tc_fence_after();
      const uint32_t d = tmem0 + uint32_t(buf * kBufCols);
      int c = sg.c0;
      // chunk pairs: one loop pass (waits, fences, issue setup) per 32 KiB;
      // the pair's activation chunks share one x stage (xload_warp pairs
      // the segment's chunks the same way; a last odd chunk has its own)
      for (; c < sg.c1; c += 2) {
        const bool pair = c + 1 < sg.c1;
        const int ri1 = ri + 1 == kSlots ? 0 : ri + 1;
        const uint32_t rph1 = ri + 1 == kSlots ? rph ^ 1 : rph;
        if (prof) {
          n_chunks += pair ? 2 : 1;
          ok = mbar_wait_p(a, &s.full[ri], rph, -11, w_full) && mbar_wait_p(a, &s.xfull[xi], xph, -12, w_x) &&
               (!pair || mbar_wait_p(a, &s.full[ri1], rph1, -11, w_full));
        } else {
          ok = mbar_spin(a, &s.full[ri], rph, -11) && mbar_spin(a, &s.xfull[xi], xph, -12) &&
               (!pair || mbar_spin(a, &s.full[ri1], rph1, -11));
        }
        if (!__all_sync(0xffffffffu, ok)) return;
        if (stamp && first_pair && leader) s.tr[6] = globaltimer();   // first pair's operands ready
        first_pair = false;
        tc_fence_after();
        const uint64_t bx = bdesc0 + uint64_t(xi * (2 * XB >> 4));   // the stage of this pair
        if (no_mma) {                    // diagnostics: no MMA, release at once
          if (leader) {
            mbar_arrive_cnt(&s.empty[ri], kConsWarps);
            if (pair) mbar_arrive_cnt(&s.empty[ri1], kConsWarps);
            mbar_arrive(&s.xempty[xi]);
          }
        } else if (pair && dbg_mode) {
          umma_chunk8_dbg(dbg_mode, d, adesc0 + uint64_t(ri * (kSlotBytes >> 4)), bx,
                          adesc0 + uint64_t(ri1 * (kSlotBytes >> 4)), bx + uint64_t(XB >> 4),
                          idesc, c != sg.c0 ? 1u : 0u, &s.empty[ri], &s.empty[ri1], kConsWarps - 1,
                          &s.xempty[xi]);
        } else if (pair) {
          umma_chunk8(d, adesc0 + uint64_t(ri * (kSlotBytes >> 4)), bx,
                      adesc0 + uint64_t(ri1 * (kSlotBytes >> 4)), bx + uint64_t(XB >> 4),
                      idesc, c != sg.c0 ? 1u : 0u, &s.empty[ri], &s.empty[ri1], kConsWarps - 1,
                      &s.xempty[xi]);
        } else {
          // UMMA_K = 16 bf16 = 32 B along the swizzled row, 4 per 64-wide chunk;
          // ring slot: 8 arrivals (one per GEMV consumer warp), 7 plain, the
          // eighth from the commit when the MMAs have read the slot
          umma_chunk4(d, adesc0 + uint64_t(ri * (kSlotBytes >> 4)), bx,
                      idesc, c != sg.c0 ? 1u : 0u, &s.empty[ri], kConsWarps - 1, &s.xempty[xi]);
        }
        __syncwarp();
        if (pair) { ri = ri1 + 1 == kSlots ? 0 : ri1 + 1; rph = ri1 + 1 == kSlots ? rph1 ^ 1 : rph1; }
        else { ri = ri1; rph = rph1; }
        if (++xi == XS) { xi = 0; xph ^= 1; }
      }
      if (leader) {
        if (no_mma) mbar_arrive(&s.tile_done[buf]);
        else umma_commit(&s.tile_done[buf]);
      }
      __syncwarp();
      ++tb_k;
    }
    if (stamp && leader) s.tr[7] = globaltimer();                  // the job's last commit issued
  }
  if (leader && prof) {
    atomicAdd(&a.stats[S_W_MMA_FULL], w_full); atomicAdd(&a.stats[S_W_MMA_X], w_x);
    atomicAdd(&a.stats[S_W_MMA_TMEM], w_tmem); atomicAdd(&a.stats[S_MMA_CHUNKS], n_chunks);
  }
}

// Epilogue of 16 accumulator columns (batch rows 16j..16j+15) of weight row
// `row` (TMEM lane): residual / interleaved SiLU / logits + running argmax.
// 16 accumulator columns (batch rows 16j..) of TMEM lane quadrant q: the
// sum of the kAccs independent accumulators, in accumulator order.
__device__ __forceinline__ void tmem_acc16(uint32_t tmem_base, int q, int buf, int j, float (&v)[16]) {
  const uint32_t t0 = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(buf * kBufCols + 16 * j);
  tmem_ld16(t0, v);
#pragma unroll
  for (int k = 1; k < kAccs; ++k) {
    float w[16];
    tmem_ld16(t0 + uint32_t(k * kAccCols), w);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] += w[i];
  }
}

// Residual operands of one 16-column group (batch rows 16j..16j+15 of
// weight row `row`), loaded ahead of the accumulator so their round trip
// overlaps the MMA / piece wait.
__device__ __forceinline__ void umma_res16(const mk_gemm_params& p, int m0, int rows_m, int col,
                                           int j, float (&rv)[16]) {
  const uint16_t* res = reinterpret_cast<const uint16_t*>(p.res);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int bi = 16 * j + i;
    rv[i] = (p.epilogue == MK_EPI_RESIDUAL && bi < rows_m)
                ? bf2f(ldg16_cg(res + size_t(m0 + bi) * p.ldres + col)) : 0.f;
  }
}

__device__ __forceinline__ void umma_epi16(const KArgs& a, Smem& s, const mk_gemm_params& p, int m0, int rows_m,
                                           int out_col0, int row, int q, int lane, int cw, int j,
                                           const float (&v)[16], const float* rpre = nullptr) {
  if (p.epilogue == MK_EPI_LOGITS) {
    float* y = reinterpret_cast<float*>(p.y);
    const int col = out_col0 + row;
    const bool valid_col = col < p.y_cols;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int bi = 16 * j + i;
      float val = valid_col ? v[i] : -INFINITY;
      if (y && valid_col && bi < rows_m) y[size_t(m0 + bi) * p.ldy + col] = val;
      int idx = col;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, val, off);
        const int i2 = __shfl_xor_sync(0xffffffffu, idx, off);
        if (v2 > val || (v2 == val && i2 < idx)) { val = v2; idx = i2; }
      }
      if (lane == 0 && bi < rows_m) {
        float& bv = s.amx_val[cw][m0 + bi];
        int& bx = s.amx_idx[cw][m0 + bi];
        if (val > bv || (val == bv && idx < bx)) { bv = val; bx = idx; }
      }
    }
  } else if (p.epilogue == MK_EPI_PARTIAL) {
    const int col = out_col0 + row;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (16 * j + i < rows_m) tp_store(a, p, m0 + 16 * j + i, col, v[i]);
  } else if (p.epilogue == MK_EPI_SILU) {
    // rows 32q..32q+15 are gate rows 16q.., rows 32q+16.. the matching up rows
    uint16_t* y = reinterpret_cast<uint16_t*>(p.y);
    const int col = out_col0 + 16 * q + (lane & 15);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float u = __shfl_down_sync(0xffffffffu, v[i], 16);
      const int bi = 16 * j + i;
      if (lane < 16 && bi < rows_m)
        st_out(&y[size_t(m0 + bi) * p.ldy + col], f2bf(v[i] / (1.f + __expf(-v[i])) * u));
    }
  } else {
    uint16_t* y = reinterpret_cast<uint16_t*>(p.y);
    const int col = out_col0 + row;
    float rv[16];
    if (rpre) {
#pragma unroll
      for (int i = 0; i < 16; ++i) rv[i] = rpre[i];
    } else {
      umma_res16(p, m0, rows_m, col, j, rv);
    }
    float sq[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int bi = 16 * j + i;
      const uint16_t o = f2bf(v[i] + rv[i]);
      if (bi < rows_m) st_out(&y[size_t(m0 + bi) * p.ldy + col], o);
      sq[i] = bi < rows_m ? bf2f(o) * bf2f(o) : 0.f;
    }
    if (p.ss_out) {
      // the next RMSNorm's statistics: sum of squares of this warp's 32
      // output columns per batch row, one partial per (tile, TMEM quadrant)
#pragma unroll
      for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sq[i] += __shfl_xor_sync(0xffffffffu, sq[i], off);
      if (lane < 16 && 16 * j + lane < rows_m) {
        float mine = sq[0];
#pragma unroll
        for (int i = 1; i < 16; ++i) if (lane == i) mine = sq[i];
        p.ss_out[size_t(out_col0 / 32 + q) * p.M + m0 + 16 * j + lane] = mine;
      }
    }
  }
}

// All 8 consumer warps (CTA warps 4-11; TMEM lane quadrant q = warp % 4,
// warps q and q+4 take alternate 16-column groups): accumulator ->
// registers -> epilogue.  A K-split piece goes to the
// worker's piece slot ([col][128 rows] fp32, coalesced); the last piece of a
// tile sums all pieces in piece order and runs the epilogue.
#ifndef MK_PIECES_IN_FLIGHT
#define MK_PIECES_IN_FLIGHT 3
#endif
constexpr int kPiecesInFlight = MK_PIECES_IN_FLIGHT;   // K-split owner: piece loads per round trip
                                                         // (4 / 6 measured slower: B=64 +1.5 / +2.3 %)

__device__ void umma_epilogue(const KArgs& a, Smem& s, const mk_gemm_params& p, int w_in_task,
                              int ct, uint32_t& tb_k) {
  const int NT = umma_nt(p);
  const int lane = ct & 31;
  const int q = (ct >> 5) & 3;
  const int cw = ct >> 5;                 // consumer warp index (amx slot)
  const int half = ct >> 7;               // which column groups (j parity)
  const int chunks = p.K / p.T_K;
  if (p.ss_in) {
    // RMSNorm folded into the weights (W * gamma): 1/rms of every batch row
    // from the producer's per-tile partial sums of squares -- one round trip
    // while the MMAs of the first segment run
    const int b = ct >> 2, sub = ct & 3;
    float t = 0.f;
    if (b < p.M)
      for (int k = sub; k < p.ss_nparts; k += 4) t += __ldcg(p.ss_in + size_t(k) * p.M + b);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    if (sub == 0 && b < kAmaxRows) s.rsn[b] = rsqrtf(t / float(p.K) + p.norm_eps);
    bar_sync(1, kCons);
  }
  SegIter it;
  it.init(p, a.W, w_in_task);
  Seg g;
  while (it.next(g)) {
    const int m0 = g.m * p.T_M;
    const int rows_m = min(p.T_M, p.M - m0);
    const int buf = tb_k & 1;
    const bool whole = g.c0 == 0 && g.c1 == chunks;
    {
      const long long t0 = (a.debug & 4) ? clock64() : 0;
      mbar_wait_warp(a, &s.tile_done[buf], (tb_k >> 1) & 1, -14);
      if ((a.debug & 4) && ct == 128) atomicAdd(&a.stats[S_W_EPI_DONE], (unsigned long long)(clock64() - t0));
    }
    tc_fence_after();
    const int row = 32 * q + lane;        // weight row inside the tile
    const int out_col0 = p.y_col0 + g.n * p.T_N;
    if (whole) {
      for (int j = half; j < NT / 16; j += 2) {
        float rv[16], v[16];
        umma_res16(p, m0, rows_m, out_col0 + row, j, rv);
        tmem_acc16(s.tmem_base, q, buf, j, v);
        if (p.ss_in) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= s.rsn[(m0 + 16 * j + i) & (kAmaxRows - 1)];
        }
        umma_epi16(a, s, p, m0, rows_m, out_col0, row, q, lane, cw, j, v, rv);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tmem_free[buf]);
      ++tb_k;
      continue;
    }
    // K-split tile.  Its owner is the worker holding the tile's first chunk
    // (pi.first_w): that segment is the owner's LAST segment, so it is
    // streamed last and the owner reduces while nothing else of its range
    // is pending.  Every other piece goes TMEM -> piece slot -> release
    // signal (no round trip waited on); the owner keeps its own partial in
    // TMEM, waits for the n-1 signals, and sums all pieces in piece order
    // (first_w, first_w+1, ...: deterministic, arrival-order independent).
    const PieceInfo pi = tile_pieces(p, a.W, g.tile);
    if (w_in_task != pi.first_w) {
      if ((a.debug & 256) && a.trace && ct == 0) s.tr[6] = globaltimer();   // accumulator ready
      float* mine = piece_ptr(p, w_in_task, g.first ? 0 : 1);
      for (int j = half; j < NT / 16; j += 2) {
        float v[16];
        tmem_acc16(s.tmem_base, q, buf, j, v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (16 * j + i < rows_m) __stcg(mine + (16 * j + i) * 128 + row, v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tmem_free[buf]);
      ++tb_k;
      bar_sync(2, kCons);
      if (ct == 0) {                        // cumulative release of the CTA's stores
        if ((a.debug & 256) && a.trace) s.tr[7] = globaltimer();     // pieces stored, CTA joined
        fence_acq_rel_gpu();
        red_release_add(&a.sub_ctr[p.tile_ctr0 + g.tile], 1u);
      }
      continue;
    }
    // owner: wait for the n-1 other pieces (their signals were sent while
    // this worker streamed its own segment), then per column group: residual
    // operands and up to three pieces in flight together, own partial from
    // TMEM, sum in piece order, epilogue; the accumulator is released last
    if (ct == 0) {
      if (a.trace && !(a.debug & 288)) s.tr[7] = globaltimer();  // own accumulator ready
      const uint32_t target = uint32_t(pi.n - 1) * a.epoch;
      Spin sp;
      while ((int32_t)(ld_acquire(&a.sub_ctr[p.tile_ctr0 + g.tile]) - target) < 0)
        if (!sp.ok(a, -18)) break;
      if (a.trace && !(a.debug & 288)) s.tr[6] = globaltimer();  // the other pieces arrived
    }
    bar_sync(2, kCons);
    for (int j = half; j < NT / 16; j += 2) {
      float rv[16], v[16];
      umma_res16(p, m0, rows_m, out_col0 + row, j, rv);
      tmem_acc16(s.tmem_base, q, buf, j, v);
      for (int w0 = pi.first_w + 1; w0 <= pi.last_w; w0 += kPiecesInFlight) {
        float t[kPiecesInFlight][16];
#pragma unroll
        for (int u = 0; u < kPiecesInFlight; ++u) {
          const int w = w0 + u;
          const bool on = w <= pi.last_w && !pi.empty(w);
          const float* src = piece_ptr(p, on ? w : pi.first_w, 0);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            t[u][i] = (on && 16 * j + i < rows_m) ? __ldcg(src + (16 * j + i) * 128 + row) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kPiecesInFlight; ++u)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += t[u][i];
      }
      if (p.ss_in) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= s.rsn[(m0 + 16 * j + i) & (kAmaxRows - 1)];
      }
      umma_epi16(a, s, p, m0, rows_m, out_col0, row, q, lane, cw, j, v, rv);
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.tmem_free[buf]);
    ++tb_k;
  }
}

__device__ void run_gemm_umma(const KArgs& a, Smem& s, Ring& r, const mk_task& t, int tix,
                              int worker, int ct, uint32_t& xs_k, uint32_t& tb_k,
                              unsigned long long& tiles) {
  const mk_gemm_params& p = *P<mk_gemm_params>(a, t);
  const int w_in_task = t.level == MK_LEVEL_CHIPLET ? worker : 0;
  if (p.epilogue == MK_EPI_LOGITS) {
    for (int e = ct; e < kConsWarps * kAmaxRows; e += kCons) {
      s.amx_val[e / kAmaxRows][e % kAmaxRows] = -INFINITY;
      s.amx_idx[e / kAmaxRows][e % kAmaxRows] = 0x7fffffff;
    }
  }
  // count the unit's segments and ring slots, hand the job to the MMA warp
  int n_seg = 0;
  long long n_slots = 0;
  {
    SegIter it;
    it.init(p, a.W, w_in_task);
    Seg g;
    while (it.next(g)) {
      ++n_seg; n_slots += g.c1 - g.c0;
      if (ct == 0 && a.tile_log) {
        unsigned long long at = atomicAdd(a.tile_cursor, 1ull);
        if ((long long)at < a.tile_cap) {
          int32_t* rec = a.tile_log + at * 4;
          rec[0] = tix; rec[1] = (t.level == MK_LEVEL_CHIPLET ? t.die * a.W : 0) + worker;
          rec[2] = g.m; rec[3] = g.n;
        }
      }
    }
  }
  bar_sync(1, kCons);
  (void)tix;                        // the job was posted at dequeue (consumers())
  MK_TRACE(a, s, ct, 3);
  umma_epilogue(a, s, p, w_in_task, ct, tb_k);
  (void)xs_k;
  bar_sync(1, kCons);
  r.k += uint32_t(n_slots);
  if (ct == 0) tiles += n_seg;
  if (p.epilogue == MK_EPI_LOGITS) {
    const int slot = p.amax_base + w_in_task;
    // a CU tile task owns only its m-tile's rows of the shared slot
    const int b_lo = p.tile_m >= 0 ? p.tile_m * p.T_M : 0;
    const int b_hi = p.tile_m >= 0 ? min(p.M, b_lo + p.T_M) : p.M;
    for (int b = b_lo + ct; b < b_hi && b < kAmaxRows; b += kCons) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
      for (int w = 0; w < kConsWarps; ++w) {
        const float v = s.amx_val[w][b];
        const int i = s.amx_idx[w][b];
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      p.amax_val[size_t(slot) * p.amax_stride + b] = best;
      p.amax_idx[size_t(slot) * p.amax_stride + b] = bi;
    }
    bar_sync(1, kCons);
  }
}

template <int F>
__device__ void run_gemm(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                         const mk_task& t, int worker, int gw, int tix, int ct,
                         unsigned long long& tiles) {
  const mk_gemm_params& p = *P<mk_gemm_params>(a, t);
  const int w_in_task = t.level == MK_LEVEL_CHIPLET ? worker : 0;
  if (p.epilogue == MK_EPI_LOGITS) {
    for (int e = ct; e < kConsWarps * kAmaxRows; e += kCons) {
      s.amx_val[e / kAmaxRows][e % kAmaxRows] = -INFINITY;
      s.amx_idx[e / kAmaxRows][e % kAmaxRows] = 0x7fffffff;
    }
    bar_sync(1, kCons);
  }
  if constexpr ((F & kFeatLean) != 0) {
    if constexpr ((F & kFeatUmma) == 0) {          // batch-1 bodies only
      if (p.ksplit) {
        if (p.stage_x) gemm_task_ks<1, true>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
        else gemm_task_ks<1, false>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
      } else if (p.stage_x) gemm_task<1, true>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
      else gemm_task<1, false>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
    } else if (ct == 0) {
      raise_error(a, MK_ERR_CONFIG, -300);         // mk_create picked the wrong instance
    }
    return;
  }
  const int rows = min(p.T_M, p.M);
#define MK_GEMM_NB(XSV)                                                              \
  if (rows <= 1) gemm_task<1, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else if (rows <= 2) gemm_task<2, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else if (rows <= 4) gemm_task<4, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else if (rows <= 8) gemm_task<8, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else gemm_task<16, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
  if ((F & kFeatKsplit) && p.ksplit) {
#define MK_GEMM_KS(XSV)                                                                 \
  if (rows <= 1) gemm_task_ks<1, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);     \
  else if (rows <= 2) gemm_task_ks<2, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else if (rows <= 4) gemm_task_ks<4, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles); \
  else gemm_task_ks<8, XSV>(a, s, ring, r, p, w_in_task, gw, tix, ct, tiles);
    if (p.stage_x) { MK_GEMM_KS(true) } else { MK_GEMM_KS(false) }
#undef MK_GEMM_KS
  } else if (p.stage_x) { MK_GEMM_NB(true) } else { MK_GEMM_NB(false) }
#undef MK_GEMM_NB
}

// ---------------------------------------------------------------------------
// RMSNorm (Qwen3RMSNorm: fp32 statistics, cast, gamma multiply), optional
// embedding gather for layer 0.  When the lowering fused the norm into the
// consuming GEMM (mk_norm_params.fused), only the gather remains.
// ---------------------------------------------------------------------------
__device__ float block_sum(Smem& s, float v, int ct) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((ct & 31) == 0) s.bred[ct >> 5] = v;
  bar_sync(1, kCons);
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < kConsWarps; ++w) tot += s.bred[w];
  bar_sync(1, kCons);
  return tot;
}

__device__ void run_rmsnorm(const KArgs& a, Smem& s, const mk_task& t, int ib, int ie, int ct) {
  const mk_norm_params& p = *P<mk_norm_params>(a, t);
  // folded / fused into the consuming GEMM and no gather or statistics to
  // produce: nothing to compute (the unit still orders and signals its event)
  if (p.fused && !p.embed && !p.ss_out && !p.x_store) return;
  const uint16_t* gam = reinterpret_cast<const uint16_t*>(p.gamma);
  constexpr int kRegChunks = 16;     // rows up to 16 * 256 wide stay in registers
  if (p.d <= kRegChunks * 256) {
    // one warp per row: the row and gamma are loaded in one round trip and
    // kept in registers, the statistics reduced by shuffles (no CTA barrier)
    const int warp = ct >> 5, lane = ct & 31;
    const uint64_t pol = policy_evict_last();
    for (int b = ib + warp; b < ie; b += kConsWarps) {
      const uint16_t* src = p.embed ? reinterpret_cast<const uint16_t*>(p.embed) + size_t(p.tokens[b]) * p.d
                                    : reinterpret_cast<const uint16_t*>(p.x) + size_t(b) * p.d;
      uint16_t* xs = p.x_store ? reinterpret_cast<uint16_t*>(p.x_store) + size_t(b) * p.d : nullptr;
      uint4 xv[kRegChunks], gv[kRegChunks];
#pragma unroll
      for (int i = 0; i < kRegChunks; ++i) {
        const int k = lane * 8 + i * 256;
        const bool on = k < p.d;
        xv[i] = on ? ldg128_cg(src + k) : make_uint4(0, 0, 0, 0);
        gv[i] = (on && !p.fused) ? ldg128_hint(gam + k, pol) : make_uint4(0, 0, 0, 0);
      }
      if (p.fused) {            // consumer GEMM normalises; keep only the gather
        if (xs) {
#pragma unroll
          for (int i = 0; i < kRegChunks; ++i)
            if (lane * 8 + i * 256 < p.d) *reinterpret_cast<uint4*>(xs + lane * 8 + i * 256) = xv[i];
        }
        if (p.ss_out) {         // the folded-norm consumer's statistics (one partial)
          float ss = 0.f;
#pragma unroll
          for (int i = 0; i < kRegChunks; ++i) {
            float f[8];
            unpack8(xv[i], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
          if (lane == 0) p.ss_out[b] = ss;
        }
        continue;
      }
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < kRegChunks; ++i) {
        float f[8];
        unpack8(xv[i], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      const float rs = rsqrtf(ss / float(p.d) + p.eps);
      uint16_t* y = reinterpret_cast<uint16_t*>(p.y) + size_t(b) * p.d;
#pragma unroll
      for (int i = 0; i < kRegChunks; ++i) {
        const int k = lane * 8 + i * 256;
        if (k >= p.d) continue;
        float f[8], g[8];
        unpack8(xv[i], f);
        unpack8(gv[i], g);
        uint16_t o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xn = bf2f(f2bf(f[e] * rs));   // hidden_states.to(input_dtype)
          o[e] = f2bf(g[e] * xn);                   // weight * hidden_states
        }
        *reinterpret_cast<uint4*>(y + k) = *reinterpret_cast<uint4*>(o);
        if (xs) *reinterpret_cast<uint4*>(xs + k) = xv[i];
      }
    }
    return;
  }
  for (int b = ib; b < ie; ++b) {
    const uint16_t* src;
    if (p.embed) src = reinterpret_cast<const uint16_t*>(p.embed) + size_t(p.tokens[b]) * p.d;
    else src = reinterpret_cast<const uint16_t*>(p.x) + size_t(b) * p.d;
    uint16_t* xs = p.x_store ? reinterpret_cast<uint16_t*>(p.x_store) + size_t(b) * p.d : nullptr;
    if (p.fused) {            // consumer GEMM normalises; keep only the gather
      if (xs)
        for (int k = ct * 8; k < p.d; k += kCons * 8)
          *reinterpret_cast<uint4*>(xs + k) = ldg128_cg(src + k);
      continue;
    }
    float ss = 0.f;
    for (int k = ct * 8; k < p.d; k += kCons * 8) {
      float f[8];
      unpack8(ldg128_cg(src + k), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
    }
    const float tot = block_sum(s, ss, ct);
    const float rs = rsqrtf(tot / float(p.d) + p.eps);
    uint16_t* y = reinterpret_cast<uint16_t*>(p.y) + size_t(b) * p.d;
    for (int k = ct * 8; k < p.d; k += kCons * 8) {
      const uint4 raw = ldg128_cg(src + k);
      float f[8], g[8];
      unpack8(raw, f);
      unpack8(ldg128_cg(gam + k), g);
      uint16_t o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xn = bf2f(f2bf(f[e] * rs));   // hidden_states.to(input_dtype)
        o[e] = f2bf(g[e] * xn);                   // weight * hidden_states
      }
      *reinterpret_cast<uint4*>(y + k) = *reinterpret_cast<uint4*>(o);
      if (xs) *reinterpret_cast<uint4*>(xs + k) = raw;
    }
  }
}

// ---------------------------------------------------------------------------
// Attention partial: QK-norm + RoPE (+ KV append for the new token) and a
// split-KV online-softmax partial over cached tokens streamed into the ring.
// ---------------------------------------------------------------------------
// Barrier-free split-KV attention.  Warp w serves q head j = w % G of the
// kv group and token subset sub = w / G; lane (tg, dl) holds dims
// [8*dl, 8*dl+8) of token group tg.  Every warp computes its own
// q_norm + RoPE (and, for the split holding the new token, k_norm + RoPE and
// v) in registers: the rotate_half partner dims come from lane dl^(LPT/2) by
// shuffle.  Each warp writes its own partial (m, l, o) as piece
// split*nsub + sub, so no shared memory and no CTA barrier is needed; the
// reduce task merges the pieces.
template <int HD>
__device__ __forceinline__ void norm_rope8(const uint16_t* src, const uint16_t* gam, float eps,
                                           const float* cs, const float* sn, int dl,
                                           float (&out)[8]) {
  constexpr int LPT = HD / 8;
  constexpr int H2 = HD / 2;
  const uint64_t pol = policy_evict_last();
  const uint4 xv = ldg128_cg(src + dl * 8);
  const uint4 gv = ldg128_hint(gam + dl * 8, pol);
  const int ci = (dl * 8) % H2;
  const uint4 c0u = ldg128_hint(cs + ci, pol), c1u = ldg128_hint(cs + ci + 4, pol);
  const uint4 s0u = ldg128_hint(sn + ci, pol), s1u = ldg128_hint(sn + ci + 4, pol);
  const float4 c0 = make_float4(__uint_as_float(c0u.x), __uint_as_float(c0u.y), __uint_as_float(c0u.z), __uint_as_float(c0u.w));
  const float4 c1 = make_float4(__uint_as_float(c1u.x), __uint_as_float(c1u.y), __uint_as_float(c1u.z), __uint_as_float(c1u.w));
  const float4 s0 = make_float4(__uint_as_float(s0u.x), __uint_as_float(s0u.y), __uint_as_float(s0u.z), __uint_as_float(s0u.w));
  const float4 s1 = make_float4(__uint_as_float(s1u.x), __uint_as_float(s1u.y), __uint_as_float(s1u.z), __uint_as_float(s1u.w));
  float f[8], g[8];
  unpack8(xv, f);
  unpack8(gv, g);
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
#pragma unroll
  for (int off = LPT >> 1; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  const float rs = rsqrtf(ss / float(HD) + eps);
  float xn[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) xn[e] = g[e] * bf2f(f2bf(f[e] * rs));
  const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  const bool first_half = dl < LPT / 2;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float partner = __shfl_xor_sync(0xffffffffu, xn[e], LPT / 2);
    out[e] = first_half ? xn[e] * cv[e] - partner * sv[e] : xn[e] * cv[e] + partner * sv[e];
  }
}

__device__ __forceinline__ float ex2(float x) {   // 2^x, -inf -> 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void phase_rec(const KArgs& a, int kind, int item, uint64_t t0, uint64_t t1) {
  unsigned long long at = atomicAdd(a.log_cursor, 1ull);
  if ((long long)at >= a.log_cap) return;
  mk_log_rec& r = a.log[at];
  r.kind = kind; r.task = -1; r.item_begin = item; r.worker = -1;
  r.smid = (int)smid(); r.die = -1; r.t_start = t0; r.t_end = t1;
}

// One pass = up to 8/G items: warp w serves item (w / G) of the pass and q
// head (w % G) of the kv group over the item's whole split, 8 tokens per
// lane group per iteration (independent dot/shuffle/exp chains).  The warp
// writes its head's partial (m, l, o) directly -- no shared memory, no CTA
// barrier.  Every warp arrives on every ring slot of the pass.
template <int HD>
__device__ void attn_pass(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                          const mk_attn_params& p, int i0, int i1, int ct) {
  constexpr int LPT = HD / 8;          // lanes per token
  constexpr int TPI = 32 / LPT;        // tokens per warp per sub-step
  constexpr int CH = 4;                // tokens per lane group per iteration
  const int G = p.group;
  const int nsub = p.sub_splits;       // warps sharing one (item, head)
  const int warp = ct >> 5, lane = ct & 31;
  const int head = warp % G, sub = (warp / G) % nsub, slot_item = warp / (G * nsub);
  const int tg = lane / LPT, dl = lane % LPT;
  const bool trace = a.log != nullptr && ct == 0;
  const uint64_t ph0 = trace ? globaltimer() : 0;

  // this warp's item and the ring slots of every item in the pass
  int my_slot = -1, n_slots = 0;
  int item = -1, pos = 0, t0 = 0, nc = 0;
  bool has_new = false;
  for (int it = i0; it < i1; ++it) {
    const int b = it / p.n_splits, sp = it % p.n_splits;
    const int ps = row_pos(p.positions, b);
    const int tt0 = sp * p.split;
    const int nci = tt0 > ps ? 0 : min(p.split, ps - tt0);
    if (it - i0 == slot_item) {
      item = it; pos = ps; t0 = tt0; nc = nci;
      has_new = tt0 <= ps && ps < tt0 + p.split;
      if (nci > 0) my_slot = n_slots;
    }
    if (nci > 0) n_slots += 2;
  }
  const bool active = item >= 0 && t0 <= pos;
  const int b = active ? item / p.n_splits : 0;
  const int sp = active ? item % p.n_splits : 0;
  if (active && !pos_ok(a, pos, p.t_max, b)) { pos = p.t_max - 1; has_new = false; }

  float q8[8];
  const uint16_t* qkv = reinterpret_cast<const uint16_t*>(p.qkv) + size_t(b) * p.ldqkv;
  const float* cs = p.rope_cos + size_t(pos) * (HD / 2);
  const float* sn = p.rope_sin + size_t(pos) * (HD / 2);
  if (active) {
    norm_rope8<HD>(qkv + (p.kv_head * G + head) * HD, reinterpret_cast<const uint16_t*>(p.q_gamma),
                   p.eps, cs, sn, dl, q8);
    const float qscale = p.scale * 1.4426950408889634f;
#pragma unroll
    for (int e = 0; e < 8; ++e) q8[e] *= qscale;
  }
  const uint64_t ph1 = trace ? globaltimer() : 0;
  uint32_t kslot = 0, vslot = 0;
  if (active && my_slot >= 0) {
    Ring rk = r; rk.k += my_slot;
    cons_wait_slot(a, s, rk);
    kslot = smem_u32(ring) + uint32_t(rk.k % kSlots) * kSlotBytes;
    Ring rv = rk; ++rv.k;
    cons_wait_slot(a, s, rv);
    vslot = smem_u32(ring) + uint32_t(rv.k % kSlots) * kSlotBytes;
  }
  const uint64_t ph2 = trace ? globaltimer() : 0;
  float mx = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = 0.f;
  // cached tokens only: TPI*CH per warp step, tail masked
  const int ncached = active ? nc : 0;
  for (int tb = sub * TPI * CH; tb < ncached; tb += nsub * TPI * CH) {
    float sc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int tk = tb + c * TPI + tg;
      uint4 k4 = make_uint4(0, 0, 0, 0);
      if (tk < ncached)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(k4.x), "=r"(k4.y), "=r"(k4.z), "=r"(k4.w)
                     : "r"(kslot + uint32_t(tk * HD * 2 + dl * 16)) : "memory");
      float acc = q8[0] * bf16lo(k4.x);
      acc = fmaf(q8[1], bf16hi(k4.x), acc);
      acc = fmaf(q8[2], bf16lo(k4.y), acc);
      acc = fmaf(q8[3], bf16hi(k4.y), acc);
      acc = fmaf(q8[4], bf16lo(k4.z), acc);
      acc = fmaf(q8[5], bf16hi(k4.z), acc);
      acc = fmaf(q8[6], bf16lo(k4.w), acc);
      acc = fmaf(q8[7], bf16hi(k4.w), acc);
      sc[c] = acc;
    }
#pragma unroll
    for (int off = LPT >> 1; off > 0; off >>= 1)
#pragma unroll
      for (int c = 0; c < CH; ++c) sc[c] += __shfl_xor_sync(0xffffffffu, sc[c], off);
    float cm = -INFINITY;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (tb + c * TPI + tg >= ncached) sc[c] = -INFINITY;
      cm = fmaxf(cm, sc[c]);
    }
    const float mn = fmaxf(mx, cm);
    if (mn != -INFINITY) {
      const float corr = ex2(mx - mn);
      l *= corr;
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] *= corr;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int tk = tb + c * TPI + tg;
        const float pr = ex2(sc[c] - mn);     // 0 for padded tokens
        l += pr;
        if (tk < ncached) {
          uint4 v4;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v4.x), "=r"(v4.y), "=r"(v4.z), "=r"(v4.w)
                       : "r"(vslot + uint32_t(tk * HD * 2 + dl * 16)) : "memory");
          o[0] = fmaf(pr, bf16lo(v4.x), o[0]); o[1] = fmaf(pr, bf16hi(v4.x), o[1]);
          o[2] = fmaf(pr, bf16lo(v4.y), o[2]); o[3] = fmaf(pr, bf16hi(v4.y), o[3]);
          o[4] = fmaf(pr, bf16lo(v4.z), o[4]); o[5] = fmaf(pr, bf16hi(v4.z), o[5]);
          o[6] = fmaf(pr, bf16lo(v4.w), o[6]); o[7] = fmaf(pr, bf16hi(v4.w), o[7]);
        }
      }
      mx = mn;
    }
  }
  // the token being decoded: k_norm + RoPE and v from the qkv row, appended
  // to the cache, folded into token group 0 of the sub-0 warp
  if (active && has_new) {
    float kn[8];
    norm_rope8<HD>(qkv + p.q_heads * HD + p.kv_head * HD,
                   reinterpret_cast<const uint16_t*>(p.k_gamma), p.eps, cs, sn, dl, kn);
    const uint4 vv = ldg128_cg(qkv + (p.q_heads + p.kv_heads) * HD + p.kv_head * HD + dl * 8);
    uint16_t kb[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { kb[e] = f2bf(kn[e]); kn[e] = bf2f(kb[e]); }   // attend to the cached key
    if (head == 0 && sub == 0 && tg == 0) {
      const size_t crow = kv_off(p, b, pos) + dl * 8;
      *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.k_cache) + crow) = *reinterpret_cast<uint4*>(kb);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.v_cache) + crow) = vv;
    }
    float sc = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) sc = fmaf(q8[e], kn[e], sc);
#pragma unroll
    for (int off = LPT >> 1; off > 0; off >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
    if (sub == 0 && tg == 0) {
      float vf[8];
      unpack8(vv, vf);
      const float mn = fmaxf(mx, sc);
      const float corr = ex2(mx - mn), pr = ex2(sc - mn);
      l = l * corr + pr;
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = fmaf(o[e], corr, pr * vf[e]);
      mx = mn;
    }
  }
  for (int k = 0; k < n_slots; ++k) cons_release_slot(s, r);
  // merge the warp's token groups (lanes tg and tg' hold the same dims)
#pragma unroll
  for (int off = LPT; off < 32; off <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, off);
    const float l2 = __shfl_xor_sync(0xffffffffu, l, off);
    const float mn = fmaxf(mx, m2);
    const float f1 = mn == -INFINITY ? 0.f : exp2f(mx - mn);
    const float f2 = mn == -INFINITY ? 0.f : exp2f(m2 - mn);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float o2 = __shfl_xor_sync(0xffffffffu, o[e], off);
      o[e] = o[e] * f1 + o2 * f2;
    }
    l = l * f1 + l2 * f2;
    mx = mn;
  }
  const uint64_t ph3 = trace ? globaltimer() : 0;
  if (nsub > 1) {
    // sub-warps of an (item, head) hand their state to sub 0 through smem
    float* xch = s.u.at.xch[warp];
    if (sub > 0 && tg == 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) xch[dl * 8 + e] = o[e];
      if (dl == 0) { xch[HD] = mx; xch[HD + 1] = l; }
    }
    bar_sync(1, kCons);
    if (sub == 0) {
      for (int k = 1; k < nsub; ++k) {
        const float* src = s.u.at.xch[warp + k * G];
        const float m2 = src[HD], l2 = src[HD + 1];
        const float mn = fmaxf(mx, m2);
        const float f1 = mn == -INFINITY ? 0.f : ex2(mx - mn);
        const float f2 = mn == -INFINITY ? 0.f : ex2(m2 - mn);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = o[e] * f1 + src[dl * 8 + e] * f2;
        l = l * f1 + l2 * f2;
        mx = mn;
      }
    }
    bar_sync(1, kCons);            // xch reusable by the next pass
  }
  if (active && tg == 0 && sub == 0) {
    float* dst = p.partial + (((size_t(b) * p.kv_heads + p.kv_head) * p.n_splits + sp) * G + head) * (HD + 4);
    *reinterpret_cast<float4*>(dst + dl * 8) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(dst + dl * 8 + 4) = make_float4(o[4], o[5], o[6], o[7]);
    if (dl == 0) { dst[HD] = mx; dst[HD + 1] = l; }
  }
  if (trace) {
    phase_rec(a, 2, i0, ph0, ph1);       // prologue (q/k norm + rope)
    phase_rec(a, 3, i0, ph1, ph2);       // waiting for the K/V slots
    phase_rec(a, 4, i0, ph2, ph3);       // token loop
  }
}

// ---------------------------------------------------------------------------
// Tensor-core split-KV attention (head_dim 128, 64-token splits).  The K/V
// cache rows are stored with their 16-byte chunks XOR-swizzled by
// (token & 7), so the ring slots feed ldmatrix without bank conflicts.  A
// pass holds 8 / wpi items (item = (row, split) of one kv head); wpi warps
// share an item, each over 64 / wpi tokens:
//   S[G heads x tokens] = Q K^T    mma.m16n8k16 (A rows = the G query heads)
//   online softmax in registers     (quad shuffles, ex2, log2-domain max)
//   O[G x 128] += P V               (P re-packed from the S fragments, V via
//                                    ldmatrix.trans)
// The warps of an item merge (m, l, o) through shared memory; the item's
// first warp writes the split partial for the reduce task.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t kv_swz(int token, int chunk) {   // byte offset in a slot
  return uint32_t(token * (kAttnHD * 2) + ((chunk ^ (token & 7)) << 4));
}

constexpr int kQRows = 8;                       // rows whose q a unit pre-rotates
struct AttnMmaScratch {
  uint16_t q[kConsWarps][kAttnMaxG][kAttnHD];  // per warp: normed + roped q of the group
  uint16_t qrow[kQRows][kAttnMaxG][kAttnHD];   // per unit: normed + roped q of its rows
  union {
    float xch[kConsWarps][kAttnMaxG][kAttnHD + 4];  // pass variant: (o[128], m, l) per head
    struct {                                        // chunked prefill: the chunk's
      uint16_t k[kChunkRows][kAttnHD];              //   normed + roped k rows
      uint16_t v[kChunkRows][kAttnHD];              //   and v rows (this kv head)
    } ch;
  };
};
static_assert(sizeof(AttnMmaScratch) <= size_t(kXsBytes), "attention scratch exceeds the union");

// Wait for ring position kpos.  Barrier-free warps may wait more than one
// ring lap ahead of the fill, where the mbarrier parity aliases: they also
// require the fetch warp's position tag of the slot to match.
__device__ __forceinline__ void attn_wait_slot(const KArgs& a, Smem& s, uint32_t kpos, bool tagged) {
  const int i = int(kpos % kSlots);
  const uint32_t par = (kpos / kSlots) & 1;
  if (!tagged) { mbar_wait(a, &s.full[i], par, -3); return; }
  Spin sp;
  for (;;) {
    if (*reinterpret_cast<volatile uint32_t*>(&s.slot_tag[i]) == kpos && mbar_test_wait(&s.full[i], par)) return;
    if (!sp.ok(a, -3)) return;
  }
}

// One warp's tokens [tok0, tok0 + tpw) of item (b, split at t0): q_norm +
// RoPE of the group's heads, K/V slots at ring positions kpos, kpos + 1, the
// decoded token folded into the slots (and appended to the cache), then
// S = Q K^T, online softmax and O = P V in registers.
__device__ __forceinline__ void attn_mma_tokens(const KArgs& a, Smem& s, uint8_t* ring,
                                                const mk_attn_params& p, int b, int pos, int t0,
                                                int nvalid, int tok0, int tpw, uint32_t kpos,
                                                bool tagged, int warp, int lane,
                                                float (&o)[16][4], float& m_run, float& l_run,
                                                bool trace, uint64_t& ph1, uint64_t& ph2,
                                                const uint16_t* qpre = nullptr) {
  const int G = p.group;
  const int g = lane >> 2, c = lane & 3;
  AttnMmaScratch& sc = *reinterpret_cast<AttnMmaScratch*>(s.u.xs);
  // q of the item's row: pre-rotated once per unit (qpre, [G][128]) or
  // normed + roped here into the warp's scratch
  const uint16_t* qs = qpre ? qpre : &sc.q[warp][0][0];
    const uint16_t* qkv = reinterpret_cast<const uint16_t*>(p.qkv) + size_t(b) * p.ldqkv;
    const float* cs = p.rope_cos + size_t(pos) * (kAttnHD / 2);
    const float* sn = p.rope_sin + size_t(pos) * (kAttnHD / 2);
    const int dl = lane & 15, half = lane >> 4;
    // q_norm + RoPE of the item's G heads -> bf16 (unscaled, as the model's q)
    for (int h = half; h < G && !qpre; h += 2) {
      float qv[8];
      norm_rope8<kAttnHD>(qkv + (p.kv_head * G + h) * kAttnHD, reinterpret_cast<const uint16_t*>(p.q_gamma),
                          p.eps, cs, sn, dl, qv);
      uint4 pk;
      pk.x = pack_bf16(qv[0], qv[1]); pk.y = pack_bf16(qv[2], qv[3]);
      pk.z = pack_bf16(qv[4], qv[5]); pk.w = pack_bf16(qv[6], qv[7]);
      *reinterpret_cast<uint4*>(&sc.q[warp][h][dl * 8]) = pk;
    }
    if (trace) ph1 = globaltimer();
    attn_wait_slot(a, s, kpos, tagged);
    attn_wait_slot(a, s, kpos + 1, tagged);
    uint8_t* kslot = ring + size_t(kpos % kSlots) * kSlotBytes;
    uint8_t* vslot = ring + size_t((kpos + 1) % kSlots) * kSlotBytes;
    if (trace) ph2 = globaltimer();
    // the token being decoded: k_norm + RoPE and v from the qkv row, into
    // the smem slots (and appended to the cache) by the warp that owns it
    const int nt = pos - t0;
    if (nt >= tok0 && nt < tok0 + tpw) {
      float kn[8];
      norm_rope8<kAttnHD>(qkv + p.q_heads * kAttnHD + p.kv_head * kAttnHD,
                          reinterpret_cast<const uint16_t*>(p.k_gamma), p.eps, cs, sn, dl, kn);
      uint4 kv4;
      if (half == 0) {
        kv4.x = pack_bf16(kn[0], kn[1]); kv4.y = pack_bf16(kn[2], kn[3]);
        kv4.z = pack_bf16(kn[4], kn[5]); kv4.w = pack_bf16(kn[6], kn[7]);
      } else {
        kv4 = ldg128_cg(qkv + (p.q_heads + p.kv_heads) * kAttnHD + p.kv_head * kAttnHD + dl * 8);
      }
      const uint32_t off = kv_swz(nt, dl);
      *reinterpret_cast<uint4*>((half == 0 ? kslot : vslot) + off) = kv4;
      const size_t crow = kv_off(p, b, pos);
      uint16_t* cache = reinterpret_cast<uint16_t*>(half == 0 ? p.k_cache : p.v_cache);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(cache + crow) + ((dl ^ (pos & 7)) << 4)) = kv4;
    }
    if (p.prefill) {
      // chunked prefill: the chunk's earlier tokens (other rows of this
      // launch, appended concurrently) come from the unit's staged rows, not
      // from the cache the slots were loaded from
      const int p0 = row_pos(p.positions, 0);
      const int lo = max(t0 + tok0, p0), hi = min(pos - 1, t0 + tok0 + tpw - 1);
      for (int P = lo + (lane >> 4); P <= hi; P += 2) {
        const int r = P - p0;
        const uint32_t off = kv_swz(P - t0, dl);
        *reinterpret_cast<uint4*>(kslot + off) = *reinterpret_cast<const uint4*>(&sc.ch.k[r][dl * 8]);
        *reinterpret_cast<uint4*>(vslot + off) = *reinterpret_cast<const uint4*>(&sc.ch.v[r][dl * 8]);
      }
    }
    __syncwarp();
    // Q fragments: row g = head g (g < G), 8 k-steps of 16 dims
    uint32_t qa0[8], qa2[8];
#pragma unroll
    for (int st = 0; st < 8; ++st) {
      qa0[st] = g < G ? *reinterpret_cast<const uint32_t*>(qs + g * kAttnHD + 16 * st + 2 * c) : 0u;
      qa2[st] = g < G ? *reinterpret_cast<const uint32_t*>(qs + g * kAttnHD + 16 * st + 8 + 2 * c) : 0u;
    }
    const uint32_t ks = smem_u32(kslot), vs = smem_u32(vslot);
    const float qscale = p.scale * 1.4426950408889634f;
    // S = Q K^T over the warp's tokens, n-tile j = tokens tok0 + 8j ..
    float sfr[8][2];
    const int nj = tpw / 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sfr[j][0] = sfr[j][1] = -INFINITY;
      if (j >= nj) continue;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int tk = tok0 + 8 * j + (lane & 7);
#pragma unroll
      for (int st = 0; st < 8; st += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks + kv_swz(tk, 2 * st + (lane >> 3)), b0, b1, b2, b3);
        mma_bf16_16816(acc, qa0[st], qa2[st], b0, b1);
        mma_bf16_16816(acc, qa0[st + 1], qa2[st + 1], b2, b3);
      }
      const int t_a = tok0 + 8 * j + 2 * c;
      sfr[j][0] = t_a < nvalid ? acc[0] * qscale : -INFINITY;
      sfr[j][1] = t_a + 1 < nvalid ? acc[1] * qscale : -INFINITY;
    }
    // softmax over the warp's tokens (row g spread over the lane quad)
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) mx = fmaxf(mx, fmaxf(sfr[j][0], sfr[j][1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    float lsum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sfr[j][0] = mx == -INFINITY ? 0.f : ex2(sfr[j][0] - mx);
      sfr[j][1] = mx == -INFINITY ? 0.f : ex2(sfr[j][1] - mx);
      lsum += sfr[j][0] + sfr[j][1];
    }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    m_run = mx; l_run = lsum;
    // O = P V: k-step t = tokens tok0 + 16t .., n-tiles of 8 dims
    const int nt16 = tpw / 16;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t >= nt16) continue;
      const uint32_t pa0 = pack_bf16(sfr[2 * t][0], sfr[2 * t][1]);
      const uint32_t pa2 = pack_bf16(sfr[2 * t + 1][0], sfr[2 * t + 1][1]);
      const int tv = tok0 + 16 * t + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vs + kv_swz(tv, u + (lane >> 4)), b0, b1, b2, b3);
        mma_bf16_16816(o[u], pa0, pa2, b0, b1);
        mma_bf16_16816(o[u + 1], pa0, pa2, b2, b3);
      }
    }
}

__device__ void attn_mma_pass(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                              const mk_attn_params& p, int i0, int i1, int ct) {
  const int G = p.group;
  const int wpi = p.sub_splits;              // warps per item (1, 2 or 4)
  const int tpw = kAttnSplit / wpi;          // tokens per warp
  const int warp = ct >> 5, lane = ct & 31;
  const int slot_item = warp / wpi, sw = warp % wpi;
  const int g = lane >> 2, c = lane & 3;     // mma fragment row / column pair
  AttnMmaScratch& sc = *reinterpret_cast<AttnMmaScratch*>(s.u.xs);

  // items of the pass and their ring slots (K, V per active item)
  int my_slot = -1, n_slots = 0, item = -1, pos = 0, t0 = 0;
  for (int it = i0; it < i1; ++it) {
    const int b = it / p.n_splits, sp = it % p.n_splits;
    const int ps = row_pos(p.positions, b);
    const int tt0 = sp * kAttnSplit;
    if (it - i0 == slot_item) { item = it; pos = ps; t0 = tt0; if (tt0 <= ps) my_slot = n_slots; }
    if (tt0 <= ps) n_slots += 2;
  }
  const bool active = my_slot >= 0;
  const int b = active ? item / p.n_splits : 0;
  const int sp = active ? item % p.n_splits : 0;
  if (active && !pos_ok(a, pos, p.t_max, b)) pos = p.t_max - 1;
  const int nvalid = active ? min(kAttnSplit, pos + 1 - t0) : 0;   // incl. the new token
  const int tok0 = sw * tpw;                                         // this warp's tokens
  const bool trace = a.log != nullptr && ct == 0;
  uint64_t ph0 = trace ? globaltimer() : 0, ph1 = ph0, ph2 = ph0;

  float m_run = -INFINITY, l_run = 0.f;
  float o[16][4];
#pragma unroll
  for (int u = 0; u < 16; ++u) o[u][0] = o[u][1] = o[u][2] = o[u][3] = 0.f;

  if (active && tok0 < nvalid)
    attn_mma_tokens(a, s, ring, p, b, pos, t0, nvalid, tok0, tpw, r.k + uint32_t(my_slot), false,
                    warp, lane, o, m_run, l_run, trace, ph1, ph2);
  // release the item's K/V slots as soon as its warps are done (each of the
  // wpi warps supplies 8 / wpi of the slot's 8 arrivals), so the fetch warp
  // refills them with the next pass while this one merges
  __syncwarp();
  if (active && lane == 0) {
    const uint32_t kpos = r.k + uint32_t(my_slot);
    mbar_arrive_cnt(&s.empty[kpos % kSlots], uint32_t(kConsWarps / wpi));
    mbar_arrive_cnt(&s.empty[(kpos + 1) % kSlots], uint32_t(kConsWarps / wpi));
  }
  r.k += uint32_t(n_slots);
  const uint64_t ph3 = trace ? globaltimer() : 0;

  // merge the item's warps; the first warp writes the split partial
  if (wpi > 1) {
    if (active && g < G) {
      float* x = sc.xch[warp][g];
#pragma unroll
      for (int u = 0; u < 16; ++u) { x[8 * u + 2 * c] = o[u][0]; x[8 * u + 2 * c + 1] = o[u][1]; }
      if (c == 0) { x[kAttnHD] = m_run; x[kAttnHD + 1] = l_run; }
    }
    bar_sync(1, kCons);
    if (active && sw == 0) {
      for (int e = lane; e < G * kAttnHD; e += 32) {
        const int h = e / kAttnHD, d = e % kAttnHD;
        float M = -INFINITY;
        for (int k = 0; k < wpi; ++k) M = fmaxf(M, sc.xch[warp + k][h][kAttnHD]);
        float on = 0.f, ln = 0.f;
        for (int k = 0; k < wpi; ++k) {
          const float* x = sc.xch[warp + k][h];
          const float f = M == -INFINITY ? 0.f : ex2(x[kAttnHD] - M);
          on = fmaf(x[d], f, on);
          ln = fmaf(x[kAttnHD + 1], f, ln);
        }
        float* dst = p.partial + (((size_t(b) * p.kv_heads + p.kv_head) * p.n_splits + sp) * G + h) * (kAttnHD + 4);
        dst[d] = on;
        if (d == 0) { dst[kAttnHD] = M; dst[kAttnHD + 1] = ln; }
      }
    }
    bar_sync(1, kCons);              // xch / q staging reusable by the next pass
    if (trace) {
      phase_rec(a, 2, i0, ph0, ph1);     // prologue (q norm + rope)
      phase_rec(a, 3, i0, ph1, ph2);     // waiting for the K/V slots
      phase_rec(a, 4, i0, ph2, ph3);     // new token + QK / softmax / PV
      phase_rec(a, 5, i0, ph3, globaltimer());   // merge + partial write
    }
  } else if (active && g < G) {
    float* dst = p.partial + (((size_t(b) * p.kv_heads + p.kv_head) * p.n_splits + sp) * G + g) * (kAttnHD + 4);
#pragma unroll
    for (int u = 0; u < 16; ++u)
      *reinterpret_cast<float2*>(dst + 8 * u + 2 * c) = make_float2(o[u][0], o[u][1]);
    if (c == 0) { dst[kAttnHD] = m_run; dst[kAttnHD + 1] = l_run; }
  }
}

// Merge every split partial of row b (this kv head's G query heads) into
// the attention output -- run by the warp whose split arrived last (the
// ATTN_REDUCE stage folded into ATTN_PARTIAL).  Lane l owns dims 4l..4l+3.
__device__ void attn_merge_row(const mk_attn_params& p, int b, int nsp, int lane) {
  const int G = p.group;
  const int stride = G * (kAttnHD + 4);
  const float* base = p.partial + (size_t(b) * p.kv_heads + p.kv_head) * p.n_splits * stride;
  uint16_t* out = reinterpret_cast<uint16_t*>(p.out);
  constexpr int kB = 8;
  for (int h = 0; h < G; ++h) {
    const float* hb = base + h * (kAttnHD + 4);
    float M = -INFINITY, den = 0.f;
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < nsp; s0 += kB) {
      float mv[kB], lv[kB];
      float4 ov[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const bool ok = s0 + u < nsp;
        const float* x = hb + size_t(s0 + u) * stride;
        mv[u] = ok ? __ldcg(x + kAttnHD) : -INFINITY;
        lv[u] = ok ? __ldcg(x + kAttnHD + 1) : 0.f;
        ov[u] = ok ? __ldcg(reinterpret_cast<const float4*>(x + 4 * lane)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float bm = M;
#pragma unroll
      for (int u = 0; u < kB; ++u) bm = fmaxf(bm, mv[u]);
      const float corr = M == -INFINITY ? 0.f : ex2(M - bm);
      den *= corr; num.x *= corr; num.y *= corr; num.z *= corr; num.w *= corr;
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const float w = mv[u] == -INFINITY ? 0.f : ex2(mv[u] - bm);
        den = fmaf(w, lv[u], den);
        num.x = fmaf(w, ov[u].x, num.x); num.y = fmaf(w, ov[u].y, num.y);
        num.z = fmaf(w, ov[u].z, num.z); num.w = fmaf(w, ov[u].w, num.w);
      }
      M = bm;
    }
    const float inv = 1.f / den;
    uint2 o2;
    o2.x = pack_bf16(num.x * inv, num.y * inv);
    o2.y = pack_bf16(num.z * inv, num.w * inv);
    *reinterpret_cast<uint2*>(out + size_t(b) * p.q_heads * kAttnHD + (p.kv_head * G + h) * kAttnHD + 4 * lane) = o2;
  }
}

// One split of row b is done (its partial written, or it has no tokens):
// count it; the warp completing the row's n_splits arrivals merges.
__device__ __forceinline__ void attn_split_arrive(const KArgs& a, const mk_attn_params& p, int b, int pos,
                                                  int lane) {
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    const uint32_t old = atom_acq_rel_add(&a.sub_ctr[p.red_ctr0 + b], 1u);
    last = (old + 1 == uint32_t(p.n_splits) * a.epoch) ? 1 : 0;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  attn_merge_row(p, b, pos / kAttnSplit + 1, lane);
}

// Barrier-free variant (one warp per item, wpi = 1): warp w takes the unit's
// items w, w + 8, ...; each warp waits only for its own item's K/V slots
// (tag-checked: it may run more than a ring lap ahead), releases them with
// all 8 arrivals as soon as it is done and writes its split partial -- no
// pass barrier, no cross-warp merge, the fetch warp streams continuously.
__device__ void attn_mma_free(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                              const mk_attn_params& p, int ib, int ie, int ct) {
  const int G = p.group;
  const int warp = ct >> 5, lane = ct & 31;
  const int g = lane >> 2, c = lane & 3;
  const uint32_t base = r.k;
  uint32_t act = 0;                          // active items before the current one
  int last_b = -1, pos = 0;
  const bool trace = a.log != nullptr && lane == 0 && warp == 0;
  // q_norm + RoPE of every row of the unit once (each row's q is shared by
  // all its splits): the per-item path then starts from shared memory
  // instead of an L2 round trip per item
  AttnMmaScratch& sc = *reinterpret_cast<AttnMmaScratch*>(s.u.xs);
  const int r0 = ib < ie ? ib / p.n_splits : 0;
  int nq = ib < ie ? min(kQRows, (ie - 1) / p.n_splits - r0 + 1) : 0;
  if (ie - ib > kConsWarps) {                // worth it: more items than warps
    const int dl = lane & 15, half = lane >> 4;
    for (int task = warp; task < nq * ((G + 1) / 2); task += kConsWarps) {
      const int rr = task / ((G + 1) / 2), h = 2 * (task % ((G + 1) / 2)) + half;
      const int bq = r0 + rr;
      int pq = row_pos(p.positions, bq);
      if (pq < 0 || pq >= p.t_max) pq = 0;     // reported by the item loop (pos_ok)
      if (h < G) {
        float qv[8];
        norm_rope8<kAttnHD>(reinterpret_cast<const uint16_t*>(p.qkv) + size_t(bq) * p.ldqkv +
                                (p.kv_head * G + h) * kAttnHD,
                            reinterpret_cast<const uint16_t*>(p.q_gamma), p.eps,
                            p.rope_cos + size_t(pq) * (kAttnHD / 2),
                            p.rope_sin + size_t(pq) * (kAttnHD / 2), dl, qv);
        uint4 pk;
        pk.x = pack_bf16(qv[0], qv[1]); pk.y = pack_bf16(qv[2], qv[3]);
        pk.z = pack_bf16(qv[4], qv[5]); pk.w = pack_bf16(qv[6], qv[7]);
        *reinterpret_cast<uint4*>(&sc.qrow[rr][h][dl * 8]) = pk;
      }
    }
    bar_sync(1, kCons);
  } else {
    nq = 0;
  }
  if (p.prefill && ib < ie) {
    // chunked prefill: k_norm + RoPE and v of every chunk row (this kv head)
    // into shared memory once per unit; items fold them into their slots
    const int dl = lane & 15, half = lane >> 4;
    for (int rr = warp; rr < p.M && rr < kChunkRows; rr += kConsWarps) {
      int pq = row_pos(p.positions, rr);
      if (pq < 0 || pq >= p.t_max) pq = 0;
      const uint16_t* row = reinterpret_cast<const uint16_t*>(p.qkv) + size_t(rr) * p.ldqkv;
      float kn[8];                 // both half-warps (norm_rope8 shuffles within halves)
      norm_rope8<kAttnHD>(row + p.q_heads * kAttnHD + p.kv_head * kAttnHD,
                          reinterpret_cast<const uint16_t*>(p.k_gamma), p.eps,
                          p.rope_cos + size_t(pq) * (kAttnHD / 2),
                          p.rope_sin + size_t(pq) * (kAttnHD / 2), dl, kn);
      if (half == 0) {
        uint4 k4;
        k4.x = pack_bf16(kn[0], kn[1]); k4.y = pack_bf16(kn[2], kn[3]);
        k4.z = pack_bf16(kn[4], kn[5]); k4.w = pack_bf16(kn[6], kn[7]);
        *reinterpret_cast<uint4*>(&sc.ch.k[rr][dl * 8]) = k4;
      } else {
        *reinterpret_cast<uint4*>(&sc.ch.v[rr][dl * 8]) =
            ldg128_cg(row + (p.q_heads + p.kv_heads) * kAttnHD + p.kv_head * kAttnHD + dl * 8);
      }
    }
    bar_sync(1, kCons);
  }
  for (int it = ib; it < ie; ++it) {
    const int b = it / p.n_splits, sp = it % p.n_splits;
    if (b != last_b) {
      pos = row_pos(p.positions, b); last_b = b;
      if (!pos_ok(a, pos, p.t_max, b)) pos = p.t_max - 1;   // garbage, but in bounds
    }
    const int t0 = sp * kAttnSplit;
    const bool mine = ((it - ib) & (kConsWarps - 1)) == warp;
    if (t0 > pos) {                        // no tokens: only the fused-merge arrival
      if (mine && p.fuse_reduce) attn_split_arrive(a, p, b, pos, lane);
      continue;
    }
    const uint32_t kpos = base + 2 * act;
    ++act;
    if (!mine) continue;
    uint64_t ph0 = trace ? globaltimer() : 0, ph1 = ph0, ph2 = ph0;
    float m_run = -INFINITY, l_run = 0.f;
    float o[16][4];
#pragma unroll
    for (int u = 0; u < 16; ++u) o[u][0] = o[u][1] = o[u][2] = o[u][3] = 0.f;
    const int nvalid = min(kAttnSplit, pos + 1 - t0);
    const bool stamp = a.trace != nullptr && ct == 0 && s.tr[3] == 0;
    attn_mma_tokens(a, s, ring, p, b, pos, t0, nvalid, 0, kAttnSplit, kpos, true, warp, lane,
                    o, m_run, l_run, trace || stamp, ph1, ph2,
                    b - r0 < nq ? &sc.qrow[b - r0][0][0] : nullptr);
    if (stamp) { s.tr[7] = ph1; s.tr[3] = ph2; }   // q norm+RoPE done / K,V slots ready
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_cnt(&s.empty[kpos % kSlots], kConsWarps);
      mbar_arrive_cnt(&s.empty[(kpos + 1) % kSlots], kConsWarps);
    }
    if (g < G) {
      float* dst = p.partial + (((size_t(b) * p.kv_heads + p.kv_head) * p.n_splits + sp) * G + g) * (kAttnHD + 4);
#pragma unroll
      for (int u = 0; u < 16; ++u)
        *reinterpret_cast<float2*>(dst + 8 * u + 2 * c) = make_float2(o[u][0], o[u][1]);
      if (c == 0) { dst[kAttnHD] = m_run; dst[kAttnHD + 1] = l_run; }
    }
    if (p.fuse_reduce) attn_split_arrive(a, p, b, pos, lane);
    if (trace) {
      const uint64_t ph3 = globaltimer();
      phase_rec(a, 2, it, ph0, ph1);
      phase_rec(a, 3, it, ph1, ph2);
      phase_rec(a, 4, it, ph2, ph3);
    }
  }
  r.k = base + 2 * act;
}

template <int F>
__device__ void run_attn_partial(const KArgs& a, Smem& s, uint8_t* ring, Ring& r,
                                 const mk_task& t, int ib, int ie, int ct) {
  const mk_attn_params& p = *P<mk_attn_params>(a, t);
  if constexpr ((F & kFeatLean) != 0) {    // lean: the one-warp-per-item tensor-core path
    if (attn_mma_path(p) && p.sub_splits == 1) attn_mma_free(a, s, ring, r, p, ib, ie, ct);
    else if (ct == 0) raise_error(a, MK_ERR_CONFIG, -301);
    return;
  }
  if (attn_mma_path(p)) {                                  // tensor-core path
    if (p.sub_splits == 1) { attn_mma_free(a, s, ring, r, p, ib, ie, ct); return; }
    const int per = kConsWarps / p.sub_splits;
    for (int i = ib; i < ie; i += per) attn_mma_pass(a, s, ring, r, p, i, min(ie, i + per), ct);
    return;
  }
  const int per = kConsWarps / (p.group * p.sub_splits);
  for (int i = ib; i < ie; i += per) {
    const int i1 = min(ie, i + per);
    switch (p.head_dim) {
      case 128: attn_pass<128>(a, s, ring, r, p, i, i1, ct); break;
      case 64: attn_pass<64>(a, s, ring, r, p, i, i1, ct); break;
      case 32: attn_pass<32>(a, s, ring, r, p, i, i1, ct); break;
      default: attn_pass<16>(a, s, ring, r, p, i, i1, ct); break;
    }
  }
}

// Merge the split partials of one kv head for rows [ib, ie).  Thread
// (head, 4 dims) streams the splits in batches of 16 -- (m, l, o[4]) of a
// whole batch in flight -- and merges them online with a running max, so
// up to 16 splits cost one L2 round trip; no barrier.
__device__ void run_attn_reduce(const KArgs& a, Smem& s, const mk_task& t, int ib, int ie, int ct) {
  const mk_attn_params& p = *P<mk_attn_params>(a, t);
  if (p.fuse_reduce) return;             // merged by the last split (attn_split_arrive)
  const int HD = p.head_dim, G = p.group;
  const int stride = G * (HD + 4);          // floats per split
  uint16_t* out = reinterpret_cast<uint16_t*>(p.out);
  constexpr int kBatch = 20;
  // the unit's rows x (G heads x HD/4 dim quads) flattened over all consumer
  // threads: several rows merge in one round trip (G*HD/4 = 128 < kCons)
  const int per_row = G * HD / 4;
  const int n_work = (ie - ib) * per_row;
  for (int idx = ct; idx < n_work; idx += kCons) {
    const int b = ib + idx / per_row, e = idx % per_row;   // 4 dims per thread
    const int nv = min(row_pos(p.positions, b) / p.split + 1, p.n_splits);
    const float* base = p.partial + (size_t(b) * p.kv_heads + p.kv_head) * p.n_splits * stride;
    {
      const int hh = (e * 4) / HD, d = (e * 4) % HD;
      const float* hb = base + hh * (HD + 4);
      float M = -INFINITY, den = 0.f;
      float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < nv; s0 += kBatch) {
        float mv[kBatch], lv[kBatch];
        float4 ov[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const bool ok = s0 + u < nv;
          const float* x = hb + size_t(s0 + u) * stride;
          mv[u] = ok ? __ldcg(x + HD) : -INFINITY;
          lv[u] = ok ? __ldcg(x + HD + 1) : 0.f;
          ov[u] = ok ? __ldcg(reinterpret_cast<const float4*>(x + d)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float bm = M;
#pragma unroll
        for (int u = 0; u < kBatch; ++u) bm = fmaxf(bm, mv[u]);
        const float corr = M == -INFINITY ? 0.f : ex2(M - bm);
        den *= corr; num.x *= corr; num.y *= corr; num.z *= corr; num.w *= corr;
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const float w = mv[u] == -INFINITY ? 0.f : ex2(mv[u] - bm);
          den = fmaf(w, lv[u], den);
          num.x = fmaf(w, ov[u].x, num.x); num.y = fmaf(w, ov[u].y, num.y);
          num.z = fmaf(w, ov[u].z, num.z); num.w = fmaf(w, ov[u].w, num.w);
        }
        M = bm;
      }
      const float inv = 1.f / den;
      uint16_t o4[4] = {f2bf(num.x * inv), f2bf(num.y * inv), f2bf(num.z * inv), f2bf(num.w * inv)};
      *reinterpret_cast<uint2*>(out + size_t(b) * p.q_heads * HD + (p.kv_head * G + hh) * HD + d) =
          *reinterpret_cast<uint2*>(o4);
    }
  }
  (void)s;
}

__device__ void run_silu(const KArgs& a, const mk_task& t, int ct) {
  const mk_silu_params& p = *P<mk_silu_params>(a, t);
  const uint16_t* gu = reinterpret_cast<const uint16_t*>(p.gu);
  uint16_t* y = reinterpret_cast<uint16_t*>(p.y);
  for (int e = ct; e < p.rows * p.cols; e += kCons) {
    const int rr = p.row0 + e / p.cols, c = p.col0 + e % p.cols;
    const float g = bf2f(ldg16_cg(gu + size_t(rr) * 2 * p.F + c));
    const float u = bf2f(ldg16_cg(gu + size_t(rr) * 2 * p.F + p.F + c));
    y[size_t(rr) * p.F + c] = f2bf(g / (1.f + __expf(-g)) * u);
  }
}

__device__ void run_argmax(const KArgs& a, Smem& s, const mk_task& t, int ib, int ie, int ct) {
  const mk_argmax_params& p = *P<mk_argmax_params>(a, t);
  for (int b = ib; b < ie; ++b) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int q = ct; q < p.n_slots; q += kCons) {
      const float v = __ldcg(p.amax_val + size_t(q) * p.M + b);
      const int i = __ldcg(p.amax_idx + size_t(q) * p.M + b);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, off);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
    }
    if ((ct & 31) == 0) { s.bred[ct >> 5] = best; s.ibred[ct >> 5] = bi; }
    bar_sync(1, kCons);
    if (ct == 0) {
      for (int w = 1; w < kConsWarps; ++w) {
        const float v2 = s.bred[w];
        const int i2 = s.ibred[w];
        if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
      }
      p.out_tokens[b] = bi;
      p.next_tokens[b] = bi;
      p.positions[b] = p.positions[b] + 1;
    }
    bar_sync(1, kCons);
  }
}

// ---------------------------------------------------------------------------
// Tensor parallelism: the per-layer allreduce of the
// row-parallel o_proj / down partials and the vocab-parallel greedy token,
// as device tasks over peer memory.  The GEMMs (MK_EPI_PARTIAL) already
// pushed their fp32 partials into every rank's exchange region; these tasks
// only exchange epoch flags (st.release.sys / ld.acquire.sys, monotone: no
// reset between steps) and reduce LOCAL memory in rank order, so every rank
// computes bit-identical sums.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t* tp_flag(const KArgs& a, int q, int64_t flag_off, int slot) {
  return reinterpret_cast<uint32_t*>(a.tp_peer[q] + flag_off) + slot;
}

// ct 0: announce this rank at the point (to every rank), wait for all ranks
__device__ bool tp_rendezvous(const KArgs& a, int64_t flag_off, bool announce) {
  if (announce) {
    fence_sc_sys();
    for (int q = 0; q < a.tp_world; ++q) st_release_sys(tp_flag(a, q, flag_off, a.tp_rank), a.epoch);
  }
  for (int q = 0; q < a.tp_world; ++q) {
    const uint32_t* f = tp_flag(a, a.tp_rank, flag_off, q);
    Spin sp;
    while ((int32_t)(ld_acquire_sys(f) - a.epoch) < 0)
      if (!sp.ok(a, -19)) return false;
  }
  return true;
}

// units split the row's d/8 column chunks; items [ib, ie) of d/8
__device__ void run_tp_allreduce(const KArgs& a, Smem& s, const mk_task& t, int ib, int ie, int ct) {
  const mk_tp_params& p = *P<mk_tp_params>(a, t);
  if (ct == 0) tp_rendezvous(a, p.flag_off, ib == 0);
  bar_sync(1, kCons);
  const float* recv = reinterpret_cast<const float*>(a.tp_peer[a.tp_rank] + p.recv_off);
  const size_t plane = size_t(p.M) * p.d;
  const int n = (ie - ib) * p.M;
  for (int e = ct; e < n; e += kCons) {
    const int b = e / (ie - ib), c = (ib + e % (ie - ib)) * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int q = 0; q < a.tp_world; ++q) {         // rank order: identical on every rank
      const float* src = recv + q * plane + size_t(b) * p.d + c;
      const float4 u = __ldcg(reinterpret_cast<const float4*>(src));
      const float4 w = __ldcg(reinterpret_cast<const float4*>(src + 4));
      acc[0] += u.x; acc[1] += u.y; acc[2] += u.z; acc[3] += u.w;
      acc[4] += w.x; acc[5] += w.y; acc[6] += w.z; acc[7] += w.w;
    }
    float r[8];
    unpack8(ldg128_cg(reinterpret_cast<const uint16_t*>(p.res) + size_t(b) * p.d + c), r);
    uint16_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = f2bf(acc[k] + r[k]);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.y) + size_t(b) * p.d + c) =
        *reinterpret_cast<uint4*>(o);
  }
}

// one unit: the local shard's best (max logit, lowest global index) per row
// goes to every rank; every rank then picks the global best the same way
__device__ void run_tp_argmax(const KArgs& a, Smem& s, const mk_task& t, int ct) {
  const mk_tp_params& p = *P<mk_tp_params>(a, t);
  const int warp = ct >> 5, lane = ct & 31;
  for (int b = warp; b < p.M; b += kConsWarps) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int q = lane; q < p.n_slots; q += 32) {
      const float v = __ldcg(p.amax_val + size_t(q) * p.M + b);
      const int i = __ldcg(p.amax_idx + size_t(q) * p.M + b);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, off);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
    }
    if (lane == 0) {
      const int gi = bi == 0x7fffffff ? bi : bi + p.vocab0;
      for (int q = 0; q < a.tp_world; ++q) {
        int32_t* g = reinterpret_cast<int32_t*>(a.tp_peer[q] + p.gather_off) + 2 * (size_t(a.tp_rank) * p.M + b);
        __stcg(reinterpret_cast<float*>(g), best);
        __stcg(g + 1, gi);
      }
    }
  }
  __syncwarp();
  fence_sc_sys();                                  // every writer, before the announcement
  bar_sync(1, kCons);
  if (ct == 0) tp_rendezvous(a, p.flag_off, true);
  bar_sync(1, kCons);
  const int32_t* gat = reinterpret_cast<const int32_t*>(a.tp_peer[a.tp_rank] + p.gather_off);
  for (int b = ct; b < p.M; b += kCons) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int q = 0; q < a.tp_world; ++q) {
      const float v = __ldcg(reinterpret_cast<const float*>(gat + 2 * (size_t(q) * p.M + b)));
      const int i = __ldcg(gat + 2 * (size_t(q) * p.M + b) + 1);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
    p.out_tokens[b] = bi;
    p.next_tokens[b] = bi;
    p.positions[b] = p.positions[b] + 1;
  }
}

// ---------------------------------------------------------------------------
// Roles
// ---------------------------------------------------------------------------
__device__ void log_rec(const KArgs& a, int kind, int task, int ib, int worker, int die,
                        uint64_t t0, uint64_t t1) {
  unsigned long long at = atomicAdd(a.log_cursor, 1ull);
  if ((long long)at >= a.log_cap) return;
  mk_log_rec& r = a.log[at];
  r.kind = kind; r.task = task; r.item_begin = ib; r.worker = worker;
  r.smid = (int)smid(); r.die = die; r.t_start = t0; r.t_end = t1;
}

__device__ void scheduler(const KArgs& a, SchedSmem& s, int g) {
  const int lane = threadIdx.x & 31;
  const int W = a.W;
  const int gw0 = g * W;
  for (int w = lane; w < W; w += 32) {
    s.tail[w] = a.mb_tail[gw0 + w];
    s.head[w] = ld_acquire64(&a.mb_head[gw0 + w]);
  }
  __syncwarp();
  unsigned long long n_disp = 0, n_mail = 0;
  bool alive = true;
  auto push = [&](int w, uint32_t payload) -> bool {
    uint64_t t = s.tail[w];
    Spin sp;
    while (t - s.head[w] >= (uint64_t)kMailbox) {
      s.head[w] = ld_acquire64(&a.mb_head[gw0 + w]);
      if (!sp.ok(a, -4)) return false;
    }
    st_release64(&a.mailbox[size_t(gw0 + w) * kMailbox + t % kMailbox],
                 ((t + 1) << 24) | payload);
    s.tail[w] = t + 1;
    return true;
  };
  const int begin = a.sched_begin[g], end = a.sched_begin[g + 1];
  int rr = 0;
  int i = begin;
  const int batch = W < 32 ? W : 32;
  while (i < end && alive) {
    const mk_unit u = a.units[i];
    const mk_task& t = a.tasks[u.task];
    if (t.level == MK_LEVEL_CHIPLET) {
      uint64_t t0 = a.log ? globaltimer() : 0;
      for (int w = lane; w < W && alive; w += 32) alive = push(w, (uint32_t)i);
      alive = __all_sync(0xffffffffu, alive);
      if (lane == 0) {
        ++n_disp; n_mail += W;
        if (a.log) log_rec(a, 0, u.task, u.item_begin, -1 - g, g, t0, globaltimer());
      }
      ++i;
    } else {
      // a run of consecutive CU units, one per lane, distinct workers
      const int j = i + lane;
      bool cu = false;
      if (lane < batch && j < end) cu = a.tasks[a.units[j].task].level != MK_LEVEL_CHIPLET;
      const unsigned msk = __ballot_sync(0xffffffffu, !cu);
      const int run = msk ? (__ffs(msk) - 1) : 32;
      if (lane < run) {
        uint64_t t0 = a.log ? globaltimer() : 0;
        alive = push((rr + lane) % W, (uint32_t)j);
        if (a.log) log_rec(a, 0, a.units[j].task, a.units[j].item_begin, -1 - g, g, t0, globaltimer());
      }
      alive = __all_sync(0xffffffffu, alive);
      if (lane == 0) { n_disp += run; n_mail += run; }
      rr = (rr + run) % W;
      i += run;
    }
  }
  for (int w = lane; w < W && alive; w += 32) alive = push(w, kEnd);
  __syncwarp();
  for (int w = lane; w < W; w += 32) a.mb_tail[gw0 + w] = s.tail[w];
  if (lane == 0) {
    atomicAdd(&a.stats[S_DISPATCH], n_disp);
    atomicAdd(&a.stats[S_MAILBOX], n_mail);
  }
}

// Producer warpgroup, two single-lane roles that never wait on task
// dependencies (weights and past KV blocks are immutable during the step):
//  * mailbox warp (warp 1): scheduler mailbox -> unit queue tq;
//  * ring warp (warp 0): walks the queued units' slot streams and TMA-copies
//    each slot into the next free shared-memory ring slot.
// Splitting them keeps the mailbox's L2 round trips off the ring refill path.
__device__ void mailbox_warp(const KArgs& a, Smem& s, int g, int worker) {
  const int lane = threadIdx.x & 31;
  const int gw = g * a.W + worker;
  uint64_t head = a.mb_head[gw];
  for (uint32_t q = 0;; ++q) {
    const int qi = q % kTQ;
    uint32_t payload = kEnd;
    if (lane == 0) {
      const bool room = mbar_wait(a, &s.tq_empty[qi], ((q / kTQ) & 1) ^ 1, -6);
      uint64_t e = kEnd;
      if (room) {
        Spin sp;
        const uint64_t* slotp = &a.mailbox[size_t(gw) * kMailbox + head % kMailbox];
        // relaxed polling (ld.acquire would invalidate this SM's L1 on every
        // iteration, evicting the other roles' stack data) + one fence
        for (;;) {
          e = ld_relaxed64(slotp);
          if ((e >> 24) == head + 1) break;
          if (!sp.ok(a, -5)) { e = kEnd; break; }
          __nanosleep(64);
        }
        fence_acq_rel_gpu();
        if ((e >> 24) == head + 1) {
          ++head;
          st_release64(&a.mb_head[gw], head);
        }
      }
      payload = room ? uint32_t(e & 0xFFFFFFu) : kEnd;
    }
    payload = __shfl_sync(0xffffffffu, payload, 0);
    if (payload == kEnd) {
      if (lane == 0) {
        s.tq[qi] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&s.tq_full[qi]);
      }
      return;
    }
    // the unit's task descriptor (8 words) and parameter block (kPBytes)
    // into the descriptor cache, one 8-byte word per lane
    const mk_unit u = a.units[payload];
    const mk_task* gt = a.tasks + u.task;
    const uint64_t* src = lane < 8 ? reinterpret_cast<const uint64_t*>(gt) + lane
                                   : reinterpret_cast<const uint64_t*>(a.params + gt->param_off) + (lane - 8);
    const uint64_t v = *src;
    if (lane < 8) reinterpret_cast<uint64_t*>(&s.tcache[qi])[lane] = v;
    else s.pcache[qi][lane - 8] = v;
    __syncwarp();
    if (lane == 0) {
      mk_task& t = s.tcache[qi];
      t.pad[0] = t.wait0 >= 0 ? a.ev_req[t.wait0] : 0;
      t.pad[1] = t.wait1 >= 0 ? a.ev_req[t.wait1] : 0;
      t.pad[2] = t.wait0 >= 0 ? a.ev_dmask[t.wait0] : 0;
      t.pad[3] = t.wait1 >= 0 ? a.ev_dmask[t.wait1] : 0;
      s.tq[qi] = make_int4(u.task, u.item_begin, u.item_end, 0);
      mbar_arrive(&s.tq_full[qi]);
    }
  }
}

// L2 prefetch warp (warp 3 of the CUDA-core instance, where it is otherwise
// idle): walks the same slot sequence as the fetch warp over the units
// already queued in tq and issues cp.async.bulk.prefetch.L2 for up to
// pf_slots slots beyond the fetch warp's position -- the weights (immutable
// during the step) keep streaming from HBM while the ring is full and the
// die waits on a dependency (attention, norms, the next event).
template <int F>
__device__ void prefetch_warp(const KArgs& a, Smem& s, int worker) {
  if ((threadIdx.x & 31) != 0 || a.pf_slots <= 0) return;
  uint32_t my_pos = 0;
  for (uint32_t q = 0;; ++q) {
    const int qi = q % kTQ;
    {   // the unit is queued (no parity aliasing: q never passes the fill)
      Spin sp;
      bool ok = true;
      while (!mbar_test_wait(&s.tq_full[qi], (q / kTQ) & 1)) {
        if (!sp.ok(a, -16)) { ok = false; break; }
        __nanosleep(128);
      }
      if (!ok) return;
    }
    const int4 ent = s.tq[qi];
    if (ent.x < 0) return;
    SlotIter<F> it;
    it.init(a, s.tcache[qi], ent.y, ent.z, worker);
    const bool gemm = s.tcache[qi].op == MK_OP_GEMM;
    const void* src;
    uint32_t bytes;
    while (it.next(a, src, bytes)) {
      Spin sp;
      while (int32_t(my_pos - *reinterpret_cast<volatile uint32_t*>(&s.ring_pos)) >= a.pf_slots) {
        if (!sp.ok(a, -16)) return;
        __nanosleep(64);
      }
      if (gemm && int32_t(my_pos - *reinterpret_cast<volatile uint32_t*>(&s.ring_pos)) >= kSlots)
        prefetch_l2(src, bytes);          // slots inside the ring window are being copied anyway
      ++my_pos;
    }
  }
}

template <int F>
__device__ void ring_warp(const KArgs& a, Smem& s, uint8_t* ring, int worker) {
  if ((threadIdx.x & 31) != 0) return;
  const uint64_t pol = policy_evict_first();
  int si = 0;                       // ring slot index / phase
  uint32_t sph = 0;
  uint32_t pos_k = 0;               // ring position (= the consumers' Ring::k)
  unsigned long long w_empty = 0;
  struct Flush {
    const KArgs& a; unsigned long long& e;
    __device__ ~Flush() { if (a.debug & 4) atomicAdd(&a.stats[S_W_RING_EMPTY], e); }
  } flush{a, w_empty};
  for (uint32_t q = 0;; ++q) {
    const int qi = q % kTQ;
    if (!mbar_wait(a, &s.tq_full[qi], (q / kTQ) & 1, -8)) return;
    const int4 ent = s.tq[qi];
    if (ent.x < 0) return;
    SlotIter<F> it;
    it.init(a, s.tcache[qi], ent.y, ent.z, worker);
    const void* src;
    uint32_t bytes;
    while (it.next(a, src, bytes)) {
      if (!mbar_wait_p(a, &s.empty[si], sph ^ 1, -2, w_empty)) return;
      *reinterpret_cast<volatile uint32_t*>(&s.slot_tag[si]) = pos_k++;
      *reinterpret_cast<volatile uint32_t*>(&s.ring_pos) = pos_k;
      if (a.debug & 2) {
        mbar_arrive(&s.full[si]);
      } else {
        mbar_arrive_expect_tx(&s.full[si], bytes);
        bulk_g2s(ring + size_t(si) * kSlotBytes, src, bytes, &s.full[si], pol);
      }
      if (++si == kSlots) { si = 0; sph ^= 1; }
    }
  }
}

template <int F>
__device__ void consumers(const KArgs& a, Smem& s, uint8_t* ring, int g, int worker) {
  const int ct = threadIdx.x - kProdThreads;
  const int gw = g * a.W + worker;
  Ring r;
  uint32_t q = 0;
  unsigned long long n_glob = 0, n_loc = 0, n_fence = 0, n_fan = 0, n_poll = 0, n_tiles = 0,
                     n_exec = 0;
  uint64_t t_start = 0;
  uint32_t xs_k = 0, tb_k = 0;      // tcgen05 path: x-ring / accumulator-buffer counters
  uint32_t xs_ph = 0;               // hoisted x staging: xs_bar phases used (consumer 0)
  for (;;) {
    const int qi = q % kTQ;
    // thread 0 takes the next unit and resolves its dependencies; the
    // decision is broadcast through shared memory so that all consumer
    // threads follow the same control flow (no divergent named barriers)
    if (ct == 0) {
      int4 ent = make_int4(-1, 0, 0, 0);
      if (mbar_wait(a, &s.tq_full[qi], (q / kTQ) & 1, -7)) ent = s.tq[qi];
      int hoist = 0;
      uint32_t xb = 0;
      const void* xsrc = nullptr;
      if (ent.x >= 0) {
        const mk_task& t = s.tcache[qi];
        const int waits[2] = {t.wait0, t.wait1};
        uint32_t polls = 0;
        if (t.op == MK_OP_GEMM) {
          // a CUDA-core GEMM that stages its x rows: one m-tile of
          // contiguous rows (+ the norm gamma) fits u.xs -> bulk-copy them
          // into shared memory as soon as the dependency resolves (gamma,
          // static, already now); the copy overlaps the op's code fetch
          const mk_gemm_params& gp = *P<mk_gemm_params>(a, t);
          if (gp.stage_x && gp.body != MK_BODY_UMMA && gp.M <= gp.T_M && gp.ldx == gp.K) {
            xb = uint32_t(gp.M) * uint32_t(gp.K) * 2u;
            const uint32_t gb = gp.norm_gamma ? uint32_t(gp.K) * 2u : 0u;
            if (xb + gb <= uint32_t(kXsBytes) && (xb & 15u) == 0 && (gb & 15u) == 0) {
              hoist = 1;
              xsrc = gp.x;
              if (gb) {
                mbar_expect_tx(&s.xs_bar, gb);
                bulk_g2s(reinterpret_cast<uint8_t*>(s.u.xs) + xb, gp.norm_gamma, gb, &s.xs_bar,
                         policy_evict_last());
              }
            }
          }
        }
        if (a.trace) {
#pragma unroll
          for (int i = 0; i < 8; ++i) s.tr[i] = 0;
          s.tr[1] = globaltimer();
        }
        if constexpr ((F & kFeatUmma) != 0) {
          // tcgen05 GEMM: hand the job to the x-load / MMA warps BEFORE the
          // dependency resolves; the x-load warp acquires the input event
          // itself and issues the activation TMA at once, so the first MMA
          // is not serialised behind this role's acquire + code fetch
          // (the previous job was consumed: its accumulator was drained)
          if (t.op == MK_OP_GEMM && P<mk_gemm_params>(a, t)->body == MK_BODY_UMMA) {
            s.job = make_int4(ent.x, t.level == MK_LEVEL_CHIPLET ? worker : 0, int(r.k), qi);
            mbar_arrive(&s.job_full);
          }
        }
        for (int k = 0; k < 2; ++k) {
          const int e = waits[k];
          if (e < 0) continue;
          Spin sp;
          for (;;) {
            ++polls;
            if (ev_done<true>(a, e, t.pad[k], t.pad[2 + k])) break;
            if (!sp.ok(a, e)) break;
          }
        }
        n_poll += polls;
        if (a.log) t_start = globaltimer();
        if (a.trace) s.tr[2] = globaltimer();
        if (hoist) {
          fence_proxy_async_global();     // generic-proxy writes of x -> TMA reads
          mbar_arrive_expect_tx(&s.xs_bar, xb);
          bulk_g2s_plain(s.u.xs, xsrc, xb, &s.xs_bar);
        }
      }
      s.xs_hoist = hoist;
      s.xs_parity = xs_ph & 1u;
      xs_ph += uint32_t(hoist);
      s.cur = ent;
      s.abort_flag = aborted(a) ? 1 : 0;
    }
    bar_sync(1, kCons);
    const int4 ent = s.cur;
    if (ent.x < 0 || s.abort_flag) break;
    MK_TRACE(a, s, ct, 6);
    const mk_task& t = s.tcache[qi];
    switch (t.op) {
      case MK_OP_GEMM:
        if constexpr ((F & kFeatUmma) != 0) {
          if (P<mk_gemm_params>(a, t)->body == MK_BODY_UMMA) {
            run_gemm_umma(a, s, r, t, ent.x, worker, ct, xs_k, tb_k, n_tiles);
            break;
          }
        }
        run_gemm<F>(a, s, ring, r, t, worker, gw, ent.x, ct, n_tiles);
        break;
      case MK_OP_RMSNORM: run_rmsnorm(a, s, t, ent.y, ent.z, ct); break;
      case MK_OP_ATTN_PARTIAL: run_attn_partial<F>(a, s, ring, r, t, ent.y, ent.z, ct); break;
      case MK_OP_ATTN_REDUCE: run_attn_reduce(a, s, t, ent.y, ent.z, ct); break;
      case MK_OP_SILU: run_silu(a, t, ct); break;
      case MK_OP_ARGMAX: run_argmax(a, s, t, ent.y, ent.z, ct); break;
      case MK_OP_TP_ALLREDUCE: run_tp_allreduce(a, s, t, ent.y, ent.z, ct); break;
      case MK_OP_TP_ARGMAX: run_tp_argmax(a, s, t, ct); break;
      default: break;
    }
    MK_TRACE(a, s, ct, 4);
    if (t.op == MK_OP_GEMM && a.tp_world > 1 && P<mk_gemm_params>(a, t)->epilogue == MK_EPI_PARTIAL)
      fence_sc_sys();                   // pushed partials performed before the local signal
    bar_sync(1, kCons);
    if (ct == 0) {
      if (a.trace) s.tr[5] = globaltimer();
      const uint64_t t_done = a.log ? globaltimer() : 0;   // work done (before publishing)
      ++n_exec;
      if (t.signal >= 0) {
        if (t.level == MK_LEVEL_CHIPLET) {
          const uint32_t old = atom_acq_rel_add(&a.die_ctr[size_t(t.signal) * a.n_sched + g], 1u);
          ++n_loc;
          if (old + 1 == uint32_t(a.W) * a.epoch) {
            fence_acq_rel_gpu();
            ++n_fence;
            red_release_add(&a.ev_ctr[t.signal], 1u);
            ++n_glob;
          }
        } else if (t.n_units > 1) {
          const uint32_t old = atom_acq_rel_add(&a.sub_ctr[t.sub_ctr], 1u);
          ++n_fan;
          if (old + 1 == uint32_t(t.n_units) * a.epoch) {
            red_release_add(&a.ev_ctr[t.signal], 1u);
            ++n_glob;
          }
        } else {
          red_release_add(&a.ev_ctr[t.signal], 1u);
          ++n_glob;
        }
      }
      if (a.log) log_rec(a, 1, ent.x, ent.y, gw, g, t_start, t_done);
      if (a.trace && n_exec <= (unsigned long long)a.trace_cap) {
        uint64_t* rec = a.trace + (size_t(gw) * a.trace_cap + (n_exec - 1)) * 8;
        rec[0] = uint64_t(uint32_t(ent.x)) | (uint64_t(uint32_t(ent.y)) << 32);
#pragma unroll
        for (int i = 1; i < 6; ++i) rec[i] = s.tr[i];
        rec[6] = globaltimer();
        // n_exec | sub-phase stamps as ns after the acquire (0: not reached)
        const uint64_t d6 = s.tr[6] ? min(s.tr[6] - s.tr[2], uint64_t(0x3FFFFF)) : 0;
        const uint64_t d7 = s.tr[7] ? min(s.tr[7] - s.tr[2], uint64_t(0x3FFFFF)) : 0;
        rec[7] = (n_exec & 0xFFFFF) | (d6 << 20) | (d7 << 42);
      }
      mbar_arrive(&s.tq_empty[qi]);
    }
    ++q;
  }
  if (ct == 0 && a.use_umma) {     // release the MMA warp
    s.job = make_int4(-1, 0, 0, 0);
    mbar_arrive(&s.job_full);
  }
  if (ct == 0) {
    atomicAdd(&a.stats[S_GLOBAL], n_glob);
    atomicAdd(&a.stats[S_LOCAL], n_loc);
    atomicAdd(&a.stats[S_FENCE], n_fence);
    atomicAdd(&a.stats[S_FANOUT], n_fan);
    atomicAdd(&a.stats[S_POLL], n_poll);
    atomicAdd(&a.stats[S_TILES], n_tiles);
    atomicAdd(&a.stats[S_EXEC], n_exec);
  }
}

}  // namespace

template <int F>
__global__ void __launch_bounds__(kThreads, 1) megakernel(const __grid_constant__ KArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  uint8_t* ring = smem_raw + kRingOffset;
  __shared__ int role[2];
  if (threadIdx.x == 0) {
    const int die = a.die_of_sm[smid()];
    const int g = a.sched_mode == MK_SCHED_FLAT ? 0 : die;
    const uint32_t raw = atomicAdd(&a.role_ctr[g], 1u);
    const int rank = int(raw - (a.epoch - 1) * uint32_t(a.group_size[g]));
    role[0] = g;
    role[1] = rank;
    for (int i = 0; i < kSlots; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], kConsWarps); s.slot_tag[i] = 0xffffffffu; }
    s.ring_pos = 0;
    for (int i = 0; i < kTQ; ++i) { mbar_init(&s.tq_full[i], 1); mbar_init(&s.tq_empty[i], 1); }
    for (int i = 0; i < kXStagesMax; ++i) { mbar_init(&s.xfull[i], 1); mbar_init(&s.xempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s.tile_done[i], 1); mbar_init(&s.tmem_free[i], kConsWarps); }
    mbar_init(&s.job_full, 1);
    mbar_init(&s.xs_bar, 1);
    fence_mbar_init();
    if (blockIdx.x == 0) atomicAdd(&a.stats[S_STEPS], 1ull);
  }
  for (int i = threadIdx.x; i < a.n_rows && i < kPosRows; i += blockDim.x) s.pos[i] = a.positions[i];
  if (threadIdx.x == 0) s.n_pos = a.positions ? min(a.n_rows, kPosRows) : 0;
  __syncthreads();
  const int g = role[0], rank = role[1];
  if (g >= a.n_sched) return;
  if (rank < 0 || rank >= a.group_size[g]) {   // role counters out of step with the epoch
    if (threadIdx.x == 0) raise_error(a, MK_ERR_CONFIG, -200);
    return;
  }
  if (rank == 0) {
    if (threadIdx.x < 32) scheduler(a, *reinterpret_cast<SchedSmem*>(ring), g);
    return;
  }
  const int worker = rank - 1;
  if (worker >= a.W) return;             // extra SMs of the larger die idle
  if ((F & kFeatUmma) && a.use_umma) {   // TMEM for the tcgen05 accumulators
    if ((threadIdx.x >> 5) == 2) {
      tmem_alloc(&s.tmem_base, kTmemCols);
      tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  // warp specialisation with register reallocation: the producer warpgroup
  // drops to kProdRegs, the two consumer warpgroups grow to kConsRegs
  if (threadIdx.x < kProdThreads) {
    // the tcgen05 instance gives the producer roles (fetch warp, MMA lane:
    // iterator state) more registers than the CUDA-core instance
    if constexpr ((F & kFeatUmma) != 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(kProdRegsUmma));
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(kProdRegs));
    if (threadIdx.x < 32) ring_warp<F>(a, s, ring, worker);
    else if (threadIdx.x < 64) mailbox_warp(a, s, g, worker);
    else if (threadIdx.x < 96 && a.use_umma) {
      if constexpr ((F & kFeatUmma) != 0) {
        mma_warp(a, s, ring);
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(s.tmem_base, kTmemCols);
      }
    } else if (a.use_umma) {
      if constexpr ((F & kFeatUmma) != 0) xload_warp(a, s);
    } else if (threadIdx.x >= 96) {
      if constexpr ((F & kFeatUmma) == 0) prefetch_warp<F>(a, s, worker);
    }
  } else {
    if constexpr ((F & kFeatUmma) != 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(kConsRegsUmma));
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(kConsRegs));
    consumers<F>(a, s, ring, g, worker);
  }
}

#else
template <int F>
__global__ void __launch_bounds__(kThreads, 1) megakernel(const __grid_constant__ KArgs a);
#endif  // MK_HOST_TU

#ifdef MK_HOST_TU   // the die probe lives with the host ABI

// ---------------------------------------------------------------------------
// Die probe: per-SM L2 hit latency to lines spread over the address space.
// ---------------------------------------------------------------------------
__global__ void probe_init(uint32_t* buf, int n_lines, int stride_words) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_lines; i += gridDim.x * blockDim.x)
    buf[size_t(i) * stride_words] = uint32_t(i) * uint32_t(stride_words);   // self-pointer
}

// Each CTA (one per SM) times a dependent chain of .cg loads (L2 hits) on
// every probe line; the clock is read behind a branch on the last loaded
// value so it cannot issue before the chain completes.
__global__ void __launch_bounds__(32, 1) probe_kernel(const uint32_t* buf, int n_lines, int stride_words,
                                                      int reps, uint32_t* lat, int* smid_of_block) {
  extern __shared__ uint8_t pad_smem[];
  if (threadIdx.x != 0) return;
  pad_smem[0] = 0;
  const uint32_t sm = smid();
  smid_of_block[blockIdx.x] = int(sm);
  constexpr int kChain = 16;
  for (int i = 0; i < n_lines; ++i) {
    uint32_t best = 0xffffffffu;
    uint32_t idx = uint32_t(i) * uint32_t(stride_words);
    for (int rep = 0; rep < reps; ++rep) {
      const long long t0 = clock64();
#pragma unroll
      for (int c = 0; c < kChain; ++c)
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(idx) : "l"(buf + idx) : "memory");
      if (idx == 0xffffffffu) smid_of_block[0] = -2;   // forces the chain to finish
      const long long t1 = clock64();
      if (rep > 0) best = min(best, uint32_t((t1 - t0) / kChain));
    }
    lat[size_t(sm) * n_lines + i] = best;
  }
}

#endif  // MK_HOST_TU
}  // namespace mk

#ifdef MK_INSTANCE
namespace mk {
template __global__ void __launch_bounds__(kThreads, 1) megakernel<MK_INSTANCE>(const __grid_constant__ KArgs a);
}  // namespace mk
#else  // host ABI
// ===========================================================================
// Host side: C ABI
// ===========================================================================
using namespace mk;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(MK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct mk_handle {
  int use_dmask = 1;             // waiters of die-task events poll die counters (MK_EV_DMASK=0: off)
  int device = 0;
  int num_sms = 0;
  int sched_mode = 0;
  int n_sched = 0;
  int W = 0;
  int n_events = 0, n_tasks = 0, n_units = 0, n_sub = 0;
  uint32_t epoch = 0;
  double watchdog_s = 5.0;
  int debug = 0;
  int use_umma = 0;
  int feat = 0;                 // kFeat* bits of the graph -> kernel instance
  const void* kernel = nullptr;
  CUtensorMap* d_tmaps = nullptr; // x tensor map per task (tcgen05 GEMMs)
  int x_stages = 1, x_stage_bytes = 2048;
  int pf_slots = 0;             // L2 prefetch run-ahead per worker (mk_set_prefetch)
  uint64_t* d_trace = nullptr;  // per-unit phase stamps (mk_trace_enable)
  const int32_t* positions = nullptr;  // borrowed: decode position per row
  int n_rows = 0;
  int trace_cap = 0;
  // device buffers
  mk_task* d_tasks = nullptr;
  mk_unit* d_units = nullptr;
  int32_t* d_sched_begin = nullptr;
  uint8_t* d_params = nullptr;
  uint32_t* d_ev_ctr = nullptr;
  int32_t* d_ev_req = nullptr;
  int32_t* d_ev_dmask = nullptr;
  uint32_t* d_die_ctr = nullptr;
  uint32_t* d_sub_ctr = nullptr;
  uint64_t* d_mailbox = nullptr;
  uint64_t* d_mb_head = nullptr;
  uint64_t* d_mb_tail = nullptr;
  int8_t* d_die_of_sm = nullptr;
  uint32_t* d_role_ctr = nullptr;
  int32_t* d_group_size = nullptr;
  unsigned long long* d_stats = nullptr;
  int* d_err = nullptr;
  int* h_err = nullptr;   // pinned copy
  mk_log_rec* d_log = nullptr;
  unsigned long long* d_log_cursor = nullptr;
  long long log_cap = 0;
  int32_t* d_tile_log = nullptr;
  unsigned long long* d_tile_cursor = nullptr;
  long long tile_cap = 0;
  std::vector<int32_t> group_size;
  int cooperative = 1;
  int tp_world = 1, tp_rank = 0;
  uint8_t* tp_peer[MK_MAX_TP] = {};
  bool has_tp_tasks = false;
  int32_t* tokens = nullptr;
  const int32_t* out_tokens = nullptr;
};

static const void* kernel_for(int feat) {
  // lean instances when the graph qualifies (kFeatLean), else the plain
  // CUDA-core graph's instance or the general one
  if (feat & kFeatLean)
    return (feat & kFeatUmma) ? (const void*)megakernel<kFeatLean | kFeatUmma | kFeatKsplit>
                              : (const void*)megakernel<kFeatLean | kFeatKsplit>;
  if ((feat & (kFeatUmma | kFeatKsplit)) == 0) return (const void*)megakernel<0>;
  return (const void*)megakernel<kFeatUmma | kFeatKsplit>;
}

template <typename T>
static int dalloc(T** p, size_t n) {
  CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)));
  return MK_OK;
}

extern "C" {

const char* mk_last_error(void) { return g_err.c_str(); }
int mk_version(void) { return 1; }

static int probe_raw(int device, std::vector<uint32_t>& h, std::vector<int>& sm_of, int& nsm,
                     int& n_lines) {
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  nsm = prop.multiProcessorCount;
  if (nsm > MK_MAX_SMS) return fail(MK_ERR_CONFIG, "too many SMs");
  n_lines = 512;
  const int stride_words = 1024 + 32, reps = 8;   // 4 KiB + 128 B apart
  uint32_t* buf = nullptr;
  uint32_t* lat = nullptr;
  int* smid_of_block = nullptr;
  CK(cudaMalloc(&buf, size_t(n_lines) * stride_words * 4));
  CK(cudaMemset(buf, 0, size_t(n_lines) * stride_words * 4));
  probe_init<<<4, 128>>>(buf, n_lines, stride_words);
  CK(cudaGetLastError());
  CK(cudaMalloc(&lat, size_t(MK_MAX_SMS) * n_lines * 4));
  CK(cudaMemset(lat, 0, size_t(MK_MAX_SMS) * n_lines * 4));
  CK(cudaMalloc(&smid_of_block, nsm * sizeof(int)));
  const int pad = 160 * 1024;   // one block per SM
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pad));
  probe_kernel<<<nsm, 32, pad>>>(buf, n_lines, stride_words, reps, lat, smid_of_block);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  h.assign(size_t(MK_MAX_SMS) * n_lines, 0);
  sm_of.assign(nsm, 0);
  CK(cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(sm_of.data(), smid_of_block, nsm * sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(buf); cudaFree(lat); cudaFree(smid_of_block);
  return MK_OK;
}

int mk_probe_raw(int device, uint32_t* lat_out, int32_t* n_lines_out) {
  std::vector<uint32_t> h;
  std::vector<int> sm_of;
  int nsm = 0, n_lines = 0;
  int rc = probe_raw(device, h, sm_of, nsm, n_lines);
  if (rc) return rc;
  if (lat_out) memcpy(lat_out, h.data(), h.size() * 4);
  if (n_lines_out) *n_lines_out = n_lines;
  return MK_OK;
}

int mk_probe(int device, mk_topology* out) {
  if (!out) return fail(MK_ERR_CONFIG, "null topology");
  std::vector<uint32_t> h;
  std::vector<int> sm_of;
  int nsm = 0, n_lines = 0;
  int rc = probe_raw(device, h, sm_of, nsm, n_lines);
  if (rc) return rc;
  // which smids exist
  std::vector<int> present(MK_MAX_SMS, 0);
  int max_sm = 0;
  for (int b = 0; b < nsm; ++b) { present[sm_of[b]] = 1; max_sm = std::max(max_sm, sm_of[b]); }
  std::vector<int> sms;
  for (int i = 0; i <= max_sm; ++i) if (present[i]) sms.push_back(i);
  // bit pattern: latency above the line's median across SMs
  std::vector<double> med(n_lines);
  for (int i = 0; i < n_lines; ++i) {
    std::vector<uint32_t> col;
    for (int sm : sms) col.push_back(h[size_t(sm) * n_lines + i]);
    std::nth_element(col.begin(), col.begin() + col.size() / 2, col.end());
    med[i] = col[col.size() / 2];
  }
  auto bits = [&](int sm, int i) { return double(h[size_t(sm) * n_lines + i]) > med[i] ? 1 : 0; };
  // 2-means on the bit vectors, seeded with the first SM
  std::vector<int> label(MK_MAX_SMS, -1);
  const int ref = sms[0];
  for (int sm : sms) {
    int d = 0;
    for (int i = 0; i < n_lines; ++i) d += bits(sm, i) != bits(ref, i);
    label[sm] = d * 2 > n_lines ? 1 : 0;
  }
  for (int iter = 0; iter < 4; ++iter) {
    std::vector<double> cen(2 * n_lines, 0.0);
    int cnt[2] = {0, 0};
    for (int sm : sms) {
      ++cnt[label[sm]];
      for (int i = 0; i < n_lines; ++i) cen[label[sm] * n_lines + i] += h[size_t(sm) * n_lines + i];
    }
    if (cnt[0] == 0 || cnt[1] == 0) break;
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < n_lines; ++i) cen[c * n_lines + i] /= cnt[c];
    for (int sm : sms) {
      double d0 = 0, d1 = 0;
      for (int i = 0; i < n_lines; ++i) {
        const double v = h[size_t(sm) * n_lines + i];
        d0 += (v - cen[i]) * (v - cen[i]);
        d1 += (v - cen[n_lines + i]) * (v - cen[n_lines + i]);
      }
      label[sm] = d1 < d0 ? 1 : 0;
    }
  }
  int cnt[2] = {0, 0};
  for (int sm : sms) ++cnt[label[sm]];
  // near/far latencies: a line's home die is the cluster that sees it faster
  double near_sum = 0, far_sum = 0;
  long near_n = 0, far_n = 0;
  double var = 0;
  if (cnt[0] > 0 && cnt[1] > 0) {
    for (int i = 0; i < n_lines; ++i) {
      double m[2] = {0, 0};
      for (int sm : sms) m[label[sm]] += h[size_t(sm) * n_lines + i];
      m[0] /= cnt[0]; m[1] /= cnt[1];
      const int home = m[0] <= m[1] ? 0 : 1;
      for (int sm : sms) {
        const double v = h[size_t(sm) * n_lines + i];
        if (label[sm] == home) { near_sum += v; ++near_n; } else { far_sum += v; ++far_n; }
        var += (v - m[label[sm]]) * (v - m[label[sm]]);
      }
    }
  }
  memset(out, 0, sizeof(*out));
  out->num_sms = nsm;
  for (int i = 0; i < MK_MAX_SMS; ++i) out->die_of_sm[i] = 0;
  const bool split_ok = cnt[0] > 0 && cnt[1] > 0 && near_n > 0 && far_n > 0;
  if (split_ok) {
    out->near_cycles = float(near_sum / near_n);
    out->far_cycles = float(far_sum / far_n);
    const double sd = std::sqrt(var / double(near_n + far_n)) + 1e-9;
    out->separation = float((out->far_cycles - out->near_cycles) / sd);
    out->num_dies = 2;
    // die 0 holds the lowest smid
    const int flip = label[sms[0]];
    for (int sm : sms) out->die_of_sm[sm] = label[sm] ^ flip;
    out->sms_per_die[0] = cnt[flip];
    out->sms_per_die[1] = cnt[flip ^ 1];
  } else {
    out->num_dies = 1;
    out->sms_per_die[0] = nsm;
    out->separation = 0.f;
  }
  return MK_OK;
}

static int validate_graph(const mk_graph_desc* g) {
  if (!g || !g->tasks || !g->event_required || !g->units || !g->sched_begin)
    return fail(MK_ERR_CONFIG, "null graph arrays");
  if (g->n_schedulers < 1 || g->workers_per_sched < 1)
    return fail(MK_ERR_CONFIG, "bad scheduler / worker count");
  if (g->sched_begin[0] != 0 || g->sched_begin[g->n_schedulers] != g->n_units)
    return fail(MK_ERR_CONFIG, "sched_begin does not cover the unit list");
  if (g->n_units >= int(kEnd)) return fail(MK_ERR_CONFIG, "too many units");
  for (int i = 0; i < g->n_tasks; ++i) {
    const mk_task& t = g->tasks[i];
    if (t.wait0 >= g->n_events || t.wait1 >= g->n_events || t.signal >= g->n_events)
      return fail(MK_ERR_CONFIG, "task " + std::to_string(i) + " references an unknown event");
    if (t.param_off < 0 || t.param_off % 8 || t.param_off > g->param_bytes)
      return fail(MK_ERR_CONFIG, "task " + std::to_string(i) + " has a bad param offset");
    if (t.level == MK_LEVEL_CHIPLET && (t.die < 0 || t.die >= g->n_schedulers))
      return fail(MK_ERR_CONFIG, "chiplet task " + std::to_string(i) + " has a bad die binding");
    if (t.n_units > 1 && (t.sub_ctr < 0 || t.sub_ctr >= g->n_sub_ctrs))
      return fail(MK_ERR_CONFIG, "task " + std::to_string(i) + " needs a sub-counter");
    if (t.op == MK_OP_GEMM) {
      const mk_gemm_params* p = reinterpret_cast<const mk_gemm_params*>(
          static_cast<const uint8_t*>(g->params) + t.param_off);
      if (p->ksplit) {
        const int R = p->T_N * (p->epilogue == MK_EPI_SILU ? 2 : 1);
        const long long tiles = (long long)((p->M + p->T_M - 1) / p->T_M) * (p->N / std::max(R, 1));
        const int need = p->body == MK_BODY_UMMA ? 128 * ((std::min(p->T_M, p->M) + 15) / 16 * 16)
                                                 : R * p->T_M;
        const int rows = std::min(p->T_M, p->M);
        const bool fast = (rows <= 1 && R == 8 && p->T_K == 1024) || (rows <= 4 && R == 16 && p->T_K == 512) ||
                          (rows <= 8 && R == 32 && p->T_K == 256);
        if (t.level != MK_LEVEL_CHIPLET || !p->kpart || p->piece_floats < need || p->tile_ctr0 < 0 ||
            p->tile_ctr0 + tiles > g->n_sub_ctrs || (p->body == MK_BODY_GEMV && !fast))
          return fail(MK_ERR_CONFIG, "k-split gemm task " + std::to_string(i) + " has bad piece/counter setup");
      }
      if (p->body == MK_BODY_UMMA) {
        const int R = p->T_N * (p->epilogue == MK_EPI_SILU ? 2 : 1);
        if (R != 128 || p->T_K != 64 || p->K % 64 || p->N % 128 || p->T_M > 64 || p->stage_x ||
            p->norm_gamma || (p->epilogue == MK_EPI_LOGITS && p->M > kAmaxRows) ||
            (p->ss_in && (p->ss_nparts < 1 || p->M > kAmaxRows)))
          return fail(MK_ERR_CONFIG, "umma gemm task " + std::to_string(i) + " has an unsupported tile");
        continue;
      }
      const int R = p->T_N * (p->epilogue == MK_EPI_SILU ? 2 : 1);
      const bool kc_ok = (p->T_K % 256 == 0) || (p->T_K == p->K && p->T_K % 8 == 0 && p->T_K < 256);
      if (!kc_ok || p->K % p->T_K || size_t(R) * p->T_K * 2 > size_t(kSlotBytes) ||
          R % kConsWarps || R > 4 * kConsWarps ||
          (p->epilogue == MK_EPI_SILU && (R / kConsWarps) % 2) ||
          p->N % R || p->T_M > kMaxNB || (p->epilogue == MK_EPI_LOGITS && p->M > kAmaxRows) ||
          (p->stage_x && size_t(std::min(p->T_M, p->M)) * p->K * 2 > size_t(kXsBytes)) ||
          (p->norm_gamma && (!p->stage_x || p->K > 6 * 2048)))
        return fail(MK_ERR_CONFIG, "gemm task " + std::to_string(i) + " has an unsupported tile (" +
                                       std::to_string(p->T_M) + "," + std::to_string(p->T_N) + "," +
                                       std::to_string(p->T_K) + ")");
    }
    if (t.op == MK_OP_ATTN_PARTIAL || t.op == MK_OP_ATTN_REDUCE) {
      const mk_attn_params* p = reinterpret_cast<const mk_attn_params*>(
          static_cast<const uint8_t*>(g->params) + t.param_off);
      const int hd = p->head_dim;
      const bool mma = attn_mma_path(*p);
      // tensor-core path: a pass's 2 * 8 / wpi K/V slots must fit the ring
      const bool ws_ok = mma ? (p->sub_splits == 1 ||   // barrier-free warps
                                ((p->sub_splits == 2 || p->sub_splits == 4) && 2 * (kConsWarps / p->sub_splits) <= kSlots))
                             : (p->group * p->sub_splits <= kConsWarps && kConsWarps % (p->group * p->sub_splits) == 0);
      if ((hd != 16 && hd != 32 && hd != 64 && hd != 128) || p->group < 1 || p->group > 8 ||
          8 % p->group || size_t(p->split) * hd * 2 > size_t(kSlotBytes) ||
          p->n_splits > kMaxSplits || p->sub_splits < 1 || !ws_ok || (mma && p->t_max % kAttnSplit) ||
          (p->page_table && p->max_pages * p->split != p->t_max) ||
          (p->prefill && (!mma || p->M > kChunkRows || p->sub_splits != 1)))
        return fail(MK_ERR_CONFIG, "attention task " + std::to_string(i) + " has unsupported shapes");
    }
  }
  for (int i = 0; i < g->n_tasks; ++i) {
    const mk_task& t = g->tasks[i];
    if (t.op == MK_OP_TP_ALLREDUCE || t.op == MK_OP_TP_ARGMAX) {
      const mk_tp_params* p = reinterpret_cast<const mk_tp_params*>(
          static_cast<const uint8_t*>(g->params) + t.param_off);
      if (t.level == MK_LEVEL_CHIPLET || p->flag_off < 0 || p->flag_off % 4 ||
          (t.op == MK_OP_TP_ALLREDUCE && (p->d % 8 || p->recv_off % 16 || !p->res || !p->y)) ||
          (t.op == MK_OP_TP_ARGMAX && (t.n_units != 1 || p->gather_off % 8)))
        return fail(MK_ERR_CONFIG, "tensor-parallel task " + std::to_string(i) + " has a bad setup");
    }
  }
  for (int u = 0; u < g->n_units; ++u)
    if (g->units[u].task < 0 || g->units[u].task >= g->n_tasks)
      return fail(MK_ERR_CONFIG, "unit " + std::to_string(u) + " references an unknown task");
  return MK_OK;
}

// Activation tensor maps of the tcgen05 GEMM tasks: x is bf16 [M][ldx]; one
// box = 64 K-elements x NT rows, 128B-swizzled (the UMMA K-major SW128
// operand layout), rows past M zero-filled.
static int build_tmaps(mk_handle* h, const mk_graph_desc* g) {
  std::vector<CUtensorMap> maps(std::max(1, g->n_tasks));
  memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
  int max_nt = 16;
  bool any = false;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  for (int i = 0; i < g->n_tasks; ++i) {
    const mk_task& t = g->tasks[i];
    if (t.op != MK_OP_GEMM) continue;
    const mk_gemm_params* p =
        reinterpret_cast<const mk_gemm_params*>(static_cast<const uint8_t*>(g->params) + t.param_off);
    if (p->body != MK_BODY_UMMA) continue;
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess) return fail(MK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const int nt = (std::min(p->T_M, p->M) + 15) / 16 * 16;
    max_nt = std::max(max_nt, nt);
    cuuint64_t dims[2] = {cuuint64_t(p->K), cuuint64_t(p->M)};
    cuuint64_t strides[1] = {cuuint64_t(p->ldx) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(nt)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p->x), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(MK_ERR_CONFIG, "task " + std::to_string(i) + ": x tensor map rejected (" + std::to_string(int(r)) + ")");
    any = true;
  }
  h->x_stage_bytes = max_nt * 128;
  int xs = 1;                                       // as many stages as fit
  // one stage holds the activation chunks of one MMA chunk pair
  xs = std::max(1, std::min(kXStagesMax, kXsBytes / (2 * h->x_stage_bytes)));
  h->x_stages = xs;
  if (any) {
    CK(cudaMalloc(&h->d_tmaps, maps.size() * sizeof(CUtensorMap)));
    CK(cudaMemcpy(h->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  }
  return MK_OK;
}

static int reset_state(mk_handle* h) {
  CK(cudaMemset(h->d_ev_ctr, 0, sizeof(uint32_t) * std::max(1, h->n_events)));
  CK(cudaMemset(h->d_die_ctr, 0, sizeof(uint32_t) * std::max(1, h->n_events * h->n_sched)));
  CK(cudaMemset(h->d_sub_ctr, 0, sizeof(uint32_t) * std::max(1, h->n_sub)));
  CK(cudaMemset(h->d_mailbox, 0, sizeof(uint64_t) * size_t(h->n_sched) * h->W * kMailbox));
  CK(cudaMemset(h->d_mb_head, 0, sizeof(uint64_t) * size_t(h->n_sched) * h->W));
  CK(cudaMemset(h->d_mb_tail, 0, sizeof(uint64_t) * size_t(h->n_sched) * h->W));
  CK(cudaMemset(h->d_role_ctr, 0, sizeof(uint32_t) * MK_MAX_DIES));
  CK(cudaMemset(h->d_err, 0, 2 * sizeof(int)));
  CK(cudaDeviceSynchronize());
  h->epoch = 0;
  return MK_OK;
}


int mk_create(int device, const mk_graph_desc* g, const mk_topology* topo, mk_handle** out) {
  if (!out || !topo) return fail(MK_ERR_CONFIG, "null argument");
  int rc = validate_graph(g);
  if (rc) return rc;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (topo->num_sms != prop.multiProcessorCount)
    return fail(MK_ERR_CONFIG, "topology was probed on a different device");
  mk_handle* h = new mk_handle();
  if (const char* ev = getenv("MK_EV_DMASK")) h->use_dmask = atoi(ev) != 0;
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  h->sched_mode = g->sched_mode;
  h->n_sched = g->n_schedulers;
  h->W = g->workers_per_sched;
  h->n_events = g->n_events;
  h->n_tasks = g->n_tasks;
  h->n_units = g->n_units;
  h->n_sub = g->n_sub_ctrs;
  h->positions = g->positions;
  h->tokens = g->tokens;
  h->out_tokens = g->out_tokens;
  h->n_rows = g->positions ? g->n_rows : 0;
  std::vector<int8_t> die_of_sm(MK_MAX_SMS, 0);
  h->group_size.assign(MK_MAX_DIES, 0);
  if (g->sched_mode == MK_SCHED_FLAT) {
    if (g->n_schedulers != 1) { delete h; return fail(MK_ERR_CONFIG, "flat mode has one scheduler"); }
    h->group_size[0] = h->num_sms;
    if (h->W > h->num_sms - 1) { delete h; return fail(MK_ERR_CONFIG, "more workers than SMs"); }
  } else {
    if (g->n_schedulers != topo->num_dies) {
      delete h;
      return fail(MK_ERR_CONFIG, "graph built for " + std::to_string(g->n_schedulers) +
                                     " dies, device has " + std::to_string(topo->num_dies));
    }
    for (int d = 0; d < topo->num_dies; ++d) {
      h->group_size[d] = topo->sms_per_die[d];
      if (h->W > topo->sms_per_die[d] - 1) {
        delete h;
        return fail(MK_ERR_CONFIG, "die " + std::to_string(d) + " has too few SMs for W");
      }
    }
    for (int i = 0; i < MK_MAX_SMS; ++i) die_of_sm[i] = int8_t(topo->die_of_sm[i]);
  }
#define DA(p, n) do { int r_ = dalloc(&p, n); if (r_) { delete h; return r_; } } while (0)
  DA(h->d_tasks, g->n_tasks);
  DA(h->d_units, g->n_units);
  DA(h->d_sched_begin, g->n_schedulers + 1);
  DA(h->d_params, g->param_bytes + kPBytes);   // the cache copy reads kPBytes per block
  DA(h->d_ev_ctr, g->n_events);
  DA(h->d_ev_req, g->n_events);
  DA(h->d_ev_dmask, g->n_events);
  DA(h->d_die_ctr, size_t(g->n_events) * g->n_schedulers);
  DA(h->d_sub_ctr, g->n_sub_ctrs);
  DA(h->d_mailbox, size_t(g->n_schedulers) * h->W * kMailbox);
  DA(h->d_mb_head, size_t(g->n_schedulers) * h->W);
  DA(h->d_mb_tail, size_t(g->n_schedulers) * h->W);
  DA(h->d_die_of_sm, MK_MAX_SMS);
  DA(h->d_role_ctr, MK_MAX_DIES);
  DA(h->d_group_size, MK_MAX_DIES);
  DA(h->d_stats, 32);
  DA(h->d_err, 2);
  DA(h->d_log_cursor, 1);
  DA(h->d_tile_cursor, 1);
#undef DA
  CK(cudaMallocHost(&h->h_err, 2 * sizeof(int)));
  CK(cudaMemcpy(h->d_tasks, g->tasks, sizeof(mk_task) * g->n_tasks, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_units, g->units, sizeof(mk_unit) * g->n_units, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_sched_begin, g->sched_begin, sizeof(int32_t) * (g->n_schedulers + 1),
                cudaMemcpyHostToDevice));
  CK(cudaMemset(h->d_params, 0, g->param_bytes + kPBytes));
  if (g->param_bytes)
    CK(cudaMemcpy(h->d_params, g->params, g->param_bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_ev_req, g->event_required, sizeof(int32_t) * g->n_events, cudaMemcpyHostToDevice));
  {
    // An event whose signallers are exactly one die task per scheduler group
    // completes when those groups' die counters reach W per launch: waiters
    // poll the die counters (acquire via the acq_rel RMW chain of the W
    // arrivals) instead of the event counter, which the last arrival still
    // bumps after its fence (ref two-level completion, runtime.py:432-480)
    // but no longer on the critical path.
    // Likewise an event signalled by one fanned-out CU task alone: waiters
    // poll its unit sub-counter for n_units arrivals (dmask = -1 - sub_ctr,
    // the cached requirement becomes n_units).
    std::vector<int32_t> dm(std::max(1, g->n_events), 0), bad(std::max(1, g->n_events), 0);
    std::vector<int32_t> nsig(std::max(1, g->n_events), 0), last(std::max(1, g->n_events), -1);
    std::vector<int32_t> req(g->event_required, g->event_required + g->n_events);
    for (int i = 0; i < g->n_tasks; ++i) {
      const mk_task& t = g->tasks[i];
      if (t.signal < 0 || t.signal >= g->n_events) continue;
      ++nsig[t.signal];
      last[t.signal] = i;
      const int grp = g->n_schedulers == 1 ? 0 : t.die;
      if (t.level != MK_LEVEL_CHIPLET || grp < 0 || grp >= g->n_schedulers || grp >= 31 ||
          (dm[t.signal] >> grp) & 1)
        bad[t.signal] = 1;
      else
        dm[t.signal] |= 1 << grp;
    }
    for (int e = 0; e < g->n_events; ++e) {
      if (bad[e] || __builtin_popcount(uint32_t(dm[e])) != g->event_required[e] || !h->use_dmask) dm[e] = 0;
      if (h->use_dmask && nsig[e] == 1 && g->event_required[e] == 1) {
        const mk_task& t = g->tasks[last[e]];
        if (t.level != MK_LEVEL_CHIPLET && t.n_units > 1 && t.sub_ctr >= 0 && t.sub_ctr < g->n_sub_ctrs) {
          dm[e] = -1 - t.sub_ctr;
          req[e] = t.n_units;
        }
      }
    }
    CK(cudaMemcpy(h->d_ev_dmask, dm.data(), sizeof(int32_t) * g->n_events, cudaMemcpyHostToDevice));
    // cached per waiter as the poll target multiplier (ev_req is read nowhere else)
    CK(cudaMemcpy(h->d_ev_req, req.data(), sizeof(int32_t) * g->n_events, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(h->d_die_of_sm, die_of_sm.data(), MK_MAX_SMS, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->d_group_size, h->group_size.data(), sizeof(int32_t) * MK_MAX_DIES,
                cudaMemcpyHostToDevice));
  CK(cudaMemset(h->d_stats, 0, 32 * sizeof(unsigned long long)));
  CK(cudaMemset(h->d_log_cursor, 0, sizeof(unsigned long long)));
  CK(cudaMemset(h->d_tile_cursor, 0, sizeof(unsigned long long)));
  for (int i = 0; i < g->n_tasks; ++i) {
    const mk_task& t = g->tasks[i];
    if (t.op != MK_OP_GEMM) continue;
    const mk_gemm_params* gp =
        reinterpret_cast<const mk_gemm_params*>(static_cast<const uint8_t*>(g->params) + t.param_off);
    if (gp->body == MK_BODY_UMMA) h->feat |= kFeatUmma;
    if (gp->ksplit) h->feat |= kFeatKsplit;
  }
  {   // lean instance: every GEMM of one body kind (batch-1 GEMV, or all
      // tcgen05) and only the one-warp-per-item tensor-core attention
    bool lean = getenv("MK_NO_LEAN") == nullptr;
    int n_umma = 0, n_gemv = 0;
    for (int i = 0; i < g->n_tasks && lean; ++i) {
      const mk_task& t = g->tasks[i];
      const uint8_t* pb = static_cast<const uint8_t*>(g->params) + t.param_off;
      if (t.op == MK_OP_GEMM) {
        const mk_gemm_params* gp = reinterpret_cast<const mk_gemm_params*>(pb);
        if (gp->body == MK_BODY_UMMA) ++n_umma;
        else { ++n_gemv; lean = std::min(gp->T_M, gp->M) <= 1; }
      } else if (t.op == MK_OP_ATTN_PARTIAL) {
        const mk_attn_params* ap = reinterpret_cast<const mk_attn_params*>(pb);
        lean = attn_mma_path(*ap) && ap->sub_splits == 1;
      }
    }
    if (lean && !(n_umma && n_gemv)) h->feat |= kFeatLean;
  }
  for (int i = 0; i < g->n_tasks; ++i)
    if (g->tasks[i].op == MK_OP_TP_ALLREDUCE || g->tasks[i].op == MK_OP_TP_ARGMAX) h->has_tp_tasks = true;
  h->kernel = kernel_for(h->feat);
  CK(cudaFuncSetAttribute(h->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->kernel, kThreads, kSmemBytes));
  if (occ != 1) {
    delete h;
    return fail(MK_ERR_CONFIG, "megakernel occupancy is " + std::to_string(occ) + ", need exactly 1");
  }
  for (int i = 0; i < g->n_tasks; ++i) {
    const mk_task& t = g->tasks[i];
    if (t.op == MK_OP_GEMM &&
        reinterpret_cast<const mk_gemm_params*>(static_cast<const uint8_t*>(g->params) + t.param_off)->body ==
            MK_BODY_UMMA)
      h->use_umma = 1;
  }
  rc = build_tmaps(h, g);
  if (rc) { delete h; return rc; }
  rc = reset_state(h);
  if (rc) { delete h; return rc; }
  *out = h;
  return MK_OK;
}

int mk_step(mk_handle* h, void* stream) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  CK(cudaSetDevice(h->device));
  KArgs a;
  a.tasks = h->d_tasks; a.units = h->d_units; a.sched_begin = h->d_sched_begin;
  a.params = h->d_params; a.ev_ctr = h->d_ev_ctr; a.ev_req = h->d_ev_req;
  a.ev_dmask = h->d_ev_dmask;
  a.die_ctr = h->d_die_ctr; a.sub_ctr = h->d_sub_ctr; a.mailbox = h->d_mailbox;
  a.mb_head = h->d_mb_head; a.mb_tail = h->d_mb_tail; a.die_of_sm = h->d_die_of_sm;
  a.role_ctr = h->d_role_ctr; a.group_size = h->d_group_size; a.stats = h->d_stats;
  a.log = h->log_cap ? h->d_log : nullptr; a.log_cursor = h->d_log_cursor; a.log_cap = h->log_cap;
  a.tile_log = h->tile_cap ? h->d_tile_log : nullptr; a.tile_cursor = h->d_tile_cursor;
  a.tile_cap = h->tile_cap;
  a.err = h->d_err; a.err_info = h->d_err + 1;
  a.watchdog_ns = (unsigned long long)(h->watchdog_s * 1e9);
  a.n_events = h->n_events; a.n_sched = h->n_sched; a.sched_mode = h->sched_mode; a.W = h->W;
  a.epoch = h->epoch + 1;   // committed below, only if the launch was accepted
  a.debug = h->debug;
  a.use_umma = h->use_umma;
  a.tmaps = h->d_tmaps;
  a.x_stages = h->x_stages;
  a.x_stage_bytes = h->x_stage_bytes;
  a.pf_slots = h->pf_slots;
  a.trace = h->trace_cap ? h->d_trace : nullptr;
  a.positions = h->positions; a.n_rows = h->n_rows;
  a.trace_cap = h->trace_cap;
  a.tp_world = h->tp_world; a.tp_rank = h->tp_rank;
  for (int q = 0; q < MK_MAX_TP; ++q) a.tp_peer[q] = h->tp_peer[q];
  if (h->has_tp_tasks && h->tp_world < 2)
    return fail(MK_ERR_CONFIG, "graph has tensor-parallel tasks: call mk_tp_init first");
  void* args[] = {&a};
  if (h->cooperative) {
    CK(cudaLaunchCooperativeKernel(h->kernel, dim3(h->num_sms), dim3(kThreads), args,
                                   kSmemBytes, static_cast<cudaStream_t>(stream)));
  } else {
    CK(cudaLaunchKernel(h->kernel, dim3(h->num_sms), dim3(kThreads), args,
                        kSmemBytes, static_cast<cudaStream_t>(stream)));
  }
  h->epoch = a.epoch;
  return MK_OK;
}

int mk_step_tokens(mk_handle* h, void* stream, const int32_t* tokens_in, int32_t* tokens_out) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  if (!h->tokens || !h->out_tokens)
    return fail(MK_ERR_CONFIG, "graph descriptor carries no token buffers");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(int32_t) * size_t(h->n_rows);
  if (tokens_in) CK(cudaMemcpyAsync(h->tokens, tokens_in, bytes, cudaMemcpyHostToDevice, st));
  const int rc = mk_step(h, stream);
  if (rc != MK_OK) return rc;
  if (tokens_out) CK(cudaMemcpyAsync(tokens_out, h->out_tokens, bytes, cudaMemcpyDeviceToHost, st));
  return MK_OK;
}

int mk_sync(mk_handle* h) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h->h_err, h->d_err, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  if (h->h_err[0] != 0) {
    const int code = h->h_err[0], info = h->h_err[1];
    reset_state(h);
    if (code == MK_ERR_CONFIG && info <= -100 && info > -200)
      return fail(code, "decode position of row " + std::to_string(-100 - info) +
                            " is outside the KV cache (t_max): step aborted");
    if (code == MK_ERR_CONFIG)
      return fail(code, "device role assignment out of step (site " + std::to_string(info) + ")");
    return fail(code, "device watchdog: no progress (event/site " + std::to_string(info) + ")");
  }
  return MK_OK;
}

int mk_counters_get(mk_handle* h, mk_counters* out) {
  if (!h || !out) return fail(MK_ERR_CONFIG, "null argument");
  CK(cudaSetDevice(h->device));
  unsigned long long s[32];
  CK(cudaMemcpy(s, h->d_stats, sizeof(s), cudaMemcpyDeviceToHost));
  out->dispatches = s[S_DISPATCH]; out->mailbox_writes = s[S_MAILBOX];
  out->global_atomics = s[S_GLOBAL]; out->local_atomics = s[S_LOCAL]; out->fences = s[S_FENCE];
  out->fanout_atomics = s[S_FANOUT]; out->polls = s[S_POLL]; out->tiles = s[S_TILES];
  out->executions = s[S_EXEC]; out->steps = s[S_STEPS];
  out->wait_ring_empty = s[S_W_RING_EMPTY]; out->wait_mma_full = s[S_W_MMA_FULL];
  out->wait_mma_x = s[S_W_MMA_X]; out->wait_mma_tmem = s[S_W_MMA_TMEM];
  out->wait_epi_done = s[S_W_EPI_DONE]; out->mma_chunks = s[S_MMA_CHUNKS];
  return MK_OK;
}

int mk_counters_reset(mk_handle* h) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  CK(cudaSetDevice(h->device));
  CK(cudaMemset(h->d_stats, 0, 32 * sizeof(unsigned long long)));
  return MK_OK;
}

int mk_log_enable(mk_handle* h, int64_t capacity) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  CK(cudaSetDevice(h->device));
  if (h->d_log) { CK(cudaFree(h->d_log)); h->d_log = nullptr; }
  h->log_cap = 0;
  if (capacity > 0) {
    CK(cudaMalloc(&h->d_log, sizeof(mk_log_rec) * capacity));
    h->log_cap = capacity;
  }
  CK(cudaMemset(h->d_log_cursor, 0, sizeof(unsigned long long)));
  return MK_OK;
}

int64_t mk_log_read(mk_handle* h, mk_log_rec* out, int64_t max_records) {
  if (!h || !out) return -fail(MK_ERR_CONFIG, "null argument");
  if (cudaSetDevice(h->device) != cudaSuccess) return -MK_ERR_CUDA;
  unsigned long long n = 0;
  if (cudaMemcpy(&n, h->d_log_cursor, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess) return -MK_ERR_CUDA;
  long long m = std::min<long long>((long long)n, std::min<long long>(h->log_cap, max_records));
  if (m > 0 && cudaMemcpy(out, h->d_log, sizeof(mk_log_rec) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -MK_ERR_CUDA;
  return (int64_t)n;
}

int mk_tile_log_enable(mk_handle* h, int64_t capacity) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  CK(cudaSetDevice(h->device));
  if (h->d_tile_log) { CK(cudaFree(h->d_tile_log)); h->d_tile_log = nullptr; }
  h->tile_cap = 0;
  if (capacity > 0) {
    CK(cudaMalloc(&h->d_tile_log, sizeof(int32_t) * 4 * capacity));
    h->tile_cap = capacity;
  }
  CK(cudaMemset(h->d_tile_cursor, 0, sizeof(unsigned long long)));
  return MK_OK;
}

int64_t mk_tile_log_read(mk_handle* h, int32_t* out4, int64_t max_records) {
  if (!h || !out4) return -fail(MK_ERR_CONFIG, "null argument");
  if (cudaSetDevice(h->device) != cudaSuccess) return -MK_ERR_CUDA;
  unsigned long long n = 0;
  if (cudaMemcpy(&n, h->d_tile_cursor, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess) return -MK_ERR_CUDA;
  long long m = std::min<long long>((long long)n, std::min<long long>(h->tile_cap, max_records));
  if (m > 0 && cudaMemcpy(out4, h->d_tile_log, sizeof(int32_t) * 4 * m, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -MK_ERR_CUDA;
  return (int64_t)n;
}

int mk_trace_enable(mk_handle* h, int32_t units_per_worker) {
  if (!h || units_per_worker < 0) return fail(MK_ERR_CONFIG, "bad trace capacity");
  CK(cudaSetDevice(h->device));
  if (h->d_trace) { CK(cudaFree(h->d_trace)); h->d_trace = nullptr; }
  h->trace_cap = 0;
  if (units_per_worker > 0) {
    const size_t n = size_t(h->n_sched) * h->W * units_per_worker * 8;
    CK(cudaMalloc(&h->d_trace, n * sizeof(uint64_t)));
    CK(cudaMemset(h->d_trace, 0, n * sizeof(uint64_t)));
    h->trace_cap = units_per_worker;
  }
  return MK_OK;
}

int64_t mk_trace_read(mk_handle* h, uint64_t* out, int64_t max_words) {
  if (!h || !out) return -fail(MK_ERR_CONFIG, "null argument");
  if (cudaSetDevice(h->device) != cudaSuccess) return -MK_ERR_CUDA;
  const int64_t n = int64_t(h->n_sched) * h->W * h->trace_cap * 8;
  const int64_t m = std::min(n, max_words);
  if (m > 0 && cudaMemcpy(out, h->d_trace, m * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -MK_ERR_CUDA;
  return n;
}

int mk_set_watchdog(mk_handle* h, double seconds) {
  if (!h || !(seconds > 0)) return fail(MK_ERR_CONFIG, "bad watchdog");
  h->watchdog_s = seconds;
  return MK_OK;
}

int mk_set_prefetch(mk_handle* h, int slots) {
  if (!h || slots < 0 || slots > 1024) return fail(MK_ERR_CONFIG, "bad prefetch depth");
  h->pf_slots = slots;
  return MK_OK;
}

int mk_set_debug(mk_handle* h, int flags) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  h->debug = flags;
  return MK_OK;
}

int mk_tp_init(mk_handle* h, int rank, int world, void* const* peer_bases) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  if (world < 1 || world > MK_MAX_TP || rank < 0 || rank >= world || (world > 1 && !peer_bases))
    return fail(MK_ERR_CONFIG, "bad tensor-parallel rank / world / peers");
  if (h->epoch != 0) return fail(MK_ERR_CONFIG, "mk_tp_init after the first step");
  for (int q = 0; q < world; ++q)
    if (!peer_bases[q]) return fail(MK_ERR_CONFIG, "null peer exchange region");
  h->tp_rank = rank;
  h->tp_world = world;
  for (int q = 0; q < MK_MAX_TP; ++q)
    h->tp_peer[q] = q < world ? static_cast<uint8_t*>(peer_bases[q]) : nullptr;
  return MK_OK;
}

int mk_tp_alloc(int device, size_t bytes, void** out) {
  if (!out || bytes == 0) return fail(MK_ERR_CONFIG, "bad exchange-region request");
  CK(cudaSetDevice(device));
  CK(cudaMalloc(out, bytes));
  CK(cudaMemset(*out, 0, bytes));
  return MK_OK;
}

int mk_tp_free(void* ptr) {
  if (ptr) CK(cudaFree(ptr));
  return MK_OK;
}

int mk_ipc_export(void* ptr, uint8_t* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t hd;
  CK(cudaIpcGetMemHandle(&hd, ptr));
  std::memcpy(handle64, &hd, sizeof(hd));
  return MK_OK;
}

int mk_ipc_import(int device, const uint8_t* handle64, void** out) {
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, sizeof(hd));
  CK(cudaSetDevice(device));
  CK(cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess));
  return MK_OK;
}

int mk_ipc_close(void* ptr) {
  if (ptr) CK(cudaIpcCloseMemHandle(ptr));
  return MK_OK;
}

int mk_set_grid(mk_handle* h, int ctas, int cooperative) {
  if (!h) return fail(MK_ERR_CONFIG, "null handle");
  if (h->epoch != 0) return fail(MK_ERR_CONFIG, "mk_set_grid after the first step");
  if (h->sched_mode != MK_SCHED_FLAT || ctas < 2 || ctas > h->num_sms || h->W > ctas - 1)
    return fail(MK_ERR_CONFIG, "mk_set_grid: flat scheduler, 2..#SMs CTAs, workers <= ctas - 1");
  CK(cudaSetDevice(h->device));
  h->num_sms = ctas;
  h->group_size[0] = ctas;
  CK(cudaMemcpy(h->d_group_size, h->group_size.data(), sizeof(int32_t) * MK_MAX_DIES,
                cudaMemcpyHostToDevice));
  h->cooperative = cooperative ? 1 : 0;
  return MK_OK;
}

int mk_destroy(mk_handle* h) {
  if (!h) return MK_OK;
  cudaSetDevice(h->device);
  cudaFree(h->d_tasks); cudaFree(h->d_units); cudaFree(h->d_sched_begin); cudaFree(h->d_params);
  cudaFree(h->d_ev_ctr); cudaFree(h->d_ev_req); cudaFree(h->d_ev_dmask); cudaFree(h->d_die_ctr); cudaFree(h->d_sub_ctr);
  cudaFree(h->d_mailbox); cudaFree(h->d_mb_head); cudaFree(h->d_mb_tail); cudaFree(h->d_die_of_sm);
  cudaFree(h->d_role_ctr); cudaFree(h->d_group_size); cudaFree(h->d_stats); cudaFree(h->d_err);
  cudaFree(h->d_log); cudaFree(h->d_log_cursor); cudaFree(h->d_tile_log); cudaFree(h->d_tile_cursor);
  cudaFree(h->d_tmaps); cudaFree(h->d_trace);
  if (h->h_err) cudaFreeHost(h->h_err);
  delete h;
  return MK_OK;
}

}  // extern "C"

#endif  // MK_INSTANCE
