// mk_ptx.cuh -- thin inline-PTX wrappers used by the persistent kernel (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace mk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t r;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
  return r;
}

// ---- gpu-scope synchronisation (event counters, mailboxes) -------------
// system scope (peer GPUs over NVLink): tensor-parallel exchange flags
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_sys() {
  asm volatile("fence.sc.sys;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Spin loops poll with relaxed loads (ld.acquire compiles to a load plus an
// L1 invalidate, CCTL.IVALL, on every iteration) and issue one acquire
// fence once the awaited value is seen.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acq_rel_add(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
               : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// ---- named barriers -----------------------------------------------------
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// ---- mbarrier ------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// non-blocking probe of a phase (no thread suspension)
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// ---- TMA 1-D bulk copy global -> shared, completion on an mbarrier ------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// the same without a cache hint (activations / norm gammas: default policy)
__device__ __forceinline__ void bulk_g2s_plain(void* dst_smem, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---- vector shared / global loads ---------------------------------------
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
// Activations are produced by other SMs inside the same launch: load them
// through L2 (.cg) so a line cached in L1 before the producer ran is never
// returned.
__device__ __forceinline__ uint4 ldg128_cg(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// GEMM output element (the reference's NON_TEMPORAL output store role,
// traversal.py:296-313): not allocated in the producing SM's L1 -- the
// consumers are other SMs and read it from L2, the GPU's coherence point
__device__ __forceinline__ void st_out(uint16_t* p, uint16_t v) {
  asm volatile("st.global.L1::no_allocate.b16 [%0], %1;" :: "l"(p), "h"(v) : "memory");
}

// small static operands (norm gammas, RoPE tables): keep them L2-resident
// while the weight stream (evict_first) passes through
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ldg128_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ldg32_cg(const void* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint16_t ldg16_cg(const void* p) {
  uint16_t v;
  asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&b);
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  f[0] = bf16lo(v.x); f[1] = bf16hi(v.x);
  f[2] = bf16lo(v.y); f[3] = bf16hi(v.y);
  f[4] = bf16lo(v.z); f[5] = bf16hi(v.z);
  f[6] = bf16lo(v.w); f[7] = bf16hi(v.w);
}

}  // namespace mk

// ---- warp-level tensor-core MMA (decode attention: 4-8 query rows) ---------
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
// D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col); rows 8-15 of A are
// zero here (a1 = a3 = 0), so only d0, d1 carry results.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---- tcgen05 / TMEM (5th-gen tensor cores) ---------------------------------
namespace mk {

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operands)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// generic-proxy global writes (seen through an acquire) -> visible to
// async-proxy (TMA) reads issued after this fence
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 2-D TMA tile load global -> shared (tensor map in global memory), completion
// on an mbarrier; coordinates are (inner element, row)
__device__ __forceinline__ void tma_load_2d(void* dst_smem, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_u32(dst_smem)), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(tmap) : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
// One K-chunk (4 x UMMA_K = 16) of the skinny GEMM into 4 independent
// accumulators (columns d, d+64, d+128, d+192), issued by the whole warp
// in one convergent block: elect.sync picks the issuing lane inside the asm
// (no divergent C++ branch around the MMAs, so the operands stay in
// uniform registers); then `arrivals` plain arrivals on `slot_bar` and a
// commit to it and to `x_bar` (both complete when the MMAs have read smem).
__device__ __forceinline__ void umma_chunk4(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                            uint32_t accumulate, uint64_t* slot_bar, uint32_t arrivals,
                                            uint64_t* x_bar) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      ".reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      ".reg .b32 e1, e2, e3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2; add.s64 a2, %1, 4; add.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2; add.s64 b2, %2, 4; add.s64 b3, %2, 6;\n\t"
      "add.u32 e1, %0, 64; add.u32 e2, %0, 128; add.u32 e3, %0, 192;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e1], a1, b1, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e2], a2, b2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e3], a3, b3, %3, p;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 _, [%5], %6;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}"
      :: "r"(d_tmem), "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate), "r"(smem_u32(slot_bar)),
         "r"(arrivals), "r"(smem_u32(x_bar))
      : "memory");
}

// Two K-chunks in one block (8 MMAs): chunk 0 on (a0, b0) releasing slot0,
// chunk 1 on (a1, b1) releasing slot1, then the pair's activation stage x.
__device__ __forceinline__ void umma_chunk8(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint64_t a1,
                                            uint64_t b1, uint32_t idesc, uint32_t accumulate,
                                            uint64_t* slot0, uint64_t* slot1, uint32_t arrivals,
                                            uint64_t* x) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t"
      ".reg .b64 c1, c2, c3, d1, d2, d3, f1, f2, f3, g1, g2, g3;\n\t"
      ".reg .b32 e1, e2, e3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "add.u32 e1, %0, 64; add.u32 e2, %0, 128; add.u32 e3, %0, 192;\n\t"
      "add.s64 c1, %1, 2; add.s64 c2, %1, 4; add.s64 c3, %1, 6;\n\t"
      "add.s64 d1, %2, 2; add.s64 d2, %2, 4; add.s64 d3, %2, 6;\n\t"
      "add.s64 f1, %3, 2; add.s64 f2, %3, 4; add.s64 f3, %3, 6;\n\t"
      "add.s64 g1, %4, 2; add.s64 g2, %4, 4; add.s64 g3, %4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e1], c1, d1, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e2], c2, d2, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e3], c3, d3, %5, p;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 _, [%7], %9;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e1], f1, g1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e2], f2, g2, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [e3], f3, g3, %5, t;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 _, [%8], %9;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n\t}"
      :: "r"(d_tmem), "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate),
         "r"(smem_u32(slot0)), "r"(smem_u32(slot1)), "r"(arrivals), "r"(smem_u32(x))
      : "memory");
}

// Diagnostics variants of umma_chunk8 (timing only; results are wrong):
// mode 1: one commit per pair (slot0 and x released by plain arrivals);
// mode 2: only the first chunk's 4 MMAs, commits as umma_chunk8.
__device__ __forceinline__ void umma_chunk8_dbg(int mode, uint32_t d_tmem, uint64_t a0, uint64_t b0,
                                                uint64_t a1, uint64_t b1, uint32_t idesc,
                                                uint32_t accumulate, uint64_t* slot0, uint64_t* slot1,
                                                uint32_t arrivals, uint64_t* x) {
  if (mode == 1) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t"
        ".reg .b64 c1, c2, c3, d1, d2, d3, f1, f2, f3, g1, g2, g3;\n\t"
        ".reg .b32 e1, e2, e3, n1;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "add.u32 e1, %0, 64; add.u32 e2, %0, 128; add.u32 e3, %0, 192; add.u32 n1, %9, 1;\n\t"
        "add.s64 c1, %1, 2; add.s64 c2, %1, 4; add.s64 c3, %1, 6;\n\t"
        "add.s64 d1, %2, 2; add.s64 d2, %2, 4; add.s64 d3, %2, 6;\n\t"
        "add.s64 f1, %3, 2; add.s64 f2, %3, 4; add.s64 f3, %3, 6;\n\t"
        "add.s64 g1, %4, 2; add.s64 g2, %4, 4; add.s64 g3, %4, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e1], c1, d1, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e2], c2, d2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e3], c3, d3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %5, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e1], f1, g1, %5, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e2], f2, g2, %5, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [e3], f3, g3, %5, t;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%7], n1;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%10];\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%8], %9;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}"
        :: "r"(d_tmem), "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate),
           "r"(smem_u32(slot0)), "r"(smem_u32(slot1)), "r"(arrivals), "r"(smem_u32(x))
        : "memory");
  } else {
    umma_chunk4(d_tmem, a0, b0, idesc, accumulate, slot0, arrivals, x);
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        :: "r"(smem_u32(slot1)), "r"(arrivals) : "memory");
  }
}

// arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 16 columns of fp32 from TMEM: thread t gets lane (base+t), cols c..c+15
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: rows of 64 bf16
// (128 B) in 1024-byte 8-row atoms; SBO = 1024 B, version bits 46-47 = 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr & 0x3FFFFu) >> 4);          // start address
  d |= uint64_t(1) << 16;                               // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;                       // SBO: next 8-row atom
  d |= uint64_t(1) << 46;                               // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                               // SWIZZLE_128B
  return d;
}

// Instruction descriptor: bf16 x bf16 -> fp32, both K-major, M x N tile.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4)                     // D = fp32
       | (1u << 7)                     // A = bf16
       | (1u << 10)                    // B = bf16
       | (uint32_t(N >> 3) << 17)      // N / 8
       | (uint32_t(M >> 4) << 24);     // M / 16
}

}  // namespace mk
