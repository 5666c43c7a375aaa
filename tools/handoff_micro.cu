// Cross-SM hand-off latency on B200 (diagnostic micro-benchmark, not product
// code).  One producer CTA writes an 8 KiB activation row and releases a
// flag; every other CTA acquires the flag and loads the row with ld.cg --
// the megakernel's stage-boundary pattern.  Reports the median time from the
// acquire to "row loaded" under four conditions:
//   mode 0: the row lives at one fixed address
//   mode 1: the row moves to a fresh 2 MiB page every iteration (TLB cold)
//   mode 2: mode 0 + background HBM streaming by warps 4..7 of every CTA
//   mode 3: mode 1 + background streaming
//   mode 4: mode 3, but the loader touches the next row's page one
//           iteration early (translation warm-up)
//   mode 5: fixed row + background TMA bulk streaming like the megakernel's
//           ring (one lane per CTA keeps 10 x 16 KiB copies in flight)
//   mode 6: mode 5 with 4 copies in flight
//   mode 7: mode 5 with 2 copies in flight
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o handoff tools/handoff_micro.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ldcg(const void* p) {
  uint4 v; asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

constexpr int kIters = 200;
constexpr size_t kPage = 2u << 20;

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256, 1) handoff(uint8_t* rows, uint32_t* flag, uint32_t* done,
                                                  const uint4* stream, size_t stream_n, int mode,
                                                  uint64_t* out, volatile int* stop) {
  extern __shared__ uint4 sm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = gridDim.x;
  const bool bg = mode >= 2;
  __shared__ __align__(8) uint64_t bars[16];
  if (mode >= 5) {
    const int depth = mode == 5 ? 10 : (mode == 6 ? 4 : 2);
    if (warp >= 4) {
      if (tid != 128) return;
      for (int i = 0; i < depth; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bars[i])));
      asm volatile("fence.mbarrier_init.release.cluster;");
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      const char* src = reinterpret_cast<const char*>(stream);
      const size_t nchunk = stream_n * 16 / 16384;
      size_t c = size_t(blockIdx.x) * 997;
      uint32_t ph[16] = {0};
      for (int i = 0; i < depth; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[i])), "r"(16384));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     :: "r"(su32(reinterpret_cast<char*>(sm) + i * 16384)), "l"(src + (c++ % nchunk) * 16384), "r"(16384),
                        "r"(su32(&bars[i])), "l"(pol) : "memory");
      }
      for (int i = 0; !*stop; i = (i + 1) % depth) {
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bars[i])), "r"(ph[i]) : "memory");
        }
        ph[i] ^= 1;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bars[i])), "r"(16384));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     :: "r"(su32(reinterpret_cast<char*>(sm) + i * 16384)), "l"(src + (c++ % nchunk) * 16384), "r"(16384),
                        "r"(su32(&bars[i])), "l"(pol) : "memory");
      }
      for (int i = 0; i < depth; ++i) {   // drain
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bars[i])), "r"(ph[i]) : "memory");
        }
      }
      return;
    }
  } else if (bg && warp >= 4) {   // background streaming
    size_t i = (size_t(blockIdx.x) * 128 + (tid - 128)) * 4;
    uint4 acc = make_uint4(0, 0, 0, 0);
    while (!*stop) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 v = ldcg(stream + (i + u) % stream_n);
        acc.x ^= v.x; acc.y ^= v.y;
      }
      i += size_t(nb) * 128 * 4;
    }
    if (acc.x == 0x12345 && acc.y == 7) out[0] = 1;
    return;
  }
  const int nt = bg ? 128 : 256;
  uint4* xs = sm + (mode >= 5 ? 10 * 1024 : 0);   // past the TMA ring
  __shared__ uint64_t t_acq;
  __shared__ uint32_t sink;
  for (int it = 0; it < kIters; ++it) {
    const int prod = it % nb;
    const size_t off = (mode == 1 || mode >= 3) ? size_t(it) * kPage : 0;
    uint8_t* row = rows + off;
    if (blockIdx.x == prod) {
      if (tid < nt) {
        if (tid == 0) {   // previous readers done (WAR)
          while (ld_acq(done) < uint32_t(it) * (nb - 1)) {}
        }
        asm volatile("bar.sync 1, %0;" :: "r"(nt));
        for (int k = tid; k < 512; k += nt) reinterpret_cast<uint4*>(row)[k] = make_uint4(it, k, 1, 2);
        __threadfence();
        if (tid == 0) out[size_t(kIters) * nb + it] = gtime();
        asm volatile("bar.sync 1, %0;" :: "r"(nt));
        if (tid == 0) red_rel(flag, 1u);
      }
      continue;
    }
    if (tid < nt) {
      if (mode == 4 && tid == 0) {   // warm the next row's translation
        const uint8_t* nxt = rows + size_t(it + 1) * kPage;
        asm volatile("prefetch.global.L2 [%0];" :: "l"(nxt));
      }
      if (tid == 0) {
        while (ld_acq(flag) < uint32_t(it + 1)) {}
        t_acq = gtime();
        out[size_t(kIters) * nb + kIters + size_t(it) * nb + blockIdx.x] = t_acq;
      }
      asm volatile("bar.sync 1, %0;" :: "r"(nt));
      uint32_t x = 0;
      for (int k = tid; k < 512; k += nt) { uint4 v = ldcg(reinterpret_cast<uint4*>(row) + k); x ^= v.x ^ v.y; xs[k] = v; }
      asm volatile("bar.sync 1, %0;" :: "r"(nt));
      if (tid == 0) {
        out[size_t(it) * nb + blockIdx.x] = gtime() - t_acq;
        sink = x;
        atomicAdd(done, 1u);
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) *stop = 1;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* rows; uint32_t* ctr; uint4* stream; uint64_t* out; int* stop;
  const size_t stream_bytes = size_t(4) << 30;
  cudaMalloc(&rows, (kIters + 2) * kPage);
  cudaMalloc(&ctr, 64);
  cudaMalloc(&stream, stream_bytes);
  cudaMemset(stream, 1, stream_bytes);
  const size_t nout = size_t(kIters) * nsm * 2 + kIters;
  cudaMalloc(&out, sizeof(uint64_t) * nout);
  cudaMalloc(&stop, 4);
  cudaFuncSetAttribute(handoff, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"fixed row", "fresh 2MiB page per row", "fixed row + HBM stream",
                         "fresh page + HBM stream", "fresh page + stream + L2 prefetch warm-up",
                         "fixed row + TMA ring 10x16K in flight", "TMA ring 4 in flight", "TMA ring 2 in flight"};
  for (int mode = 0; mode < 8; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 64); cudaMemset(stop, 0, 4); cudaMemset(out, 0, sizeof(uint64_t) * nout);
      handoff<<<nsm, 256, 200 * 1024>>>(rows, ctr, ctr + 8, stream, stream_bytes / 16, mode, out, stop);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<uint64_t> h(nout);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<double> v;
    for (int it = 10; it < kIters; ++it)
      for (int b = 0; b < nsm; ++b) if (b != it % nsm && h[size_t(it) * nsm + b]) v.push_back(h[size_t(it) * nsm + b] / 1e3);
    std::sort(v.begin(), v.end());
    std::vector<double> hop;
    const uint64_t* rel = h.data() + size_t(kIters) * nsm;
    const uint64_t* acq = rel + kIters;
    for (int it = 10; it < kIters; ++it)
      for (int b = 0; b < nsm; ++b)
        if (b != it % nsm && acq[size_t(it) * nsm + b]) hop.push_back((double(acq[size_t(it) * nsm + b]) - double(rel[it])) / 1e3);
    std::sort(hop.begin(), hop.end());
    printf("mode %d: release->acquire  p10 %.2f  p50 %.2f  p90 %.2f us\n", mode, hop[hop.size() / 10],
           hop[hop.size() / 2], hop[hop.size() * 9 / 10]);
    printf("mode %d (%s): acquire->row loaded  p10 %.2f  p50 %.2f  p90 %.2f  max %.2f us  (n=%zu)\n", mode,
           names[mode], v[v.size() / 10], v[v.size() / 2], v[v.size() * 9 / 10], v.back(), v.size());
  }
  return 0;
}
