// tma_stream_bench.cu — read bandwidth of the k_mv_batched pipeline shape on B200: one
// persistent CTA per SM (or two), a producer lane issuing cp.async.bulk copies into a ring of
// shared-memory stages (mbarrier complete_tx), consumer warps reading every staged double.
// Variables: stages, stage bytes, copies per stage (segment granularity), CTAs per SM.
// Baseline: plain coalesced 16-B loads from many warps.  Prints one JSON line per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// CTA-shared ring: warp 0 produces, warps 1.. consume every stage (the k_mv_batched shape)
__global__ void k_ring(const char* __restrict__ src, int64_t bytes_per_cta, int stages, int stage_bytes, int segs,
                       double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  unsigned char* buf = smem + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nc = blockDim.x / 32 - 1;
  const char* base = src + blockIdx.x * bytes_per_cta;
  const int nb = (int)(bytes_per_cta / stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nc); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    const int seg = stage_bytes / segs;
    for (int it = 0; it < nb; ++it) {
      const int st = it % stages;
      if (it >= stages) mbar_wait(&empty[st], (unsigned)(((it / stages) - 1) & 1));
      if (lane == 0) mbar_expect_tx(&full[st], (unsigned)stage_bytes);
      __syncwarp();
      for (int s = lane; s < segs; s += 32)
        bulk_g2s(buf + st * stage_bytes + s * seg, base + (int64_t)it * stage_bytes + s * seg, seg, &full[st]);
    }
    return;
  }
  double acc = 0;
  for (int it = 0; it < nb; ++it) {
    const int st = it % stages;
    mbar_wait(&full[st], (unsigned)((it / stages) & 1));
    const double* d = reinterpret_cast<const double*>(buf + st * stage_bytes);
    for (int i = (warp - 1) * 32 + lane; i < stage_bytes / 8; i += nc * 32) acc += d[i];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
  }
  if (acc == 12345.678) out[0] = acc;
}

// per-warp rings: every warp streams its own sub-range through its own `stages` buffers,
// issuing its own copies (no producer warp, no cross-warp barrier)
__global__ void k_warpring(const char* __restrict__ src, int64_t bytes_per_warp, int stages, int stage_bytes, int segs,
                           double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  unsigned char* buf = smem + 1024 + (size_t)warp * stages * stage_bytes;
  const char* base = src + ((int64_t)blockIdx.x * nw + warp) * bytes_per_warp;
  const int nb = (int)(bytes_per_warp / stage_bytes);
  const int seg = stage_bytes / segs;
  if (lane == 0) for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int it) {
    const int st = it % stages;
    if (lane == 0) mbar_expect_tx(&full[st], (unsigned)stage_bytes);
    __syncwarp();
    for (int s = lane; s < segs; s += 32)
      bulk_g2s(buf + st * stage_bytes + s * seg, base + (int64_t)it * stage_bytes + s * seg, seg, &full[st]);
  };
  for (int it = 0; it < stages && it < nb; ++it) issue(it);
  double acc = 0;
  for (int it = 0; it < nb; ++it) {
    const int st = it % stages;
    mbar_wait(&full[st], (unsigned)((it / stages) & 1));
    const double* d = reinterpret_cast<const double*>(buf + st * stage_bytes);
    for (int i = lane; i < stage_bytes / 8; i += 32) acc += d[i];
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (it + stages < nb) issue(it + stages);
  }
  if (acc == 12345.678) out[0] = acc;
}

// the k_mv_batched segment pattern: per stage, nx copies of xb bytes from a small L2-resident
// vector (x_sigma), one header copy, and the rest of the stage as one contiguous data run
__global__ void k_ring_mixed(const char* __restrict__ src, const char* __restrict__ xsrc, int64_t bytes_per_cta,
                             int stages, int stage_bytes, int nx, int xb, double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  unsigned char* buf = smem + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nc = blockDim.x / 32 - 1;
  const int run = stage_bytes - nx * xb - 256;
  const char* base = src + blockIdx.x * bytes_per_cta;
  const int nb = (int)(bytes_per_cta / run);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nc); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    for (int it = 0; it < nb; ++it) {
      const int st = it % stages;
      if (it >= stages) mbar_wait(&empty[st], (unsigned)(((it / stages) - 1) & 1));
      if (lane == 0) mbar_expect_tx(&full[st], (unsigned)stage_bytes);
      __syncwarp();
      unsigned char* sb = buf + st * stage_bytes;
      if (lane == 0) bulk_g2s(sb, base + 256 * (it % 64), 256, &full[st]);
      if (lane == 1) bulk_g2s(sb + 256, base + (int64_t)it * run, run, &full[st]);
      for (int s = lane; s < nx; s += 32) {
        const int64_t xo = ((int64_t)(it * 37 + s * 101) * 256) % (2 << 20);
        bulk_g2s(sb + 256 + run + s * xb, xsrc + xo, xb, &full[st]);
      }
    }
    return;
  }
  double acc = 0;
  for (int it = 0; it < nb; ++it) {
    const int st = it % stages;
    mbar_wait(&full[st], (unsigned)((it / stages) & 1));
    const double* d = reinterpret_cast<const double*>(buf + st * stage_bytes);
    for (int i = (warp - 1) * 32 + lane; i < stage_bytes / 8; i += nc * 32) acc += d[i];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_plain(const double2* __restrict__ src, int64_t n2, double* __restrict__ out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(src + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 8LL << 30;   // 8 GiB, >> L2
  char* src;
  double* out;
  cudaMalloc(&src, total + 4096);
  cudaMalloc(&out, 8);
  cudaMemset(src, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
  };
  {
    float ms = timeit([&] { k_plain<<<sms * 8, 512>>>((const double2*)src, total / 16, out); });
    printf("{\"variant\":\"plain_ldg128\",\"GBps\":%.1f}\n", total / (ms * 1e-3) / 1e9);
  }
  struct V { int stages, stage_kb, segs, threads, ctas_per_sm; };
  V vs[] = {{4, 48, 1, 512, 1},  {4, 48, 12, 512, 1}, {4, 48, 48, 512, 1}, {6, 32, 1, 512, 1}, {8, 24, 1, 512, 1},
            {8, 24, 8, 512, 1},  {12, 16, 1, 512, 1}, {16, 12, 1, 512, 1}, {2, 48, 1, 256, 2}, {4, 24, 1, 256, 2},
            {8, 12, 1, 256, 2},  {4, 48, 1, 256, 1},  {4, 48, 1, 128, 1}};
  for (const V& v : vs) {
    const int sb = v.stage_kb * 1024;
    const int smem = 256 + v.stages * sb;
    if (smem > 227 * 1024) continue;
    cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * v.ctas_per_sm;
    const int64_t per = (total / grid) / sb * sb;
    float ms = timeit([&] { k_ring<<<grid, v.threads, smem>>>(src, per, v.stages, sb, v.segs, out); });
    printf("{\"variant\":\"ring\",\"stages\":%d,\"stage_kb\":%d,\"segs\":%d,\"threads\":%d,\"ctas_per_sm\":%d,\"GBps\":%.1f,\"err\":\"%s\"}\n",
           v.stages, v.stage_kb, v.segs, v.threads, v.ctas_per_sm, (double)per * grid / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    char* xs;
    cudaMalloc(&xs, 4 << 20);
    cudaMemset(xs, 0, 4 << 20);
    struct M { int nx, xb; };
    M ms_[] = {{0, 0}, {8, 256}, {16, 192}, {32, 192}, {48, 128}, {16, 512}};
    for (const M& m : ms_) {
      const int sb = 48 * 1024, stages = 4;
      const int smem = 256 + stages * sb;
      cudaFuncSetAttribute(k_ring_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int run = sb - m.nx * m.xb - 256;
      const int64_t per = (total / sms) / run * run;
      float ms = timeit([&] { k_ring_mixed<<<sms, 512, smem>>>(src, xs, per, stages, sb, m.nx, m.xb, out); });
      printf("{\"variant\":\"ring_mixed\",\"nx\":%d,\"xb\":%d,\"data_GBps\":%.1f,\"err\":\"%s\"}\n", m.nx, m.xb,
             (double)per * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  struct W { int warps, stages, stage_kb, segs; };
  W ws[] = {{8, 3, 9, 1}, {8, 3, 9, 4}, {8, 2, 13, 1}, {16, 2, 6, 1}, {16, 3, 4, 1}, {4, 4, 13, 1}, {8, 4, 6, 1}};
  for (const W& w : ws) {
    const int sb = w.stage_kb * 1024;
    const int smem = 1024 + w.warps * w.stages * sb;
    if (smem > 227 * 1024) continue;
    cudaFuncSetAttribute(k_warpring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int64_t per = (total / (sms * w.warps)) / sb * sb;
    float ms = timeit([&] { k_warpring<<<sms, w.warps * 32, smem>>>(src, per, w.stages, sb, w.segs, out); });
    printf("{\"variant\":\"warpring\",\"warps\":%d,\"stages\":%d,\"stage_kb\":%d,\"segs\":%d,\"GBps\":%.1f,\"err\":\"%s\"}\n",
           w.warps, w.stages, w.stage_kb, w.segs, (double)per * sms * w.warps / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
