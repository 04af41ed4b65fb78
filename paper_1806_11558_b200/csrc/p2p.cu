// p2p.cu — the sharded solve's collectives as libhm kernels over NVLink peer memory (SURVEY
// §8(f)-4: "a fused NVLink P2P ... reduce-scatter in the matvec epilogue instead of NCCL";
// the paper's per-product global sum, and the dot-product reductions of the
// Krylov solver).
//
// Every rank allocates one exchange buffer and exports it as a CUDA IPC handle; the caller
// gathers the handles (torch process group = plumbing) and hands them to hm_p2p_import, which
// maps every peer's buffer into this process.  Buffer layout (bytes, F = capacity in doubles):
//   [0, 8F)            xfull  — the gathered x of the sharded matvec (rank q's slice at q S)
//   [8F, 16F)          ypart  — this rank's partial product over its own leaves (length N)
//   [16F, +2 p 1024 8) ar     — dot-product partials, two phases [e & 1][q][1024]
//   then               flags  — [3 kinds][kMaxPeers] u64 epochs written by the peers
//   then               ticket — u32, last-block detection of the all-gather kernel
// Synchronisation: monotonically increasing epochs per kind (identical on all ranks, which
// issue the same sequence of collectives); a producer makes its data visible with a
// system-scope fence and then stores the epoch into every peer's flag slot with st.release.sys;
// a consumer spins with ld.acquire.sys until all p flags reach the epoch.  Reuse hazards:
//   * xfull / ypart: rank q writes my xfull (epoch e + 1) only after its reduce-scatter e,
//     which waited for my "ypart e ready" flag, raised after my matvec e had read xfull; my
//     ypart is rewritten by my matvec e + 1 only after my all-gather e + 1, which waits for q's
//     all-gather e + 1, issued after q's reduce-scatter e had read my ypart.
//   * ar: two phases (epoch parity); a peer can be at most one all-reduce ahead.
//   * the solution gather at the end of a solve goes to ypart, not xfull: nothing orders it
//     against a peer's first all-gather of its next solve, but the solve's last collective
//     is an all-reduce (true residual), after which no rank reads any ypart of that product.
// Sums run over q = 0 .. p-1 in rank order, so every rank obtains bit-identical scalars.

#include <cstring>

#include "hm_internal.cuh"

namespace hm {

namespace {

constexpr int kArSlot = 1024;   // doubles per rank per phase (>= restart + 2 for restart <= 1000)
enum { FL_AG = 0, FL_RS = 1, FL_AR = 2 };

struct Peers {
  char* base[kMaxPeers];
  int p, r;
  int64_t F;
};

__device__ __forceinline__ size_t off_ar(int64_t F) { return (size_t)16 * F; }
__device__ __forceinline__ size_t off_flags(int64_t F, int p) { return off_ar(F) + (size_t)2 * p * kArSlot * 8; }
__device__ __forceinline__ unsigned long long* flag(const Peers& P, int q, int kind, int from) {
  return reinterpret_cast<unsigned long long*>(P.base[q] + off_flags(P.F, P.p)) + kind * kMaxPeers + from;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
// raise my flag of `kind` on every rank, then wait until every rank raised its flag on mine
__device__ void signal_and_wait(const Peers& P, int kind, unsigned long long epoch) {
  __threadfence_system();
  for (int q = 0; q < P.p; ++q) st_release_sys(flag(P, q, kind, P.r), epoch);
  for (int q = 0; q < P.p; ++q)
    while (ld_acquire_sys(flag(P, P.r, kind, q)) < epoch) __nanosleep(64);
}

// all-gather: x (this rank's n-long slice) -> region[r S + t] on every rank (region 0: xfull,
// F: ypart); the last block to finish raises the flags and waits for the peers' (the kernel
// ends when the gathered vector is complete)
__global__ void __launch_bounds__(256) k_p2p_allgather(Peers P, const double* __restrict__ x, int64_t n, int64_t S,
                                                       int64_t region, unsigned long long epoch) {
  __shared__ bool last;
  const int64_t o = region + (int64_t)P.r * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[t];
    for (int q = 0; q < P.p; ++q) reinterpret_cast<double*>(P.base[q])[o + t] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ticket = reinterpret_cast<unsigned*>(P.base[P.r] + off_flags(P.F, P.p) + 3 * kMaxPeers * 8);
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (last) {
      *ticket = 0;
      signal_and_wait(P, FL_AG, epoch);
    }
  }
}

// Fused normalisation + all-gather (GMRES: v = w / h for the next product): out[t] = a[t] / *s
// for this rank's slice, and the same value stored into every rank's xfull at r S + t, then the
// all-gather's flags — the product that follows reads xfull without a separate all-gather.
__global__ void __launch_bounds__(256) k_p2p_scale_publish(Peers P, const double* __restrict__ a,
                                                           const double* __restrict__ sden, double* __restrict__ out,
                                                           int64_t n, int64_t S, unsigned long long epoch) {
  __shared__ bool last;
  const double f = 1.0 / *sden;
  const int64_t o = (int64_t)P.r * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = a[t] * f;
    out[t] = v;
    for (int q = 0; q < P.p; ++q) reinterpret_cast<double*>(P.base[q])[o + t] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ticket = reinterpret_cast<unsigned*>(P.base[P.r] + off_flags(P.F, P.p) + 3 * kMaxPeers * 8);
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (last) {
      *ticket = 0;
      signal_and_wait(P, FL_AG, epoch);
    }
  }
}

// reduce-scatter: y[t] = sum_q ypart_q[r S + t] (q ascending) once every rank's ypart is final
__global__ void __launch_bounds__(256) k_p2p_reduce_scatter(Peers P, double* __restrict__ y, int64_t n, int64_t S,
                                                            unsigned long long epoch) {
  if (threadIdx.x == 0) signal_and_wait(P, FL_RS, epoch);   // every block: idempotent stores
  __syncthreads();
  const int64_t o = P.F + (int64_t)P.r * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P.p; ++q) s += __ldcg(reinterpret_cast<const double*>(P.base[q]) + o + t);
    y[t] = s;
  }
}

// all-reduce of n <= kArSlot doubles, one block: partials to every rank's phase slot, flags,
// then the rank-ordered sum
__global__ void __launch_bounds__(256) k_p2p_allreduce(Peers P, double* __restrict__ buf, int n,
                                                       unsigned long long epoch) {
  const size_t ph = (size_t)(epoch & 1) * P.p * kArSlot;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = buf[i];
    for (int q = 0; q < P.p; ++q)
      reinterpret_cast<double*>(P.base[q] + off_ar(P.F))[ph + (size_t)P.r * kArSlot + i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) signal_and_wait(P, FL_AR, epoch);
  __syncthreads();
  const double* mine = reinterpret_cast<const double*>(P.base[P.r] + off_ar(P.F)) + ph;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P.p; ++q) s += __ldcg(mine + (size_t)q * kArSlot + i);
    buf[i] = s;
  }
}

Peers peers(const Context& C) {
  Peers P;
  std::memset(&P, 0, sizeof(P));
  for (int q = 0; q < C.world; ++q) P.base[q] = C.p2p.peer[q];
  P.p = C.world;
  P.r = C.rank;
  P.F = C.p2p.F;
  return P;
}

size_t buffer_bytes(int64_t F, int p) {
  return (size_t)16 * F + (size_t)2 * p * kArSlot * 8 + 3 * kMaxPeers * 8 + 64;
}

}  // namespace

bool p2p_on(const Context& C) { return C.world > 1 && C.p2p.ready && C.solve_comm == 1; }

double* p2p_xfull(Context& C) { return reinterpret_cast<double*>(C.p2p.peer[C.rank]); }
double* p2p_ypart(Context& C) { return reinterpret_cast<double*>(C.p2p.peer[C.rank]) + C.p2p.F; }

void p2p_export(Context& C, int64_t n_max, void* handle_out) {
  if (C.world < 2 || C.world > kMaxPeers) fail(HM_ERR_STATE, "hm_p2p_export: needs 2 <= world_size <= 8");
  if (C.p2p.own) fail(HM_ERR_STATE, "hm_p2p_export: already exported");
  if (n_max < 1) fail(HM_ERR_ARG, "hm_p2p_export: n_max must be >= 1");
  const int64_t S = (n_max + C.world - 1) / C.world;
  const int64_t F = S * C.world + 32;
  const size_t bytes = buffer_bytes(F, C.world);
  void* p = nullptr;
  HM_CUDA(cudaMalloc(&p, bytes));
  HM_CUDA(cudaMemset(p, 0, bytes));
  HM_CUDA(cudaDeviceSynchronize());
  C.p2p.own = static_cast<char*>(p);
  C.p2p.F = F;
  C.p2p.n_max = n_max;
  cudaIpcMemHandle_t h;
  HM_CUDA(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(h) == HM_P2P_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
}

void p2p_import(Context& C, const void* handles) {
  if (!C.p2p.own) fail(HM_ERR_STATE, "hm_p2p_import: call hm_p2p_export first");
  if (C.p2p.ready) fail(HM_ERR_STATE, "hm_p2p_import: already imported");
  const char* hb = static_cast<const char*>(handles);
  for (int q = 0; q < C.world; ++q) {
    if (q == C.rank) {
      C.p2p.peer[q] = C.p2p.own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)q * HM_P2P_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    HM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    C.p2p.peer[q] = static_cast<char*>(p);
    C.p2p.opened[q] = true;
  }
  C.p2p.ready = true;
  C.solve_comm = 1;
}

void p2p_release(Context& C) {
  for (int q = 0; q < kMaxPeers; ++q)
    if (C.p2p.opened[q]) cudaIpcCloseMemHandle(C.p2p.peer[q]);
  if (C.p2p.own) cudaFree(C.p2p.own);
  C.p2p = P2PState{};
}

void p2p_check_capacity(Context& C, int64_t S) {
  if (S * C.world + 32 > C.p2p.F)
    fail(HM_ERR_STATE, "hm_solve: N = " + std::to_string(C.N) + " exceeds the P2P exchange buffer (n_max = " +
                           std::to_string(C.p2p.n_max) + "); export a larger one or set option solve_comm = 0");
}

void p2p_allgather(Context& C, const double* x, int64_t n, int64_t S, bool into_ypart) {
  KScope ks(C, KF_COMM);
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(n, 256), 148 * 4));
  k_p2p_allgather<<<g, 256, 0, C.stream>>>(peers(C), x, n, S, into_ypart ? C.p2p.F : 0, ++C.p2p.ep_ag);
  HM_CHECK_LAUNCH();
}

void p2p_scale_publish(Context& C, const double* a, const double* sden, double* out, int64_t n, int64_t S) {
  KScope ks(C, KF_COMM);
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(n, 256), 148 * 4));
  k_p2p_scale_publish<<<g, 256, 0, C.stream>>>(peers(C), a, sden, out, n, S, ++C.p2p.ep_ag);
  HM_CHECK_LAUNCH();
}

void p2p_reduce_scatter(Context& C, double* y, int64_t n, int64_t S) {
  KScope ks(C, KF_COMM);
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(n, 256), 148 * 4));
  k_p2p_reduce_scatter<<<g, 256, 0, C.stream>>>(peers(C), y, n, S, ++C.p2p.ep_rs);
  HM_CHECK_LAUNCH();
}

void p2p_allreduce(Context& C, double* buf, int64_t n) {
  KScope ks(C, KF_COMM);
  for (int64_t i = 0; i < n; i += kArSlot) {
    k_p2p_allreduce<<<1, 256, 0, C.stream>>>(peers(C), buf + i, (int)std::min<int64_t>(kArSlot, n - i),
                                             ++C.p2p.ep_ar);
    HM_CHECK_LAUNCH();
  }
}

}  // namespace hm
