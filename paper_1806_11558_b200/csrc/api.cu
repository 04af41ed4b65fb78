// api.cu — the extern "C" boundary of libhm (include/hm.h), the VMM factor pool and the
// NCCL plumbing.  Every entry point converts internal exceptions to an hm_status and a
// message retrievable with hm_last_error.
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <thread>
#include <sstream>

#include "entry.cuh"

using hm::Context;

struct hm_ctx_s {
  Context C;
};

namespace hm {

unsigned long long g_launches = 0;

// ---- driver entry points (no link-time dependency on libcuda: resolved through cudart) ----
namespace {
struct Drv {
  PFN_cuMemGetAllocationGranularity_v10020 gran = nullptr;
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemAddressFree_v10020 vfree = nullptr;
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemRelease_v10020 rel = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 access = nullptr;
  PFN_cuGetErrorString_v6000 errstr = nullptr;
};
Drv& drv() {
  static Drv d;
  static bool loaded = false;
  if (!loaded) {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      HM_CUDA(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !*fn) fail(HM_ERR_CUDA, std::string("driver symbol missing: ") + name);
    };
    get("cuMemGetAllocationGranularity", (void**)&d.gran);
    get("cuMemAddressReserve", (void**)&d.reserve);
    get("cuMemAddressFree", (void**)&d.vfree);
    get("cuMemCreate", (void**)&d.create);
    get("cuMemRelease", (void**)&d.rel);
    get("cuMemMap", (void**)&d.map);
    get("cuMemUnmap", (void**)&d.unmap);
    get("cuMemSetAccess", (void**)&d.access);
    get("cuGetErrorString", (void**)&d.errstr);
    loaded = true;
  }
  return d;
}
void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  if (drv().errstr) drv().errstr(r, &s);
  throw Error{r == CUDA_ERROR_OUT_OF_MEMORY ? HM_ERR_OOM : HM_ERR_CUDA, std::string(what) + ": " + (s ? s : "?")};
}
}  // namespace

// ---- VMM pool -------------------------------------------------------------------------
void VmmPool::init(int dev, size_t max_bytes) {
  release();
  device = dev;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  cu_check(drv().gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  if (gran == 0) gran = 2u << 20;
  reserved = ((max_bytes + gran - 1) / gran) * gran;
  cu_check(drv().reserve(&base, reserved, 0, 0, 0), "cuMemAddressReserve");
  mapped = used = 0;
}

void VmmPool::ensure(size_t bytes) {
  if (bytes <= mapped) return;
  if (bytes > reserved) fail(HM_ERR_OOM, "factor pool exceeds its reserved range");
  size_t chunk = std::max(((bytes - mapped + gran - 1) / gran) * gran, std::min(reserved - mapped, (size_t)256 << 20));
  chunk = std::min(chunk, reserved - mapped);
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  CUmemGenericAllocationHandle h;
  cu_check(drv().create(&h, chunk, &prop, 0), "cuMemCreate");
  CUresult r = drv().map(base + mapped, chunk, 0, h, 0);
  if (r != CUDA_SUCCESS) { drv().rel(h); cu_check(r, "cuMemMap"); }
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(drv().access(base + mapped, chunk, &acc, 1), "cuMemSetAccess");
  handles.push_back(h);
  sizes.push_back(chunk);
  mapped += chunk;
}

void VmmPool::release() {
  if (!base) return;
  cudaDeviceSynchronize();
  size_t off = 0;
  for (size_t i = 0; i < handles.size(); ++i) {
    drv().unmap(base + off, sizes[i]);
    drv().rel(handles[i]);
    off += sizes[i];
  }
  drv().vfree(base, reserved);
  handles.clear(); sizes.clear();
  base = 0; reserved = mapped = used = 0;
}

__global__ void k_seg_table(const int64_t* __restrict__ pre, int64_t nseg, int64_t e0, int32_t* __restrict__ tab) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= nseg) return;
  const int64_t lo = pre[a] - e0, hi = pre[a + 1] - e0;
  for (int64_t w = (lo + 31) >> 5; (w << 5) < hi; ++w) tab[w] = (int32_t)a;
}

// ---- kernel-family timers -------------------------------------------------------------------
cudaEvent_t KTimer::get() {
  if (pool.empty()) {
    cudaEvent_t e;
    HM_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = pool.back();
  pool.pop_back();
  return e;
}
void KTimer::mark(cudaStream_t st) {
  if (!on) return;
  if (!ref) ref = get();
  cudaEventRecord(ref, st);
}
void KTimer::adopt(KTimer& o) {
  pend.insert(pend.end(), o.pend.begin(), o.pend.end());
  o.pend.clear();
}
void KTimer::resolve() {
  std::vector<std::pair<double, double>> ev;   // eval-family intervals from ref
  double ev_sum = 0;
  for (auto& p : pend) {
    float t = 0;
    if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
      ms[p.fam] += t;
      n[p.fam] += 1;
      if (p.fam == KF_EVAL_NEAR || p.fam == KF_EVAL_ACA) {
        ev_sum += t;
        float t0 = 0;
        if (ref && cudaEventElapsedTime(&t0, ref, p.a) == cudaSuccess) ev.emplace_back(t0, (double)t0 + t);
        else cudaGetLastError();
      }
    } else {
      cudaGetLastError();
    }
    pool.push_back(p.a);
    pool.push_back(p.b);
  }
  pend.clear();
  if (ref && ev.size()) {   // union of the intervals
    std::sort(ev.begin(), ev.end());
    double u = 0, lo = ev[0].first, hi = ev[0].second;
    for (auto& iv : ev) {
      if (iv.first > hi) { u += hi - lo; lo = iv.first; hi = iv.second; }
      else hi = std::max(hi, iv.second);
    }
    eval_union_ms += u + (hi - lo);
  } else {
    eval_union_ms += ev_sum;
  }
  if (ref) { pool.push_back(ref); ref = nullptr; }
}
void KTimer::reset() {
  for (int f = 0; f < KF_NUM; ++f) { ms[f] = 0; n[f] = 0; }
  eval_union_ms = 0;
}
KTimer::~KTimer() {
  for (auto& p : pend) { pool.push_back(p.a); pool.push_back(p.b); }
  if (ref) pool.push_back(ref);
  for (auto e : pool) cudaEventDestroy(e);
}

// ---- NCCL ---------------------------------------------------------------------------------
void allreduce_sum(Context& C, double* buf, int64_t n) {
  KScope ks(C, KF_COMM);
  HM_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, C.comm, C.stream));
}

}  // namespace hm

namespace {

template <class F>
hm_status guarded(hm_ctx ctx, F&& f) {
  if (!ctx) return HM_ERR_ARG;
  try {
    ctx->C.err.clear();
    HM_CUDA(cudaSetDevice(ctx->C.device));
    f(ctx->C);
    return HM_OK;
  } catch (const hm::Error& e) {
    ctx->C.err = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    ctx->C.err = "host allocation failed";
    return HM_ERR_OOM;
  } catch (const std::exception& e) {
    ctx->C.err = e.what();
    return HM_ERR_ARG;
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Timer {
  Context& C;
  cudaEvent_t a, b;
  explicit Timer(Context& c) : C(c) {
    HM_CUDA(cudaEventCreate(&a));
    HM_CUDA(cudaEventCreate(&b));
    HM_CUDA(cudaEventRecord(a, C.stream));
  }
  double ms() {
    float t = 0;
    HM_CUDA(cudaEventRecord(b, C.stream));
    HM_CUDA(cudaEventSynchronize(b));
    HM_CUDA(cudaEventElapsedTime(&t, a, b));
    return t;
  }
  ~Timer() { cudaEventDestroy(a); cudaEventDestroy(b); }
};

void need_tree(Context& C) { if (!C.have_tree) hm::fail(HM_ERR_STATE, "no tree: call hm_build_tree first"); }
void need_setup(Context& C) { if (!C.have_setup) hm::fail(HM_ERR_STATE, "no H-matrix: call hm_setup first"); }

// Host/device staging of an N-vector argument
struct Vec {
  Context& C;
  const double* src;
  double* dst;
  bool host;
  hm::DBuf<double>* buf;
  Vec(Context& c, hm::DBuf<double>& b, const double* in, double* out) : C(c), src(in), dst(out), buf(&b) {
    host = !is_device_ptr(in ? (const void*)in : (const void*)out);
    if (host) {
      buf->alloc(C.N);
      if (in)
        HM_CUDA(cudaMemcpyAsync(buf->get(), in, C.N * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    }
  }
  const double* in() const { return host ? buf->get() : src; }
  double* out() const { return host ? buf->get() : dst; }
  void finish() {
    if (host && dst) {
      HM_CUDA(cudaMemcpyAsync(dst, buf->get(), C.N * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
      HM_CUDA(cudaStreamSynchronize(C.stream));
    }
  }
};

}  // namespace

extern "C" {

hm_status hm_nccl_unique_id(void* id_out) {
  if (!id_out) return HM_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return HM_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return HM_OK;
}

hm_status hm_create(hm_ctx* out, int device, int rank, int world_size, const void* nccl_unique_id,
                    void* cuda_stream) {
  if (!out) return HM_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) { cudaGetLastError(); return HM_ERR_CUDA; }
  if (device < 0 || device >= ndev || world_size < 1 || rank < 0 || rank >= world_size) return HM_ERR_ARG;
  if (world_size > 1 && !nccl_unique_id) return HM_ERR_ARG;
  hm_ctx ctx = new (std::nothrow) hm_ctx_s;
  if (!ctx) return HM_ERR_OOM;
  ctx->C.device = device;
  ctx->C.rank = rank;
  ctx->C.world = world_size;
  hm_status s = guarded(ctx, [&](Context& C) {
    if (cuda_stream) {
      C.stream = (cudaStream_t)cuda_stream;
    } else {
      HM_CUDA(cudaStreamCreate(&C.stream));   // blocking: ordered with the legacy default stream
      C.own_stream = true;
    }
    if (world_size > 1) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof(id));
      HM_NCCL(ncclCommInitRank(&C.comm, world_size, id, rank));
    }
    hm::upload_quadrature_tables();
  });
  if (s != HM_OK) {
    delete ctx;
    return s;
  }
  *out = ctx;
  return HM_OK;
}

hm_status hm_p2p_export(hm_ctx ctx, int64_t n_max, void* handle_out) {
  return guarded(ctx, [&](Context& C) {
    if (!handle_out) hm::fail(HM_ERR_ARG, "hm_p2p_export: NULL handle_out");
    hm::p2p_export(C, n_max, handle_out);
  });
}

hm_status hm_p2p_import(hm_ctx ctx, const void* handles) {
  return guarded(ctx, [&](Context& C) {
    if (!handles) hm::fail(HM_ERR_ARG, "hm_p2p_import: NULL handles");
    hm::p2p_import(C, handles);
  });
}

hm_status hm_destroy(hm_ctx ctx) {
  if (!ctx) return HM_OK;
  cudaSetDevice(ctx->C.device);
  if (ctx->C.stream) cudaStreamSynchronize(ctx->C.stream);
  hm::p2p_release(ctx->C);
  if (ctx->C.comm) ncclCommDestroy(ctx->C.comm);
  bool own = ctx->C.own_stream;
  cudaStream_t st = ctx->C.stream;
  {
    hm::Context& C = ctx->C;
    if (C.s_hi) { cudaStreamSynchronize(C.s_hi); cudaStreamDestroy(C.s_hi); }
    if (C.s_lo) { cudaStreamSynchronize(C.s_lo); cudaStreamDestroy(C.s_lo); }
    for (cudaEvent_t e : {C.ev_fork, C.ev_join[0], C.ev_join[1], C.mv_ev[0], C.mv_ev[1]}) if (e) cudaEventDestroy(e);
    if (C.mv_side) { cudaStreamSynchronize(C.mv_side); cudaStreamDestroy(C.mv_side); }
  }
  delete ctx;
  if (own && st) cudaStreamDestroy(st);
  return HM_OK;
}

const char* hm_last_error(hm_ctx ctx) { return ctx ? ctx->C.err.c_str() : "null context"; }

hm_status hm_set_option(hm_ctx ctx, const char* key, double v) {
  return guarded(ctx, [&](Context& C) {
    std::string k = key ? key : "";
    auto bad = [&]() { hm::fail(HM_ERR_ARG, "hm_set_option: bad value for " + k); };
    if (!std::isfinite(v)) bad();
    if (k == "k_max") { if (v < 1 || v > 256) bad(); C.k_max = (int)v; }
    else if (k == "solver") { if (v != 0 && v != 1) bad(); C.solver = (int)v; }
    else if (k == "restart") { if (v < 1 || v > 1000) bad(); C.restart = (int)v; }
    else if (k == "max_iter") { if (v < 1) bad(); C.max_iter = (int)v; }
    else if (k == "aca_chunk_mb") { if (v < 1) bad(); C.aca_chunk_mb = v; }
    else if (k == "aca_kws") { if (v < 1 || v > 256) bad(); C.aca_kws = v; }
    else if (k == "lr_f32") { if (v != 0 && v != 1) bad(); C.lr_f32 = (int)v; }
    else if (k == "aca_upd_occ") { if (v < 0 || v > 2) bad(); C.aca_upd_occ = (int)v; }
    else if (k == "cost_model") { if (v != 0 && v != 1 && v != 2) bad(); C.cost_model = (int)v; }
    else if (k == "part_ranks") { if (v < 1 || v > 4096) bad(); C.part_ranks = (int)v; }
    else if (k == "part_rank") { if (v < 0 || v > 4095) bad(); C.part_rank = (int)v; }
    else if (k == "record_pivots") { if (v != 0 && v != 1 && v != -1) bad(); C.record_pivots = (int)v; }
    else if (k == "mv_kernel") { if (v < 0 || v > 5) bad(); C.mv_kind = (int)v; if (C.have_setup) hm::plan_matvec(C); }
    else if (k == "mv_profile") {
      if (v != 0 && v != 1) bad();
      if (v == 1) { C.mv_prof.alloc(4); HM_CUDA(cudaMemsetAsync(C.mv_prof.get(), 0, 32, C.stream)); }
      else C.mv_prof.release();
    }
    else if (k == "mv_small_max") { if (v < 0 || v > 49152) bad(); C.mv_small_max = (int)v; if (C.have_setup) hm::plan_matvec(C); }
    else if (k == "mv_scramble") { if (v != 0 && v != 1) bad(); C.mv_scramble = (int)v; }
    else if (k == "setup_overlap") { if (v != 0 && v != 1) bad(); C.setup_overlap = (int)v; }
    else if (k == "near_perf") { if (v != 0 && v != 1) bad(); C.near_perf = (int)v; }
    else if (k == "aca_perf") { if (v != 0 && v != 1) bad(); C.aca_perf = (int)v; }
    else if (k == "solve_comm") {
      if (v != 0 && v != 1) bad();
      if (v == 1 && !C.p2p.ready) hm::fail(HM_ERR_STATE, "option solve_comm = 1 needs hm_p2p_import");
      C.solve_comm = (int)v;
    }
    else if (k == "mv_concurrent") { if (v != 0 && v != 1) bad(); C.mv_concurrent = (int)v; }
    else if (k == "kernel_timing") {
      if (v != 0 && v != 1) bad();
      HM_CUDA(cudaStreamSynchronize(C.stream));
      C.kt.resolve();
      C.kt.reset();
      C.kt.on = v == 1;
    }
    else hm::fail(HM_ERR_ARG, "hm_set_option: unknown key '" + k + "'");
  });
}

hm_status hm_get_option(hm_ctx ctx, const char* key, double* v) {
  return guarded(ctx, [&](Context& C) {
    std::string k = key ? key : "";
    if (!v) hm::fail(HM_ERR_ARG, "null value pointer");
    if (k == "k_max") *v = C.k_max;
    else if (k == "solver") *v = C.solver;
    else if (k == "restart") *v = C.restart;
    else if (k == "max_iter") *v = C.max_iter;
    else if (k == "aca_chunk_mb") *v = C.aca_chunk_mb;
    else if (k == "aca_kws") *v = C.aca_kws;
    else if (k == "lr_f32") *v = C.lr_f32;
    else if (k == "aca_upd_occ") *v = C.aca_upd_occ;
    else if (k == "cost_model") *v = C.cost_model;
    else if (k == "part_ranks") *v = C.part_ranks;
    else if (k == "part_rank") *v = C.part_rank;
    else if (k == "record_pivots") *v = C.record_pivots;
    else if (k == "kernel_timing") *v = C.kt.on ? 1 : 0;
    else if (k == "mv_kernel") *v = C.mv_kind;
    else if (k == "setup_overlap") *v = C.setup_overlap;
    else if (k == "solve_comm") *v = C.solve_comm;
    else if (k == "near_perf") *v = C.near_perf;
    else if (k == "aca_perf") *v = C.aca_perf;
    else if (k == "mv_concurrent") *v = C.mv_concurrent;
    else hm::fail(HM_ERR_ARG, "hm_get_option: unknown key '" + k + "'");
  });
}

hm_status hm_build_tree(hm_ctx ctx, const hm_mesh* mesh, int leaf_size, double eta) {
  return guarded(ctx, [&](Context& C) {
    if (!mesh || !mesh->vertices || !mesh->triangles) hm::fail(HM_ERR_ARG, "hm_build_tree: null mesh");
    if (leaf_size < 1) hm::fail(HM_ERR_ARG, "hm_build_tree: leaf_size < 1");
    if (!(eta >= 0) || !std::isfinite(eta)) hm::fail(HM_ERR_ARG, "hm_build_tree: eta must be finite and >= 0");
    if (mesh->panel_vertices != 0 && mesh->panel_vertices != 3 && mesh->panel_vertices != 4)
      hm::fail(HM_ERR_ARG, "hm_build_tree: panel_vertices must be 0, 3 or 4");
    if (mesh->n_triangles < 1 || mesh->n_triangles > (1LL << 30) || mesh->n_vertices < 3)
      hm::fail(HM_ERR_ARG, "hm_build_tree: bad mesh sizes");
    if (mesh->panel_vertices == 4 && mesh->n_triangles > (1LL << 29))
      hm::fail(HM_ERR_ARG, "hm_build_tree: at most 2^29 quadrilaterals");
    C.have_setup = false;
    Timer t(C);
    hm::build_tree(C, *mesh, leaf_size, eta);
    C.times.tree_ms = t.ms();
  });
}

// Near field beside ACA: the near-field evaluation (a few tens of launches of long FP64
// kernels) runs on a least-priority stream from its own host thread while ACA's lock-step
// loop drives a greatest-priority stream, so the near-field CTAs fill the SM time ACA leaves
// idle (its pivot/update/compaction launches, host round trips and chunk tails) and yield
// to every ACA launch.  Both write disjoint storage; results are identical to the serial
// order.  The matvec plan (host work + upload; it needs ACA's ranks, not the near-field
// values) is built while the near-field tail still runs.  near_ms is the near-field thread's
// own span, aca_ms ACA's.
static void run_overlapped(Context& C) {
  if (!C.s_hi) {
    int least = 0, greatest = 0;
    HM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    HM_CUDA(cudaStreamCreateWithPriority(&C.s_hi, cudaStreamNonBlocking, greatest));
    HM_CUDA(cudaStreamCreateWithPriority(&C.s_lo, cudaStreamNonBlocking, least));
    HM_CUDA(cudaEventCreateWithFlags(&C.ev_fork, cudaEventDisableTiming));
    HM_CUDA(cudaEventCreateWithFlags(&C.ev_join[0], cudaEventDisableTiming));
    HM_CUDA(cudaEventCreateWithFlags(&C.ev_join[1], cudaEventDisableTiming));
  }
  HM_CUDA(cudaEventRecord(C.ev_fork, C.stream));
  HM_CUDA(cudaStreamWaitEvent(C.s_hi, C.ev_fork, 0));
  HM_CUDA(cudaStreamWaitEvent(C.s_lo, C.ev_fork, 0));
  C.kt.mark(C.stream);
  C.kt_near.on = C.kt.on;
  std::exception_ptr near_err;
  std::thread th([&C, &near_err]() {
    try {
      HM_CUDA(cudaSetDevice(C.device));
      const auto t0 = std::chrono::steady_clock::now();
      hm::near_eval(C, C.s_lo, C.kt_near);
      C.near_eval_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } catch (...) {
      near_err = std::current_exception();
    }
  });
  cudaStream_t user = C.stream;
  C.stream = C.s_hi;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    hm::setup_aca(C);
  } catch (...) {
    C.stream = user;
    th.join();
    cudaStreamSynchronize(C.s_lo);
    throw;
  }
  HM_CUDA(cudaStreamSynchronize(C.s_hi));
  C.times.aca_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  try {
    const auto t1 = std::chrono::steady_clock::now();
    hm::plan_matvec(C);
    HM_CUDA(cudaStreamSynchronize(C.s_hi));
    C.times.plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
  } catch (...) {
    C.stream = user;
    th.join();
    cudaStreamSynchronize(C.s_lo);
    throw;
  }
  C.stream = user;
  th.join();
  if (near_err) std::rethrow_exception(near_err);
  C.times.near_ms = C.near_eval_ms;
  HM_CUDA(cudaEventRecord(C.ev_join[0], C.s_hi));
  HM_CUDA(cudaEventRecord(C.ev_join[1], C.s_lo));
  HM_CUDA(cudaStreamWaitEvent(C.stream, C.ev_join[0], 0));
  HM_CUDA(cudaStreamWaitEvent(C.stream, C.ev_join[1], 0));
  C.kt.adopt(C.kt_near);
}

hm_status hm_setup(hm_ctx ctx, double eps_aca) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (!(eps_aca >= 0) || !std::isfinite(eps_aca)) hm::fail(HM_ERR_ARG, "hm_setup: eps_aca must be finite and >= 0");
    C.have_setup = false;
    C.eps_aca = eps_aca;
    Timer all(C);
    struct JoinPlanner {   // on any failure below: no planner thread outlives this call
      Context& c;
      bool armed = true;
      ~JoinPlanner() { if (armed) hm::plan_dense_abort(c); }
    } join_planner{C};
    hm::near_prepare(C);
    hm::plan_dense_begin(C);
    if (C.setup_overlap && C.dense_doubles > 0) {
      run_overlapped(C);               // near field beside ACA, plan beside the near-field tail
      hm::near_check(C);
    } else {
      {
        Timer t(C);
        hm::near_eval(C, C.stream, C.kt);
        C.times.near_ms = t.ms();
      }
      {
        Timer t(C);
        hm::setup_aca(C);
        C.times.aca_ms = t.ms();
      }
      hm::near_check(C);
      Timer t(C);
      hm::plan_matvec(C);
      C.times.plan_ms = t.ms();
    }
    join_planner.armed = false;
    C.times.setup_ms = all.ms();
    C.kt.resolve();
    C.have_setup = true;
  });
}

hm_status hm_matvec(hm_ctx ctx, const double* x, double* y) {
  return guarded(ctx, [&](Context& C) {
    need_setup(C);
    if (!x || !y || (const void*)x == (const void*)y) hm::fail(HM_ERR_ARG, "hm_matvec: bad x/y");
    Vec vx(C, C.xapp, x, nullptr);
    Vec vy(C, C.yapp, nullptr, y);
    C.xin.alloc(C.N);
    C.yin.alloc(C.N);
    hm::gather_perm(C, vx.in(), C.xin.get());
    hm::matvec_internal(C, C.xin.get(), C.yin.get());
    hm::scatter_perm(C, C.yin.get(), vy.out());
    vy.finish();
  });
}

hm_status hm_solve(hm_ctx ctx, const double* rhs, double* sol, double tol, int* iters_out,
                   double* rel_residual_out) {
  return guarded(ctx, [&](Context& C) {
    need_setup(C);
    if (!rhs || !sol) hm::fail(HM_ERR_ARG, "hm_solve: null vector");
    if (!(tol > 0) || !std::isfinite(tol)) hm::fail(HM_ERR_ARG, "hm_solve: tol must be > 0");
    Timer t(C);
    Vec vb(C, C.xapp, rhs, nullptr);
    Vec vx(C, C.yapp, nullptr, sol);
    C.xin.alloc(C.N);
    C.yin.alloc(C.N);
    hm::gather_perm(C, vb.in(), C.xin.get());
    int it = 0;
    double rr = 0;
    hm::solve(C, C.xin.get(), C.yin.get(), tol, &it, &rr);
    hm::scatter_perm(C, C.yin.get(), vx.out());
    vx.finish();
    C.times.solve_ms = t.ms();
    C.kt.resolve();
    C.times.solve_iters = it;
    C.times.solve_relres = rr;
    if (iters_out) *iters_out = it;
    if (rel_residual_out) *rel_residual_out = rr;
  });
}

hm_status hm_potential(hm_ctx ctx, const double* sol, int64_t m, const double* points, double* out) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (!sol || m < 0 || (m > 0 && (!points || !out))) hm::fail(HM_ERR_ARG, "hm_potential: bad arguments");
    if (m == 0) return;
    Vec va(C, C.xapp, sol, nullptr);
    const bool hp = !is_device_ptr(points), ho = !is_device_ptr(out);
    const double* X = points;
    if (hp) {
      C.pot_x.alloc(3 * m);
      HM_CUDA(cudaMemcpyAsync(C.pot_x.get(), points, 3 * m * sizeof(double), cudaMemcpyHostToDevice, C.stream));
      X = C.pot_x.get();
    }
    double* o = out;
    if (ho) { C.pot_out.alloc(m); o = C.pot_out.get(); }
    hm::potential(C, va.in(), m, X, o);
    if (ho) HM_CUDA(cudaMemcpyAsync(out, o, m * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_assemble_rhs(hm_ctx ctx, int kind, double* f) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (!f || (kind != 0 && kind != 1)) hm::fail(HM_ERR_ARG, "hm_assemble_rhs: bad arguments");
    Vec vf(C, C.xapp, nullptr, f);
    hm::assemble_rhs(C, kind, vf.out());
    vf.finish();
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_get_perm(hm_ctx ctx, int32_t* perm) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (!perm) hm::fail(HM_ERR_ARG, "null perm");
    HM_CUDA(cudaMemcpyAsync(perm, C.perm.get(), C.N * sizeof(int32_t), cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_get_codes(hm_ctx ctx, uint64_t* codes) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (!codes) hm::fail(HM_ERR_ARG, "null codes");
    HM_CUDA(cudaMemcpyAsync(codes, C.codes_app.get(), C.N * sizeof(uint64_t), cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_get_leaves(hm_ctx ctx, int kind, int64_t* count, int32_t* quads, int64_t* ob, int64_t* oe) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (kind != 0 && kind != 1) hm::fail(HM_ERR_ARG, "kind must be 0 or 1");
    int64_t n = kind == 0 ? C.nadm : C.ndense;
    if (count) *count = n;
    if (ob) *ob = kind == 0 ? C.adm_begin : C.dense_begin;
    if (oe) *oe = kind == 0 ? C.adm_end : C.dense_end;
    if (quads && n) {
      HM_CUDA(cudaMemcpyAsync(quads, kind == 0 ? C.adm.get() : C.dense.get(), n * sizeof(hm::Quad),
                              cudaMemcpyDeviceToHost, C.stream));
      HM_CUDA(cudaStreamSynchronize(C.stream));
    }
  });
}

hm_status hm_get_clusters(hm_ctx ctx, int64_t* count, int32_t* lo, int32_t* hi, int32_t* depth, double* bbox) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (count) *count = C.ncl;
    auto cp = [&](void* dst, const void* src, size_t b) {
      if (dst) HM_CUDA(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, C.stream));
    };
    cp(lo, C.cl_lo.get(), C.ncl * 4);
    cp(hi, C.cl_hi.get(), C.ncl * 4);
    cp(depth, C.cl_depth.get(), C.ncl * 4);
    cp(bbox, C.cl_box.get(), C.ncl * 48);
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_eval_entries(hm_ctx ctx, int64_t n, const int64_t* pairs, double* out) {
  return guarded(ctx, [&](Context& C) {
    need_tree(C);
    if (n < 0 || (n > 0 && (!pairs || !out))) hm::fail(HM_ERR_ARG, "hm_eval_entries: bad arguments");
    for (int64_t e = 0; e < 2 * n; ++e)
      if (pairs[e] < 0 || pairs[e] >= C.N) hm::fail(HM_ERR_ARG, "hm_eval_entries: index out of range");
    if (n == 0) return;
    hm::DBuf<int64_t> dp;
    hm::DBuf<double> dout;
    dp.alloc(2 * n);
    dout.alloc(n);
    HM_CUDA(cudaMemcpyAsync(dp.get(), pairs, 2 * n * sizeof(int64_t), cudaMemcpyHostToDevice, C.stream));
    hm::eval_entries(C, n, dp.get(), dout.get());
    HM_CUDA(cudaMemcpyAsync(out, dout.get(), n * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_get_dense_block(hm_ctx ctx, int64_t leaf, double* block) {
  return guarded(ctx, [&](Context& C) {
    need_setup(C);
    if (leaf < C.dense_begin || leaf >= C.dense_end || !block) hm::fail(HM_ERR_ARG, "leaf not owned by this rank");
    int64_t off[2];
    HM_CUDA(cudaMemcpyAsync(off, C.doff.get() + (leaf - C.dense_begin), 2 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
    HM_CUDA(cudaMemcpyAsync(block, C.dstore.get() + off[0], (off[1] - off[0]) * sizeof(double),
                            cudaMemcpyDeviceToHost, C.stream));
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_get_lowrank(hm_ctx ctx, int64_t leaf, int32_t* k, double* U, double* V, int32_t* pivots) {
  return guarded(ctx, [&](Context& C) {
    need_setup(C);
    if (leaf < C.adm_begin || leaf >= C.adm_end) hm::fail(HM_ERR_ARG, "leaf not owned by this rank");
    const int64_t b = leaf - C.adm_begin;
    if (C.h_adm.size() != (size_t)C.nadm) hm::fail(HM_ERR_STATE, "leaf list not cached");
    const hm::Quad q = C.h_adm[leaf];
    const int64_t m = q.rhi - q.rlo, n = q.chi - q.clo;
    const int32_t kk = C.h_rank[b];
    if (k) *k = kk;
    if (C.lr_esz == 4 && kk > 0 && (U || V)) {        // binary32 factors (option lr_f32): widened exactly
      std::vector<float> f((size_t)(m + n) * kk);
      const float* base = (const float*)C.fpool.base + C.h_foff[b];
      HM_CUDA(cudaMemcpyAsync(f.data(), base, f.size() * sizeof(float), cudaMemcpyDeviceToHost, C.stream));
      HM_CUDA(cudaStreamSynchronize(C.stream));
      if (U) for (int64_t x = 0; x < m * kk; ++x) U[x] = f[x];
      if (V) for (int64_t x = 0; x < n * kk; ++x) V[x] = f[m * kk + x];
    } else {
      const double* base = (const double*)C.fpool.base + C.h_foff[b];
      if (U && kk > 0)
        HM_CUDA(cudaMemcpyAsync(U, base, m * kk * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
      if (V && kk > 0)
        HM_CUDA(cudaMemcpyAsync(V, base + m * kk, n * kk * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    }
    if (pivots) {
      if (C.h_piv.size() != (size_t)(C.adm_end - C.adm_begin)) hm::fail(HM_ERR_STATE, "pivots not recorded: set option record_pivots = 1 before hm_setup");
      std::memcpy(pivots, C.h_piv[b].data(), C.h_piv[b].size() * sizeof(int32_t));
    }
    HM_CUDA(cudaStreamSynchronize(C.stream));
  });
}

hm_status hm_quadrature_table(int n, double* nodes, double* weights) {
  if (n < 1 || n > 8 || !nodes || !weights) return HM_ERR_ARG;
  hm::quadrature_table_host(n, nodes, weights);
  return HM_OK;
}

hm_status hm_get_stats(hm_ctx ctx, char* buf, int64_t len) {
  return guarded(ctx, [&](Context& C) {
    HM_CUDA(cudaStreamSynchronize(C.stream));
    C.kt.resolve();
    std::ostringstream o;
    o.precision(17);
    int64_t kmin = 0, kmax = 0;
    double ksum = 0;
    std::vector<int64_t> hist(65, 0);
    for (size_t b = 0; b < C.h_rank.size() && C.have_setup; ++b) {
      int k = C.h_rank[b];
      ksum += k;
      kmax = std::max<int64_t>(kmax, k);
      kmin = b == 0 ? k : std::min<int64_t>(kmin, k);
      hist[std::min(k, 64)]++;
    }
    o << "{\"N\":" << C.N << ",\"rank\":" << C.rank << ",\"world\":" << C.world << ",\"leaf_size\":" << C.leaf_size
      << ",\"eta\":" << C.eta << ",\"clusters\":" << C.ncl << ",\"adm_leaves\":" << C.nadm
      << ",\"dense_leaves\":" << C.ndense << ",\"adm_owned\":[" << C.adm_begin << "," << C.adm_end << "]"
      << ",\"dense_owned\":[" << C.dense_begin << "," << C.dense_end << "]"
      << ",\"dense_doubles\":" << C.dense_doubles << ",\"factor_doubles\":" << C.factor_doubles
      << ",\"stored_bytes\":" << 8 * C.dense_doubles + (int64_t)C.lr_esz * C.factor_doubles
      << ",\"factor_bytes_per_entry\":" << C.lr_esz << ",\"eps_aca\":" << C.eps_aca
      << ",\"k_mean\":" << (C.h_rank.empty() ? 0.0 : ksum / C.h_rank.size()) << ",\"k_min\":" << kmin
      << ",\"k_max_seen\":" << kmax << ",\"evals_near\":" << C.evals_near << ",\"evals_aca\":" << C.evals_aca
      << ",\"entries_aca\":" << C.entries_aca << ",\"aca_steps\":" << C.aca_steps << ",\"aca_chunks\":" << C.aca_chunks
      << ",\"aca_overflow\":" << C.aca_overflow << ",\"aca_releases\":" << C.aca_releases << ",\"tree_ms\":" << C.times.tree_ms << ",\"tree_phase_ms\":[" << C.times.tree_phase_ms[0] << ","
      << C.times.tree_phase_ms[1] << "," << C.times.tree_phase_ms[2] << "," << C.times.tree_phase_ms[3] << ","
      << C.times.tree_phase_ms[4] << "," << C.times.tree_phase_ms[5] << "]"
      << ",\"plan_phase_ms\":[" << C.times.plan_phase_ms[0] << "," << C.times.plan_phase_ms[1] << ","
      << C.times.plan_phase_ms[2] << "]"
      << ",\"aca_phase_ms\":[" << C.times.aca_phase_ms[0] << "," << C.times.aca_phase_ms[1] << ","
      << C.times.aca_phase_ms[2] << "," << C.times.aca_phase_ms[3] << "," << C.times.aca_phase_ms[4] << ","
      << C.times.aca_phase_ms[5] << "," << C.times.aca_phase_ms[6] << "," << C.times.aca_phase_ms[7] << ","
      << C.times.aca_phase_ms[8] << "]"
      << ",\"near_ms\":" << C.times.near_ms << ",\"aca_ms\":" << C.times.aca_ms << ",\"plan_ms\":" << C.times.plan_ms
      << ",\"setup_ms\":" << C.times.setup_ms << ",\"solve_ms\":" << C.times.solve_ms
      << ",\"solve_iters\":" << C.times.solve_iters << ",\"solve_relres\":" << C.times.solve_relres
      << ",\"launches\":" << hm::g_launches << ",\"mv_batches\":" << C.mv_nbatches << ",\"mv_segs\":" << C.mv_nsegs << ",\"lr_small\":" << C.n_lr_small << ",\"lr_large\":" << C.n_lr_large << ",\"rank_hist\":[";
    for (int k = 0; k <= 64; ++k) o << (k ? "," : "") << hist[k];
    o << "]";
    if (C.mv_prof.n) {
      unsigned long long pr[4] = {0, 0, 0, 0};
      HM_CUDA(cudaMemcpy(pr, C.mv_prof.get(), sizeof(pr), cudaMemcpyDeviceToHost));
      o << ",\"mv_prof_cycles\":[" << pr[0] << "," << pr[1] << "," << pr[2] << "]";
    }
    o << ",\"kt\":{\"on\":" << (C.kt.on ? 1 : 0);
    const char* fam[hm::KF_NUM] = {"eval_near", "eval_aca", "aca_other", "matvec", "krylov", "comm"};
    for (int f = 0; f < hm::KF_NUM; ++f)
      o << ",\"" << fam[f] << "_ms\":" << C.kt.ms[f] << ",\"" << fam[f] << "_n\":" << C.kt.n[f];
    o << ",\"eval_union_ms\":" << C.kt.eval_union_ms << "}}";
    std::string s = o.str();
    if (!buf || len < (int64_t)s.size() + 1)
      hm::fail(HM_ERR_ARG, "hm_get_stats: buffer too small, need " + std::to_string(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
