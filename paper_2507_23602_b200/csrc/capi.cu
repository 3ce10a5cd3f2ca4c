// capi.cu -- C ABI (include/rsot_cuda.h) over the sm_100a evaluator kernels.
//
// Owns the device state that the reference keeps implicitly on the host:
// resident targets (TargetMeasure + the cell list that replaces the R*-tree
// of spatial_index.cpp), resident atom shards (SourceAtoms), per-context
// workspace, the stream, and the NCCL communicator for the one allreduce per
// evaluation.  NCCL is resolved with dlopen at rsot_cuda_ctx_set_comm time so
// the library coexists with the NCCL copy torch may already have loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <memory>
#include <vector>

#include "../../include/rsot_cuda.h"
#include "kernels.cuh"
#include "geodesic.cuh"
#include "refine.cuh"
#include "truncated.cuh"

using namespace rsot_cuda;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define RSOT_CK(call)                                                         \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      return fail(RSOT_CUDA_RUNTIME_ERROR,                                    \
                  std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

// ---- NCCL via dlopen -------------------------------------------------------
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t,
                            ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // RSOT_NCCL_LIBRARY picks a library explicitly; otherwise the soname,
    // which resolves to an NCCL the process has already loaded (e.g. torch's)
    const char* env = std::getenv("RSOT_NCCL_LIBRARY");
    const char* names[] = {env && *env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.handle = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.handle, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.handle, "ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.handle, "ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.handle, "ncclAllGather"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.handle, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.handle, "ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.CommDestroy;
  });
  return api;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * (n ? n : 1));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct rsot_cuda_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // workspace
  DevBuf<double> psi, b2, scal, part, partS, shiftA, atomL, atomLam, atomJ,
      atomD, partG, res, g_out, scalars_out, gathered;
  DevBuf<int> flagged;
  TruncWorkspace trunc;
  RefineWorkspace refine;
  GeoWorkspace geo;
  double* h_pinned = nullptr;  // small pinned staging for scalars
  bool timing = false;
  int precision = RSOT_CUDA_PRECISION_FP64;
  cudaEvent_t ev[8] = {};
  double last_ms[3] = {0, 0, 0};
  // CUDA graph of one dense device evaluation (prologue, both passes, split
  // reductions, the collective, finalisation: ~13 launches -> 1), replayed
  // while atoms, targets, eps and the workspace stay the same
  struct DenseGraph {
    cudaGraphExec_t exec = nullptr;
    const void* atoms = nullptr;
    const void* targets = nullptr;
    double eps = 0.0;
    size_t nq = 0, n = 0;
    uint64_t ws_key = 0;
    unsigned long long launches = 0;
    bool broken = false;  // capture failed once: stay on direct launches
  } graph;
  int vrank = 0, vworld = 1;  // rsot_cuda_ctx_set_virtual_rank (no communicator)
};

struct rsot_cuda_targets {
  rsot_cuda_ctx* ctx = nullptr;
  size_t n = 0;
  double4* y = nullptr;  // {y0, y1, y2, ln nu}
  double* nu = nullptr;
  TargetCells cells;     // cell list (built on demand for a radius)
};

struct rsot_cuda_atoms {
  rsot_cuda_ctx* ctx = nullptr;
  size_t nq = 0;
  double4* x = nullptr;  // {x0, x1, x2, m}
  AtomCells cells;       // Hilbert order (built on first truncated use)
  bool partitioned = false;  // every atom on every rank; evaluations split the work
  double mass_sum = 0.0;     // sum of the masses (bounds every gradient contribution)
  bool local = false;        // evaluated whole on this rank, never combined across ranks
};

namespace {

DeviceTargets make_dt(const rsot_cuda_targets* t) {
  DeviceTargets d;
  d.y = t->y;
  d.nu = t->nu;
  d.n = static_cast<int>(t->n);
  d.lo = make_double3(t->cells.bbox_lo[0], t->cells.bbox_lo[1], t->cells.bbox_lo[2]);
  d.hi = make_double3(t->cells.bbox_hi[0], t->cells.bbox_hi[1], t->cells.bbox_hi[2]);
  return d;
}

int set_device(rsot_cuda_ctx* ctx) {
  RSOT_CK(cudaSetDevice(ctx->device));
  return RSOT_CUDA_OK;
}

int ensure_workspace(rsot_cuda_ctx* c, size_t nq, size_t n, const DenseLaunch& p) {
  RSOT_CK(c->psi.ensure(n));
  RSOT_CK(c->b2.ensure(n));
  RSOT_CK(c->scal.ensure(kNumSlots));
  RSOT_CK(c->part.ensure(4 * 1024));
  RSOT_CK(c->partS.ensure(static_cast<size_t>(p.splitsA) * (nq ? nq : 1)));
  RSOT_CK(c->shiftA.ensure(nq));
  RSOT_CK(c->atomL.ensure(nq));
  RSOT_CK(c->atomLam.ensure(nq));
  RSOT_CK(c->atomJ.ensure(nq));
  RSOT_CK(c->atomD.ensure(nq));
  RSOT_CK(c->flagged.ensure(nq));
  RSOT_CK(c->partG.ensure(static_cast<size_t>(p.splitsB) * n));
  RSOT_CK(c->res.ensure(n + kResTail));
  RSOT_CK(c->g_out.ensure(n));
  RSOT_CK(c->scalars_out.ensure(kResTail));
  if (c->comm) RSOT_CK(c->gathered.ensure(static_cast<size_t>(c->world) * (n + kResTail)));
  return RSOT_CUDA_OK;
}

EvalBuffers buffers(rsot_cuda_ctx* c, double* g_out, double* scalars_out) {
  EvalBuffers b;
  b.psi = c->psi.p;
  b.b2 = c->b2.p;
  b.scal = c->scal.p;
  b.part = c->part.p;
  b.partS = c->partS.p;
  b.shiftA = c->shiftA.p;
  b.atomL = c->atomL.p;
  b.atomLam = c->atomLam.p;
  b.atomJ = c->atomJ.p;
  b.atomD = c->atomD.p;
  b.flagged = c->flagged.p;
  b.partG = c->partG.p;
  b.res = c->res.p;
  b.g_out = g_out ? g_out : c->g_out.p;
  b.scalars_out = scalars_out ? scalars_out : c->scalars_out.p;
  b.timing = c->timing ? c->ev : nullptr;
  return b;
}

// Enqueues this rank's share of one evaluation reading psi from b.psi
// (device): the packed partial buffer b.res = [g + nu | J + sum psi nu | D |
// pairs | empty | visited] before the cross-rank combination.
int enqueue_partial(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                    EvalBuffers& b, double eps, double cutoff, DebugOut* dbg, int cost) {
  const cudaStream_t s = c->stream;
  const DeviceTargets dt = make_dt(t);
  DeviceAtoms da{a->x, static_cast<int>(a->nq)};
  // partitioned atoms: this rank's share of the work (truncated: balanced
  // chunk ranges chosen on the device; dense / geodesic: equal atom ranges)
  int prank = 0, pworld = 1;
  if (a->partitioned) {
    if (c->comm && c->world > 1) {
      prank = c->rank;
      pworld = c->world;
    } else if (!c->comm && c->vworld > 1) {
      prank = c->vrank;
      pworld = c->vworld;
    }
  }
  const bool trunc_path = cost != RSOT_CUDA_COST_SQGEODESIC && std::isfinite(cutoff);
  if (pworld > 1 && !trunc_path) {
    size_t lo = 0, hi = 0;
    rsot_cuda_shard_range(a->nq, prank, pworld, &lo, &hi);
    da = DeviceAtoms{a->x + lo, static_cast<int>(hi - lo)};
  }
  if (b.timing) cudaEventRecord(b.timing[0], s);
  launch_prologue(dt, b, eps, s);
  if (cost == RSOT_CUDA_COST_SQGEODESIC) {
    const int rc = run_geodesic(c->geo, da, dt, b, eps, cutoff, s, g_last_error,
                                dbg ? dbg->count : nullptr, dbg ? dbg->hash : nullptr,
                                dbg ? dbg->log_s : nullptr);
    if (rc != 0) return fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error);
  } else if (std::isfinite(cutoff)) {
    // every truncated gradient contribution m_q p_qj / S_q <= m_q goes into
    // the fixed-point accumulator, whose top limb holds totals below 2^42
    if (!(a->mass_sum < 0x1p40))
      return fail(RSOT_CUDA_INVALID_ARGUMENT,
                  "truncated evaluation: total atom mass >= 2^40 exceeds the fixed-point gradient "
                  "accumulator (normalise the masses)");
    const int rc = run_truncated(c->trunc, da, a->cells, dt, t->cells, b, eps,
                                 cutoff, c->num_sms, dbg, s, g_last_error,
                                 c->precision == RSOT_CUDA_PRECISION_FP32, prank, pworld);
    if (rc != 0) return fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error);
  } else {
    const DenseLaunch plan = plan_dense(da.nq, dt.n, c->num_sms);
    launch_dense(da, dt, b, plan, eps, s);
    if (dbg) launch_dense_debug(da, dt, b, *dbg, s);
  }
  return RSOT_CUDA_OK;
}

// Enqueues one evaluation reading psi from b.psi (device) and leaving the
// final gradient / scalars in b.g_out / b.scalars_out.
int enqueue_eval(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                 EvalBuffers& b, double eps, double cutoff, DebugOut* dbg,
                 int cost = RSOT_CUDA_COST_SQEUCLIDEAN) {
  const cudaStream_t s = c->stream;
  const DeviceTargets dt = make_dt(t);
  const int rc = enqueue_partial(c, a, t, b, eps, cutoff, dbg, cost);
  if (rc) return rc;
  if (c->comm && !a->local) {
    // one collective per evaluation: every rank gathers all packed partial
    // buffers and sums them in rank order, so the result is bitwise the same
    // on every rank and run to run (independent of NCCL's ring / tree / NVLS
    // choice)
    NcclApi& api = nccl();
    const size_t len = t->n + kResTail;
    const ncclResult_t r = api.AllGather(b.res, c->gathered.p, len, ncclDouble, c->comm, s);
    if (r != ncclSuccess)
      return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("ncclAllGather: ") + api.GetErrorString(r));
    launch_rank_sum(c->gathered.p, c->world, len, b.res, s);
  }
  launch_finalize(dt, b, s);
  if (b.timing) cudaEventRecord(b.timing[5], s);
  RSOT_CK(cudaGetLastError());
  return RSOT_CUDA_OK;
}

void record_timing(rsot_cuda_ctx* c) {
  if (!c->timing) return;
  float a = 0.f, bb = 0.f, tot = 0.f;
  cudaEventElapsedTime(&a, c->ev[1], c->ev[2]);
  cudaEventElapsedTime(&bb, c->ev[3], c->ev[4]);
  cudaEventElapsedTime(&tot, c->ev[0], c->ev[5]);
  c->last_ms[0] = a;
  c->last_ms[1] = bb;
  c->last_ms[2] = tot;
}

int check_ready(rsot_cuda_ctx* ctx, rsot_cuda_atoms* a, rsot_cuda_targets* t) {
  if (!ctx || !a || !t) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null handle");
  if (a->ctx != ctx || t->ctx != ctx)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "handles belong to another context");
  return set_device(ctx);
}

int finish_host_eval(rsot_cuda_ctx* c, rsot_cuda_targets* t, double* g_out,
                     rsot_cuda_scalars* out) {
  const cudaStream_t s = c->stream;
  RSOT_CK(cudaMemcpyAsync(c->h_pinned, c->scalars_out.p, sizeof(double) * kResTail,
                          cudaMemcpyDeviceToHost, s));
  RSOT_CK(cudaMemcpyAsync(c->h_pinned + kResTail, c->scal.p + kSlotNonFinite,
                          sizeof(double), cudaMemcpyDeviceToHost, s));
  RSOT_CK(cudaMemcpyAsync(g_out, c->g_out.p, sizeof(double) * t->n,
                          cudaMemcpyDeviceToHost, s));
  unsigned* ovf = reinterpret_cast<unsigned*>(c->h_pinned + kResTail + 1);
  RSOT_CK(trunc_read_overflow(ovf, s));
  RSOT_CK(cudaStreamSynchronize(s));
  record_timing(c);
  if (c->h_pinned[kResTail] != 0.0)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "potential has non-finite entries");
  if (*ovf) {
    trunc_clear_overflow();
    return fail(RSOT_CUDA_RUNTIME_ERROR,
                "gradient accumulator overflow: a single atom-target contribution >= 2^41 "
                "(masses far from normalised)");
  }
  out->J = c->h_pinned[kResJ];
  out->D = c->h_pinned[kResD];
  out->candidate_pairs = static_cast<uint64_t>(c->h_pinned[kResPairs]);
  out->empty_candidate_atoms = static_cast<uint64_t>(c->h_pinned[kResEmpty]);
  out->atoms_visited = static_cast<uint64_t>(c->h_pinned[kResVisited]);
  return RSOT_CUDA_OK;
}

}  // namespace

extern "C" {

int rsot_cuda_abi_version(void) { return RSOT_CUDA_ABI_VERSION; }

uint64_t rsot_cuda_kernel_launches(void) { return g_kernel_launches.load(); }

const char* rsot_cuda_last_error(void) { return g_last_error.c_str(); }

int rsot_cuda_ctx_create(int device, rsot_cuda_ctx** out) {
  if (!out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(RSOT_CUDA_NO_DEVICE, "no CUDA device visible");
  }
  if (device < 0 || device >= count)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "device ordinal out of range");
  cudaDeviceProp prop;
  RSOT_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(RSOT_CUDA_NO_DEVICE,
                "device is not sm_100 (built for sm_100a only): " +
                    std::string(prop.name));
  auto* c = new (std::nothrow) rsot_cuda_ctx();
  if (!c) return fail(RSOT_CUDA_RUNTIME_ERROR, "out of host memory");
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  RSOT_CK(cudaSetDevice(device));
  RSOT_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  RSOT_CK(cudaMallocHost(&c->h_pinned, sizeof(double) * 64));
  for (auto& e : c->ev) RSOT_CK(cudaEventCreate(&e));
  *out = c;
  return RSOT_CUDA_OK;
}

int rsot_cuda_ctx_destroy(rsot_cuda_ctx* c) {
  if (!c) return RSOT_CUDA_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  c->psi.release(); c->b2.release(); c->scal.release(); c->part.release();
  c->partS.release(); c->shiftA.release(); c->atomL.release();
  c->atomLam.release(); c->atomJ.release(); c->atomD.release();
  c->partG.release(); c->res.release(); c->g_out.release();
  c->scalars_out.release(); c->flagged.release(); c->gathered.release();
  c->trunc.release();
  c->refine.release();
  c->geo.release();
  if (c->graph.exec) cudaGraphExecDestroy(c->graph.exec);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  delete c;
  return RSOT_CUDA_OK;
}

void* rsot_cuda_ctx_stream(rsot_cuda_ctx* c) { return c ? c->stream : nullptr; }

int rsot_cuda_ctx_synchronize(rsot_cuda_ctx* c) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  RSOT_CK(cudaSetDevice(c->device));
  RSOT_CK(cudaStreamSynchronize(c->stream));
  record_timing(c);
  return RSOT_CUDA_OK;
}

int rsot_cuda_ctx_num_sms(rsot_cuda_ctx* c) { return c ? c->num_sms : 0; }

int rsot_cuda_comm_unique_id(unsigned char id_out[128]) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(RSOT_CUDA_RUNTIME_ERROR, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess)
    return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id_out, id.internal, 128);
  return RSOT_CUDA_OK;
}

int rsot_cuda_ctx_set_comm(rsot_cuda_ctx* c, int rank, int world,
                           const unsigned char id[128]) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "bad rank/world");
  c->rank = rank;
  c->world = world;
  if (c->graph.exec) cudaGraphExecDestroy(c->graph.exec);
  c->graph = rsot_cuda_ctx::DenseGraph();
  // (a 1-rank communicator is created too: it runs the same gather +
  // rank-ordered sum, which lets a single GPU exercise the collective path)
  NcclApi& api = nccl();
  if (!api.ok) return fail(RSOT_CUDA_RUNTIME_ERROR, "libnccl.so.2 not loadable");
  const int rc = set_device(c);
  if (rc) return rc;
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  const ncclResult_t r = api.CommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess)
    return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
  return RSOT_CUDA_OK;
}

void rsot_cuda_shard_range(size_t nq, int rank, int world, size_t* lo, size_t* hi) {
  if (world <= 1 || nq < 2) {
    *lo = rank == 0 ? 0 : nq;
    *hi = nq;
    if (rank != 0) *lo = *hi = nq;
    return;
  }
  const size_t w = static_cast<size_t>(world) < nq ? static_cast<size_t>(world) : nq;
  const size_t chunk = (nq + w - 1) / w;
  size_t l = static_cast<size_t>(rank) * chunk;
  size_t h = l + chunk;
  if (l > nq) l = nq;
  if (h > nq) h = nq;
  *lo = l;
  *hi = h;
}

int rsot_cuda_targets_create(rsot_cuda_ctx* c, const double* xyz, const double* nu,
                             size_t n, rsot_cuda_targets** out) {
  if (!c || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (n == 0) return fail(RSOT_CUDA_INVALID_ARGUMENT, "spatial index: empty point set");
  if (!xyz || !nu) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null data pointer");
  if (n > (1u << 30)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "too many targets");
  int rc = set_device(c);
  if (rc) return rc;
  // validation before any device allocation (every point, from j = 0)
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) lo[d] = hi[d] = xyz[d];
  std::vector<double4> h(n);
  for (size_t j = 0; j < n; ++j) {
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[3 * j + d];
      if (!std::isfinite(v))
        return fail(RSOT_CUDA_INVALID_ARGUMENT, "target point has non-finite coordinates");
      lo[d] = std::min(lo[d], v);
      hi[d] = std::max(hi[d], v);
    }
    h[j] = make_double4(xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2], std::log(nu[j]));
  }
  std::unique_ptr<rsot_cuda_targets> t(new (std::nothrow) rsot_cuda_targets());
  if (!t) return fail(RSOT_CUDA_RUNTIME_ERROR, "out of host memory");
  for (int d = 0; d < 3; ++d) {
    t->cells.bbox_lo[d] = lo[d];
    t->cells.bbox_hi[d] = hi[d];
  }
  t->cells.bbox_set = true;
  t->ctx = c;
  t->n = n;
  // (on any error below the partially built handle is released)
  auto release = [&](cudaError_t e, const char* what) {
    cudaFree(t->y);
    cudaFree(t->nu);
    t->y = nullptr;
    t->nu = nullptr;
    return fail(RSOT_CUDA_RUNTIME_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e = cudaMalloc(&t->y, sizeof(double4) * n);
  if (e != cudaSuccess) return release(e, "cudaMalloc(targets)");
  e = cudaMalloc(&t->nu, sizeof(double) * n);
  if (e != cudaSuccess) return release(e, "cudaMalloc(weights)");
  e = cudaMemcpyAsync(t->y, h.data(), sizeof(double4) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->nu, nu, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return release(e, "target upload");
  *out = t.release();
  return RSOT_CUDA_OK;
}

int rsot_cuda_targets_destroy(rsot_cuda_targets* t) {
  if (!t) return RSOT_CUDA_OK;
  cudaSetDevice(t->ctx->device);
  cudaStreamSynchronize(t->ctx->stream);
  cudaFree(t->y);
  cudaFree(t->nu);
  t->cells.release();
  delete t;
  return RSOT_CUDA_OK;
}

size_t rsot_cuda_targets_size(const rsot_cuda_targets* t) { return t ? t->n : 0; }

int rsot_cuda_atoms_create(rsot_cuda_ctx* c, const double* xyz, const double* mass,
                           size_t nq, rsot_cuda_atoms** out) {
  if (!c || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (nq && (!xyz || !mass)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null data pointer");
  if (nq > (1u << 30)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "too many atoms");
  int rc = set_device(c);
  if (rc) return rc;
  // validation before any device allocation: finite coordinates, finite
  // non-negative masses (every atom, from q = 0)
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, msum = 0.0;
  if (nq)
    for (int d = 0; d < 3; ++d) lo[d] = hi[d] = xyz[d];
  std::vector<double4> h(nq);
  for (size_t q = 0; q < nq; ++q) {
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[3 * q + d];
      if (!std::isfinite(v))
        return fail(RSOT_CUDA_INVALID_ARGUMENT, "atom point has non-finite coordinates");
      lo[d] = std::min(lo[d], v);
      hi[d] = std::max(hi[d], v);
    }
    if (!(mass[q] >= 0.0) || !std::isfinite(mass[q]))
      return fail(RSOT_CUDA_INVALID_ARGUMENT, "atom mass is negative or non-finite");
    msum += mass[q];
    h[q] = make_double4(xyz[3 * q], xyz[3 * q + 1], xyz[3 * q + 2], mass[q]);
  }
  std::unique_ptr<rsot_cuda_atoms> a(new (std::nothrow) rsot_cuda_atoms());
  if (!a) return fail(RSOT_CUDA_RUNTIME_ERROR, "out of host memory");
  for (int d = 0; d < 3; ++d) {
    a->cells.bbox_lo[d] = lo[d];
    a->cells.bbox_hi[d] = hi[d];
  }
  a->cells.bbox_set = true;
  a->ctx = c;
  a->nq = nq;
  a->mass_sum = msum;
  cudaError_t e = cudaMalloc(&a->x, sizeof(double4) * (nq ? nq : 1));
  if (e == cudaSuccess && nq)
    e = cudaMemcpyAsync(a->x, h.data(), sizeof(double4) * nq, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    cudaFree(a->x);
    return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("atom upload: ") + cudaGetErrorString(e));
  }
  *out = a.release();
  return RSOT_CUDA_OK;
}

int rsot_cuda_atoms_create_partitioned(rsot_cuda_ctx* c, const double* xyz, const double* mass,
                                       size_t nq, rsot_cuda_atoms** out) {
  const int rc = rsot_cuda_atoms_create(c, xyz, mass, nq, out);
  if (rc == RSOT_CUDA_OK) (*out)->partitioned = true;
  return rc;
}

int rsot_cuda_atoms_create_local(rsot_cuda_ctx* c, const double* xyz, const double* mass, size_t nq,
                                 rsot_cuda_atoms** out) {
  const int rc = rsot_cuda_atoms_create(c, xyz, mass, nq, out);
  if (rc == RSOT_CUDA_OK) (*out)->local = true;
  return rc;
}

int rsot_cuda_ctx_set_virtual_rank(rsot_cuda_ctx* c, int rank, int world) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  if (world < 1 || rank < 0 || rank >= world) return fail(RSOT_CUDA_INVALID_ARGUMENT, "bad rank/world");
  if (c->comm) return fail(RSOT_CUDA_INVALID_ARGUMENT, "context has a communicator");
  c->vrank = rank;
  c->vworld = world;
  return RSOT_CUDA_OK;
}

int rsot_cuda_atoms_destroy(rsot_cuda_atoms* a) {
  if (!a) return RSOT_CUDA_OK;
  cudaSetDevice(a->ctx->device);
  cudaStreamSynchronize(a->ctx->stream);
  cudaFree(a->x);
  a->cells.release();
  delete a;
  return RSOT_CUDA_OK;
}

size_t rsot_cuda_atoms_size(const rsot_cuda_atoms* a) { return a ? a->nq : 0; }

namespace {
bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RSOT_CUDA_GRAPHS");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// everything a captured dense evaluation bakes in besides (atoms, targets,
// eps, sizes): workspace and data pointers, the communicator, the bbox
uint64_t workspace_key(const rsot_cuda_ctx* c, const rsot_cuda_atoms* a, const rsot_cuda_targets* t) {
  const void* ptrs[] = {a->x, t->y, t->nu, static_cast<const void*>(c->comm),
                        c->psi.p, c->b2.p, c->scal.p, c->part.p, c->partS.p, c->shiftA.p, c->atomL.p, c->atomLam.p, c->atomJ.p, c->atomD.p, c->partG.p,
                        c->res.p, c->g_out.p, c->scalars_out.p, c->gathered.p, c->flagged.p};
  uint64_t h = 1469598103934665603ull;
  for (const void* p : ptrs) h = (h ^ reinterpret_cast<uintptr_t>(p)) * 1099511628211ull;
  h = (h ^ static_cast<uint64_t>(c->vrank * 65536 + c->vworld * 2 + (a->partitioned ? 1 : 0))) *
      1099511628211ull;
  for (int k = 0; k < 3; ++k) {
    uint64_t u, v;
    std::memcpy(&u, &t->cells.bbox_lo[k], 8);
    std::memcpy(&v, &t->cells.bbox_hi[k], 8);
    h = (h ^ u) * 1099511628211ull;
    h = (h ^ v) * 1099511628211ull;
  }
  return h;
}

// Dense device evaluation through a captured CUDA graph: psi is copied into
// the context's buffer, the graph replays, the results are copied out.
// Outputs stay in the context's g_out / scalars_out when d_g_out is null.
int eval_dense_graph(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                     const double* h_psi, const double* d_psi, double eps, double* d_g_out,
                     double* d_scalars) {
  int rc = 0;
  auto& G = c->graph;
  const uint64_t key = workspace_key(c, a, t);
  if (!(G.exec && G.atoms == a && G.targets == t && G.eps == eps && G.nq == a->nq && G.n == t->n &&
        G.ws_key == key)) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G.exec = nullptr;
    EvalBuffers b = buffers(c, nullptr, nullptr);
    b.timing = nullptr;
    cudaGraph_t graph = nullptr;
    RSOT_CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const unsigned long long l0 = g_kernel_launches.load();
    rc = enqueue_eval(c, a, t, b, eps, INFINITY, nullptr);
    const cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
    const unsigned long long captured = g_kernel_launches.load() - l0;
    g_kernel_launches.fetch_sub(captured);  // counted again at every replay
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    cudaError_t ei = e;
    if (ei == cudaSuccess) ei = cudaGraphInstantiate(&G.exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      // e.g. a communicator that refuses capture: same kernels, launched directly
      cudaGetLastError();
      G.exec = nullptr;
      G.broken = true;
      return -1;  // caller launches directly
    }
    G.atoms = a;
    G.targets = t;
    G.eps = eps;
    G.nq = a->nq;
    G.n = t->n;
    G.ws_key = key;
    G.launches = captured;
  }
  RSOT_CK(cudaMemcpyAsync(c->psi.p, h_psi ? h_psi : d_psi, sizeof(double) * t->n,
                          h_psi ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
  RSOT_CK(cudaGraphLaunch(G.exec, c->stream));
  g_kernel_launches.fetch_add(G.launches);
  if (d_g_out) {
    RSOT_CK(cudaMemcpyAsync(d_g_out, c->g_out.p, sizeof(double) * t->n, cudaMemcpyDeviceToDevice,
                            c->stream));
    RSOT_CK(cudaMemcpyAsync(d_scalars, c->scalars_out.p, sizeof(double) * kResTail,
                            cudaMemcpyDeviceToDevice, c->stream));
  }
  return RSOT_CUDA_OK;
}
}  // namespace

static int eval_common(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                       const double* psi_host, const double* psi_dev, double eps,
                       double cutoff, double* g_dev, double* scal_dev,
                       DebugOut* dbg, int cost = RSOT_CUDA_COST_SQEUCLIDEAN) {
  if (!(eps > 0.0)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "epsilon must be > 0");
  if (std::isnan(cutoff)) cutoff = INFINITY;  // isfinite(NaN) is false: dense
  const DenseLaunch plan = plan_dense(static_cast<int>(a->nq), static_cast<int>(t->n), c->num_sms);
  int rc = ensure_workspace(c, a->nq, t->n, plan);
  if (rc) return rc;
  // dense evaluations without debug outputs or per-kernel timing replay a
  // captured graph
  if (!std::isfinite(cutoff) && cost == RSOT_CUDA_COST_SQEUCLIDEAN && !dbg && !c->timing && a->nq > 0 &&
      !c->graph.broken && graphs_enabled()) {
    rc = eval_dense_graph(c, a, t, psi_host, psi_dev, eps, g_dev, scal_dev);
    if (rc != -1) return rc;
  }
  EvalBuffers b = buffers(c, g_dev, scal_dev);
  if (psi_host)
    RSOT_CK(cudaMemcpyAsync(b.psi, psi_host, sizeof(double) * t->n,
                            cudaMemcpyHostToDevice, c->stream));
  else
    b.psi = const_cast<double*>(psi_dev);
  return enqueue_eval(c, a, t, b, eps, cutoff, dbg, cost);
}

int rsot_cuda_eval(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                   const double* psi, double eps, double cutoff, double* g_out,
                   rsot_cuda_scalars* out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!psi || !g_out || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  rc = eval_common(c, a, t, psi, nullptr, eps, cutoff, nullptr, nullptr, nullptr);
  if (rc) return rc;
  return finish_host_eval(c, t, g_out, out);
}

int rsot_cuda_eval_cost(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                        const double* psi, double eps, double cutoff, int cost_kind,
                        double* g_out, rsot_cuda_scalars* out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!psi || !g_out || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (cost_kind != RSOT_CUDA_COST_SQEUCLIDEAN && cost_kind != RSOT_CUDA_COST_SQGEODESIC)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown cost kind");
  rc = eval_common(c, a, t, psi, nullptr, eps, cutoff, nullptr, nullptr, nullptr, cost_kind);
  if (rc) return rc;
  return finish_host_eval(c, t, g_out, out);
}


int rsot_cuda_eval_device(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                          const double* d_psi, double eps, double cutoff,
                          double* d_g_out, double* d_scalars) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!d_psi || !d_g_out || !d_scalars)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  return eval_common(c, a, t, nullptr, d_psi, eps, cutoff, d_g_out, d_scalars, nullptr);
}

// Debug / test entry point: one evaluation as `world` virtual ranks of a
// multi-GPU run on this GPU.  Each virtual rank's packed partial buffer is
// computed exactly as that rank would (partitioned atoms: its work-balanced
// chunk range or contiguous shard) and copied into the gather buffer at the
// rank's offset, which stands in for ncclAllGather; the rank-ordered sum and
// the finalisation are the same launches that follow the collective in
// enqueue_eval.
int rsot_cuda_eval_virtual_world(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                                 const double* psi, double eps, double cutoff, int world,
                                 double* g_out, rsot_cuda_scalars* out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!psi || !g_out || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (world < 1 || world > 1024) return fail(RSOT_CUDA_INVALID_ARGUMENT, "bad world size");
  if (c->comm) return fail(RSOT_CUDA_INVALID_ARGUMENT, "context has a communicator");
  if (!a->partitioned && world > 1)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "virtual ranks need partitioned atoms");
  if (!(eps > 0.0)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "epsilon must be > 0");
  if (std::isnan(cutoff)) cutoff = INFINITY;
  const DenseLaunch plan = plan_dense(static_cast<int>(a->nq), static_cast<int>(t->n), c->num_sms);
  rc = ensure_workspace(c, a->nq, t->n, plan);
  if (rc) return rc;
  const size_t len = t->n + kResTail;
  RSOT_CK(c->gathered.ensure(static_cast<size_t>(world) * len));
  EvalBuffers b = buffers(c, nullptr, nullptr);
  b.timing = nullptr;
  const cudaStream_t s = c->stream;
  RSOT_CK(cudaMemcpyAsync(b.psi, psi, sizeof(double) * t->n, cudaMemcpyHostToDevice, s));
  const int vr = c->vrank, vw = c->vworld;
  for (int r = 0; r < world && rc == 0; ++r) {
    c->vrank = r;
    c->vworld = world;
    rc = enqueue_partial(c, a, t, b, eps, cutoff, nullptr, RSOT_CUDA_COST_SQEUCLIDEAN);
    if (rc == 0 && cudaMemcpyAsync(c->gathered.p + static_cast<size_t>(r) * len, b.res, sizeof(double) * len,
                                   cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      rc = fail(RSOT_CUDA_RUNTIME_ERROR, "gather copy failed");
  }
  c->vrank = vr;
  c->vworld = vw;
  if (rc) return rc;
  launch_rank_sum(c->gathered.p, world, len, b.res, s);
  launch_finalize(make_dt(t), b, s);
  RSOT_CK(cudaGetLastError());
  return finish_host_eval(c, t, g_out, out);
}

// Host mirrors of the combination kernels (the same element functions,
// kernels.cuh), for the multi-process CPU tests of the host logic.
void rsot_cuda_host_rank_sum(const double* gathered, int world, size_t len, double* out) {
  if (!gathered || !out || world < 1) return;
  for (size_t i = 0; i < len; ++i) out[i] = rank_sum_element(gathered, world, len, i);
}

void rsot_cuda_host_finalize(const double* res, const double* nu, size_t n, double psi_nu, double* g_out,
                             double* scalars_out) {
  if (!res || !nu || !g_out || !scalars_out) return;
  for (size_t j = 0; j < n; ++j) g_out[j] = finalize_gradient_element(res, nu, j);
  finalize_scalars(res, n, psi_nu, scalars_out);
}

int rsot_cuda_check_status(rsot_cuda_ctx* c) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  RSOT_CK(cudaSetDevice(c->device));
  RSOT_CK(cudaMemcpyAsync(c->h_pinned, c->scal.p + kSlotNonFinite, sizeof(double),
                          cudaMemcpyDeviceToHost, c->stream));
  unsigned* ovf = reinterpret_cast<unsigned*>(c->h_pinned + 1);
  RSOT_CK(trunc_read_overflow(ovf, c->stream));
  RSOT_CK(cudaStreamSynchronize(c->stream));
  if (c->h_pinned[0] != 0.0)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "potential has non-finite entries");
  if (*ovf) {
    trunc_clear_overflow();
    return fail(RSOT_CUDA_RUNTIME_ERROR, "gradient accumulator overflow (masses far from normalised)");
  }
  return RSOT_CUDA_OK;
}

int rsot_cuda_eval_debug(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                         const double* psi, double eps, double cutoff, double* g_out,
                         rsot_cuda_scalars* out, uint32_t* cand_count,
                         uint64_t* cand_hash, double* log_s) {
  return rsot_cuda_eval_debug_cost(c, a, t, psi, eps, cutoff, RSOT_CUDA_COST_SQEUCLIDEAN, g_out,
                                   out, cand_count, cand_hash, log_s);
}

int rsot_cuda_eval_debug_cost(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                              const double* psi, double eps, double cutoff, int cost_kind,
                              double* g_out, rsot_cuda_scalars* out, uint32_t* cand_count,
                              uint64_t* cand_hash, double* log_s) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!psi || !g_out || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (cost_kind != RSOT_CUDA_COST_SQEUCLIDEAN && cost_kind != RSOT_CUDA_COST_SQGEODESIC)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown cost kind");
  DebugOut dbg;
  const size_t nq = a->nq ? a->nq : 1;
  RSOT_CK(cudaMalloc(&dbg.count, sizeof(uint32_t) * nq));
  RSOT_CK(cudaMalloc(&dbg.hash, sizeof(uint64_t) * nq));
  RSOT_CK(cudaMalloc(&dbg.log_s, sizeof(double) * nq));
  rc = eval_common(c, a, t, psi, nullptr, eps, cutoff, nullptr, nullptr, &dbg, cost_kind);
  if (rc == 0) rc = finish_host_eval(c, t, g_out, out);
  if (rc == 0 && a->nq) {
    if (cand_count)
      cudaMemcpy(cand_count, dbg.count, sizeof(uint32_t) * a->nq, cudaMemcpyDeviceToHost);
    if (cand_hash)
      cudaMemcpy(cand_hash, dbg.hash, sizeof(uint64_t) * a->nq, cudaMemcpyDeviceToHost);
    if (log_s)
      cudaMemcpy(log_s, dbg.log_s, sizeof(double) * a->nq, cudaMemcpyDeviceToHost);
  }
  cudaFree(dbg.count);
  cudaFree(dbg.hash);
  cudaFree(dbg.log_s);
  return rc;
}

int rsot_cuda_nearest(rsot_cuda_ctx* c, rsot_cuda_targets* t, const double* xyz,
                      size_t m, uint64_t* out) {
  if (!c || !t || (m && (!xyz || !out)))
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  int rc = set_device(c);
  if (rc) return rc;
  if (m == 0) return RSOT_CUDA_OK;
  rc = run_nearest_points(c->trunc, make_dt(t),
                          t->cells, xyz, m, out, c->stream, g_last_error);
  return rc ? fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error) : RSOT_CUDA_OK;
}

int rsot_cuda_covering_cost(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                            double* out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  double c0 = 0.0;
  rc = run_covering_cost(c->trunc, DeviceAtoms{a->x, static_cast<int>(a->nq)},
                         make_dt(t), t->cells,
                         &c0, c->stream, g_last_error);
  if (rc) return fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error);
  if (c->comm && !a->local) {
    // max over ranks: all values are >= 0, so a max-allreduce is exact.
    RSOT_CK(cudaMemcpyAsync(c->scal.p, &c0, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    NcclApi& api = nccl();
    const ncclResult_t r = api.AllReduce(c->scal.p, c->scal.p, 1, ncclDouble, ncclMax,
                                         c->comm, c->stream);
    if (r != ncclSuccess)
      return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("ncclAllReduce: ") + api.GetErrorString(r));
    RSOT_CK(cudaMemcpyAsync(c->h_pinned, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    RSOT_CK(cudaStreamSynchronize(c->stream));
    c0 = c->h_pinned[0];
  }
  *out = c0;
  return RSOT_CUDA_OK;
}

int rsot_cuda_covering_cost_kind(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t, int cost_kind,
                                 double* out) {
  if (cost_kind == RSOT_CUDA_COST_SQEUCLIDEAN) return rsot_cuda_covering_cost(c, a, t, out);
  if (cost_kind != RSOT_CUDA_COST_SQGEODESIC) return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown cost kind");
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (a->nq == 0) return fail(RSOT_CUDA_INVALID_ARGUMENT, "covering cost: empty input");
  double tstar = 0.0;
  rc = run_geo_covering_dot(c->geo, DeviceAtoms{a->x, static_cast<int>(a->nq)}, make_dt(t), &tstar, c->stream,
                            g_last_error);
  if (rc) return fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error);
  // cost.hpp:24-25 on the host (the reference's libm acos), monotone in t
  const double g = std::acos(tstar);
  double c0 = g * g;
  if (c->comm && !a->local) {
    RSOT_CK(cudaMemcpyAsync(c->scal.p, &c0, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    NcclApi& api = nccl();
    const ncclResult_t r = api.AllReduce(c->scal.p, c->scal.p, 1, ncclDouble, ncclMax, c->comm, c->stream);
    if (r != ncclSuccess)
      return fail(RSOT_CUDA_RUNTIME_ERROR, std::string("ncclAllReduce: ") + api.GetErrorString(r));
    RSOT_CK(cudaMemcpyAsync(c->h_pinned, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    RSOT_CK(cudaStreamSynchronize(c->stream));
    c0 = c->h_pinned[0];
  }
  *out = c0;
  return RSOT_CUDA_OK;
}

int rsot_cuda_softmax_refine(rsot_cuda_ctx* c, rsot_cuda_targets* coarse,
                             const double* coarse_psi, const double* fine_xyz, size_t n_fine,
                             rsot_cuda_atoms* a, double eps, double cutoff, double* psi_out) {
  int rc = check_ready(c, a, coarse);
  if (rc) return rc;
  if (!coarse_psi || (n_fine && (!fine_xyz || !psi_out)))
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (!(eps > 0.0)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "epsilon must be > 0");
  for (size_t j = 0; j < coarse->n; ++j)
    if (!std::isfinite(coarse_psi[j]))
      return fail(RSOT_CUDA_INVALID_ARGUMENT, "potential has non-finite entries");
  if (a->nq == 0)  // the reference's phase 2 yields -eps*(-inf) -> require_finite throws
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "potential has non-finite entries");
  if (n_fine == 0) return RSOT_CUDA_OK;
  if (std::isnan(cutoff)) cutoff = INFINITY;
  const DenseLaunch plan = plan_dense(static_cast<int>(a->nq), static_cast<int>(coarse->n), c->num_sms);
  rc = ensure_workspace(c, a->nq, coarse->n, plan);
  if (rc) return rc;
  EvalBuffers b = buffers(c, nullptr, nullptr);
  b.timing = nullptr;
  RSOT_CK(cudaMemcpyAsync(b.psi, coarse_psi, sizeof(double) * coarse->n, cudaMemcpyHostToDevice,
                          c->stream));
  const DeviceTargets dt = make_dt(coarse);
  launch_prologue(dt, b, eps, c->stream);
  rc = run_softmax_refine(c->refine, DeviceAtoms{a->x, static_cast<int>(a->nq)}, dt, b, fine_xyz,
                          static_cast<int>(n_fine), eps, cutoff, c->num_sms, psi_out, c->stream,
                          g_last_error);
  return rc ? fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error) : RSOT_CUDA_OK;
}

int rsot_cuda_plan_candidates(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                              double cutoff, int cost_kind, const uint64_t* offsets,
                              uint64_t* idx_out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (cost_kind != RSOT_CUDA_COST_SQEUCLIDEAN && cost_kind != RSOT_CUDA_COST_SQGEODESIC)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown cost kind");
  if (!offsets || (a->nq && offsets[a->nq] && !idx_out))
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (std::isnan(cutoff)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "cutoff is NaN");
  if (!std::isfinite(cutoff)) {  // dense: every target, ascending (plan.cpp:40-42)
    for (size_t q = 0; q < a->nq; ++q) {
      if (offsets[q + 1] - offsets[q] != t->n)
        return fail(RSOT_CUDA_INVALID_ARGUMENT, "offsets do not match the dense candidate count");
      for (size_t j = 0; j < t->n; ++j) idx_out[offsets[q] + j] = j;
    }
    return RSOT_CUDA_OK;
  }
  rc = run_plan_candidates(c->trunc, DeviceAtoms{a->x, static_cast<int>(a->nq)}, make_dt(t),
                           t->cells, cutoff, cost_kind == RSOT_CUDA_COST_SQGEODESIC, offsets,
                           idx_out, c->stream, g_last_error);
  return rc ? fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error) : RSOT_CUDA_OK;
}

int rsot_cuda_plan_moments(rsot_cuda_ctx* c, rsot_cuda_atoms* a, rsot_cuda_targets* t,
                           const double* psi, double eps, int cost_kind, const double* log_s,
                           const uint64_t* offsets, const uint64_t* idx, double* marginal_out,
                           double* moment_out, double* map_out, uint64_t* modal_out) {
  int rc = check_ready(c, a, t);
  if (rc) return rc;
  if (!psi || (a->nq && !log_s) || (offsets && offsets[a->nq] && !idx))
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  if (!(eps > 0.0)) return fail(RSOT_CUDA_INVALID_ARGUMENT, "epsilon must be > 0");
  if (cost_kind != RSOT_CUDA_COST_SQEUCLIDEAN && cost_kind != RSOT_CUDA_COST_SQGEODESIC)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown cost kind");
  for (size_t j = 0; j < t->n; ++j)
    if (!std::isfinite(psi[j]))
      return fail(RSOT_CUDA_INVALID_ARGUMENT, "potential has non-finite entries");
  if (offsets && idx)
    for (uint64_t k = 0; k < offsets[a->nq]; ++k)
      if (idx[k] >= t->n) return fail(RSOT_CUDA_INVALID_ARGUMENT, "candidate index out of range");
  rc = run_plan_moments(DeviceAtoms{a->x, static_cast<int>(a->nq)}, make_dt(t), psi, eps,
                        cost_kind == RSOT_CUDA_COST_SQGEODESIC, log_s,
                        offsets, idx, a->cells.bbox_lo, marginal_out, moment_out, map_out,
                        modal_out, c->stream, g_last_error);
  return rc ? fail(RSOT_CUDA_RUNTIME_ERROR, g_last_error) : RSOT_CUDA_OK;
}

int rsot_cuda_ctx_set_precision(rsot_cuda_ctx* c, int precision) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  if (precision != RSOT_CUDA_PRECISION_FP64 && precision != RSOT_CUDA_PRECISION_FP32)
    return fail(RSOT_CUDA_INVALID_ARGUMENT, "unknown precision");
  c->precision = precision;
  return RSOT_CUDA_OK;
}

int rsot_cuda_ctx_set_timing(rsot_cuda_ctx* c, int enable) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  c->timing = enable != 0;
  return RSOT_CUDA_OK;
}

int rsot_cuda_last_kernel_ms(rsot_cuda_ctx* c, double* a, double* b, double* tot) {
  if (!c) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null context");
  if (a) *a = c->last_ms[0];
  if (b) *b = c->last_ms[1];
  if (tot) *tot = c->last_ms[2];
  return RSOT_CUDA_OK;
}

int rsot_cuda_measure_fp64_peak(rsot_cuda_ctx* c, double* out) {
  if (!c || !out) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  int rc = set_device(c);
  if (rc) return rc;
  *out = measure_dfma_rate(c->stream);
  RSOT_CK(cudaGetLastError());
  return RSOT_CUDA_OK;
}

int rsot_cuda_measure_fp32_peaks(rsot_cuda_ctx* c, double* ffma_per_s, double* ex2_per_s) {
  if (!c || !ffma_per_s || !ex2_per_s) return fail(RSOT_CUDA_INVALID_ARGUMENT, "null argument");
  int rc = set_device(c);
  if (rc) return rc;
  measure_fp32_rates(c->stream, ffma_per_s, ex2_per_s);
  RSOT_CK(cudaGetLastError());
  return RSOT_CUDA_OK;
}

}  // extern "C"
