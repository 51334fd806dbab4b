// comm.cu — the multi-GPU layer of the C ABI: views partitioned by camera over
// one process per GPU (or one process driving several), Gaussians replicated, and the one
// collective of the path: an NCCL all-reduce (sum) of the per-Gaussian gradients.
//
//   fgs_comm_get_unique_id / fgs_comm_init      one rank per process (ncclCommInitRank), the id
//                                                shared out of band (MPI, torch.distributed, a file)
//   fgs_comm_init_all                            one process, several devices (ncclCommInitAll)
//   fgs_allreduce_gradients                      in-place sum of the five gradient arrays
//   fgs_fwd_bwd_views                            this rank's views forward + backward accumulated
//                                                into one gradient set, then the all-reduce -- the
//                                                last view's K4b in kGradChunks Gaussian-id ranges,
//                                                each range's all-reduce on a communication stream
//                                                as soon as the range is written, overlapping the
//                                                next range's K4b.
//
// NCCL is loaded at first use with dlopen("libnccl.so.2") (in a PyTorch process this resolves to the
// NCCL torch already loaded), so libfgs.so does not depend on it for single-GPU use. The reference
// has no multi-GPU path (its contract is one camera per call, inc/splatting.hpp:330-332); the
// multi-view sum is this build's.

#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fgs.h"
#include "fgs_kernels.h"

// from fgs_api.cu
int fgs_internal_fail(fgs_context* ctx, int code, const char* msg);
cudaStream_t fgs_internal_stream(fgs_context* ctx);
int fgs_internal_device(fgs_context* ctx);
float* fgs_internal_scratch_image(fgs_context* ctx, size_t floats);  // context-owned, grows only
int fgs_internal_backward(fgs_context* ctx, const fgs_gaussians* scene, const fgs_camera* camera,
                          const float* dl_dimage, const fgs_backward_options* options, fgs_gradients* grads,
                          const std::function<int(int, int64_t, int64_t)>& chunk_done);

namespace {

struct Nccl {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.err = std::string("NCCL not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
           sym(n.CommInitAll, "ncclCommInitAll") && sym(n.CommDestroy, "ncclCommDestroy") &&
           sym(n.AllReduce, "ncclAllReduce") && sym(n.GroupStart, "ncclGroupStart") &&
           sym(n.GroupEnd, "ncclGroupEnd") && sym(n.GetErrorString, "ncclGetErrorString");
    if (!n.ok) n.err = "NCCL library lacks an entry point";
  });
  return n;
}

}  // namespace

struct fgs_comm {
  fgs_context* ctx = nullptr;
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;    // communication stream (non-blocking)
  cudaEvent_t ready[fgs::kGradChunks + 1] = {};
  cudaEvent_t done = nullptr;
};

namespace {

int nccl_fail(fgs_context* ctx, ncclResult_t r, const char* where) {
  const std::string m = std::string(where) + ": " + nccl().GetErrorString(r);
  return fgs_internal_fail(ctx, FGS_ECUDA, m.c_str());
}

int setup(fgs_comm* c) {
  cudaSetDevice(c->device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return FGS_ECUDA;
  for (auto& e : c->ready)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return FGS_ECUDA;
  if (cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) != cudaSuccess) return FGS_ECUDA;
  return FGS_OK;
}

// The five field arrays' slices [id0, id1) (widths 3, 4, 3, 1, 48), summed in place over the ranks
// as one NCCL group on the communication stream.
ncclResult_t allreduce_range(fgs_comm* c, fgs_gradients* g, int64_t id0, int64_t id1) {
  const Nccl& N = nccl();
  float* p[5] = {g->d_means, g->d_rotations, g->d_log_scales, g->d_opacity_logits, g->d_sh};
  const int w[5] = {3, 4, 3, 1, 48};
  ncclResult_t r = N.GroupStart();
  if (r != ncclSuccess) return r;
  for (int k = 0; k < 5; ++k) {
    float* base = p[k] + id0 * w[k];
    const size_t count = static_cast<size_t>(id1 - id0) * w[k];
    if (count == 0) continue;
    r = N.AllReduce(base, base, count, ncclFloat32, ncclSum, c->comm, c->stream);
    if (r != ncclSuccess) {
      N.GroupEnd();
      return r;
    }
  }
  return N.GroupEnd();
}

}  // namespace

namespace {
int fwd_bwd_views_impl(fgs_context* ctx, fgs_comm* comm, const fgs_gaussians* scene, const fgs_camera* cameras,
                       int nviews, const float* const* dl_dimages, const fgs_render_options* ropt,
                       const fgs_backward_options* bopt, fgs_gradients* grads, float* const* images);
}  // namespace

extern "C" {

int fgs_comm_get_unique_id(uint8_t id[128]) {
  if (!id) return FGS_EINVAL;
  const Nccl& N = nccl();
  if (!N.ok) return FGS_ECUDA;
  ncclUniqueId u;
  if (N.GetUniqueId(&u) != ncclSuccess) return FGS_ECUDA;
  static_assert(sizeof(u) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(id, &u, 128);
  return FGS_OK;
}

int fgs_comm_init(fgs_context* ctx, const uint8_t id[128], int nranks, int rank, fgs_comm** out) {
  if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return ctx ? fgs_internal_fail(ctx, FGS_EINVAL, "comm_init: bad arguments") : FGS_EINVAL;
  *out = nullptr;
  const Nccl& N = nccl();
  if (!N.ok) return fgs_internal_fail(ctx, FGS_ECUDA, N.err.c_str());
  auto* c = new fgs_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  c->device = fgs_internal_device(ctx);
  if (setup(c) != FGS_OK) {
    fgs_comm_destroy(c);
    return fgs_internal_fail(ctx, FGS_ECUDA, "comm_init: stream/event creation failed");
  }
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  const ncclResult_t r = N.CommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    const int rc = nccl_fail(ctx, r, "ncclCommInitRank");
    c->comm = nullptr;
    fgs_comm_destroy(c);
    return rc;
  }
  *out = c;
  return FGS_OK;
}

int fgs_comm_init_all(fgs_context* const* ctxs, int ndev, fgs_comm** comms) {
  if (!ctxs || !comms || ndev < 1) return FGS_EINVAL;
  const Nccl& N = nccl();
  if (!N.ok) return fgs_internal_fail(ctxs[0], FGS_ECUDA, N.err.c_str());
  std::vector<int> devs(ndev);
  std::vector<ncclComm_t> cs(ndev);
  for (int i = 0; i < ndev; ++i) devs[i] = fgs_internal_device(ctxs[i]);
  const ncclResult_t r = N.CommInitAll(cs.data(), ndev, devs.data());
  if (r != ncclSuccess) return nccl_fail(ctxs[0], r, "ncclCommInitAll");
  for (int i = 0; i < ndev; ++i) {
    auto* c = new fgs_comm();
    c->ctx = ctxs[i];
    c->nranks = ndev;
    c->rank = i;
    c->device = devs[i];
    c->comm = cs[i];
    if (setup(c) != FGS_OK) return fgs_internal_fail(ctxs[i], FGS_ECUDA, "comm_init_all: stream/event creation failed");
    comms[i] = c;
  }
  return FGS_OK;
}

int fgs_comm_destroy(fgs_comm* c) {
  if (!c) return FGS_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  for (auto& e : c->ready)
    if (e) cudaEventDestroy(e);
  if (c->done) cudaEventDestroy(c->done);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return FGS_OK;
}

int fgs_allreduce_gradients(fgs_comm* c, fgs_gradients* grads, int64_t n) {
  if (!c || !grads) return FGS_EINVAL;
  fgs_context* ctx = c->ctx;
  if (cudaSetDevice(c->device) != cudaSuccess) return fgs_internal_fail(ctx, FGS_ECUDA, "allreduce: set device");
  cudaStream_t st = fgs_internal_stream(ctx);
  // the communication stream follows the compute stream, and the compute stream the result
  if (cudaEventRecord(c->ready[0], st) != cudaSuccess || cudaStreamWaitEvent(c->stream, c->ready[0], 0) != cudaSuccess)
    return fgs_internal_fail(ctx, FGS_ECUDA, "allreduce: stream ordering");
  const ncclResult_t r = allreduce_range(c, grads, 0, n);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllReduce");
  if (cudaEventRecord(c->done, c->stream) != cudaSuccess || cudaStreamWaitEvent(st, c->done, 0) != cudaSuccess)
    return fgs_internal_fail(ctx, FGS_ECUDA, "allreduce: stream ordering");
  return FGS_OK;
}

int fgs_fwd_bwd_views(fgs_context* ctx, fgs_comm* comm, const fgs_gaussians* scene, const fgs_camera* cameras,
                      int nviews, const float* const* dl_dimages, const fgs_render_options* ropt,
                      const fgs_backward_options* bopt, fgs_gradients* grads, float* const* images) {
  if (!ctx) return FGS_EINVAL;
  nvtxRangePushA("fgs.fwd_bwd_views");
  const int rc = fwd_bwd_views_impl(ctx, comm, scene, cameras, nviews, dl_dimages, ropt, bopt, grads, images);
  nvtxRangePop();
  return rc;
}

}  // extern "C"

namespace {
int fwd_bwd_views_impl(fgs_context* ctx, fgs_comm* comm, const fgs_gaussians* scene, const fgs_camera* cameras,
                       int nviews, const float* const* dl_dimages, const fgs_render_options* ropt,
                       const fgs_backward_options* bopt, fgs_gradients* grads, float* const* images) {
  if (!scene || (nviews > 0 && (!cameras || !dl_dimages)) || !grads || nviews < 0)
    return fgs_internal_fail(ctx, FGS_EINVAL, "fwd_bwd_views: null argument");
  if (comm && comm->ctx != ctx) return fgs_internal_fail(ctx, FGS_EINVAL, "fwd_bwd_views: communicator of another context");
  fgs_backward_options bo = bopt ? *bopt : fgs_backward_options{{1.f, 1.f, 1.f}, 1, 0, 0};
  const bool acc0 = bo.accumulate != 0;
  const int64_t n = scene->n;
  cudaStream_t st = fgs_internal_stream(ctx);
  if (cudaSetDevice(fgs_internal_device(ctx)) != cudaSuccess) return fgs_internal_fail(ctx, FGS_ECUDA, "set device");
  // images: caller's, else one scratch image reused by every view
  float* scratch = nullptr;
  size_t scratch_px = 0;
  for (int v = 0; v < nviews; ++v)
    if (!images || !images[v]) scratch_px = std::max(scratch_px, static_cast<size_t>(cameras[v].width) * cameras[v].height);
  if (scratch_px && !(scratch = fgs_internal_scratch_image(ctx, scratch_px * 3)))
    return fgs_internal_fail(ctx, FGS_ENOMEM, "fwd_bwd_views: image scratch");
  int rc = FGS_OK;
  for (int v = 0; v < nviews && rc == FGS_OK; ++v) {
    float* img = images && images[v] ? images[v] : scratch;
    rc = fgs_forward(ctx, scene, &cameras[v], ropt, img, nullptr, nullptr);
    if (rc != FGS_OK) break;
    bo.accumulate = (v > 0 || acc0) ? 1 : 0;
    const bool last = v + 1 == nviews;
    if (!last || !comm) {
      rc = fgs_internal_backward(ctx, scene, &cameras[v], dl_dimages[v], &bo, grads, nullptr);
    } else {
      // last view: each Gaussian-id range is reduced over the ranks as soon as K4b wrote it
      rc = fgs_internal_backward(ctx, scene, &cameras[v], dl_dimages[v], &bo, grads,
                                 [&](int c, int64_t id0, int64_t id1) -> int {
                                   if (cudaEventRecord(comm->ready[c], st) != cudaSuccess ||
                                       cudaStreamWaitEvent(comm->stream, comm->ready[c], 0) != cudaSuccess)
                                     return fgs_internal_fail(ctx, FGS_ECUDA, "fwd_bwd_views: stream ordering");
                                   const ncclResult_t r = allreduce_range(comm, grads, id0, id1);
                                   return r == ncclSuccess ? FGS_OK : nccl_fail(ctx, r, "ncclAllReduce");
                                 });
      if (rc == FGS_OK && (cudaEventRecord(comm->done, comm->stream) != cudaSuccess ||
                           cudaStreamWaitEvent(st, comm->done, 0) != cudaSuccess))
        rc = fgs_internal_fail(ctx, FGS_ECUDA, "fwd_bwd_views: stream ordering");
    }
  }
  if (rc == FGS_OK && nviews == 0 && !acc0) {  // a rank without views contributes zeros
    float* p[5] = {grads->d_means, grads->d_rotations, grads->d_log_scales, grads->d_opacity_logits, grads->d_sh};
    const int w[5] = {3, 4, 3, 1, 48};
    for (int k = 0; k < 5 && rc == FGS_OK; ++k)
      if (n > 0 && cudaMemsetAsync(p[k], 0, static_cast<size_t>(n) * w[k] * sizeof(float), st) != cudaSuccess)
        rc = fgs_internal_fail(ctx, FGS_ECUDA, "fwd_bwd_views: zero gradients");
  }
  if (rc == FGS_OK && comm && nviews == 0) rc = fgs_allreduce_gradients(comm, grads, n);
  return rc;
}
}  // namespace
