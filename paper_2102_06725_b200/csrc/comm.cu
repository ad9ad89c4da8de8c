// Data-parallel gradient all-reduce (communicator.py:69-105) as a C-ABI
// communicator over NCCL: one rank per process / GPU, NVLink/NVSwitch between
// them.  NCCL is resolved at run time (dlopen of the libnccl the process
// already has, usually torch's) so libnnl.so itself links no NCCL and loads
// on hosts without it; the declarations come from nccl.h at build time.
//
// One call, nnl_comm_allreduce_mean, is the whole bucket exchange on the
// caller's stream:
//   pack      gradients (fp16 / f32) -> f32 bucket     (k_bucket_pack)
//   exchange  NNL_COMM_NCCL : ncclAllReduce(sum) in place (ring / NVLS order)
//             NNL_COMM_EXACT: the reference's rank-ordered fold, bit-exact
//               (R9): every rank owns one 1/W slice of the bucket; grouped
//               ncclSend/ncclRecv hand it each peer's copy of that slice
//               (the reduce-scatter's traffic), a kernel folds
//               ((b0 + b1) + b2) + ... in ascending rank order, and an
//               in-place ncclAllGather returns the folded slices (the
//               all-gather's traffic): the same bytes as a ring all-reduce.
//   unpack    grad = q(sum / f32(W)), OR of non-finite results (k_bucket_unpack)
// Everything is stream-ordered and CUDA-graph capturable.
#include <dlfcn.h>

#include <mutex>

#include "common.cuh"
#include "nccl.h"

namespace nnl {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;
std::string g_nccl_why;

void load_nccl() {
  // the process's NCCL first (torch loads libnccl.so.2 before any comm exists)
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  const char* env = getenv("NNL_NCCL_LIB");
  if (!h && env) h = dlopen(env, RTLD_NOW);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW);
  if (!h) {
    g_nccl_why = std::string("libnccl not found: ") + (dlerror() ? dlerror() : "?");
    return;
  }
#define NNL_SYM(field, name)                                                   \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));     \
  if (!g_nccl.field) {                                                          \
    g_nccl_why = "libnccl lacks " name;                                         \
    return;                                                                     \
  }
  NNL_SYM(GetUniqueId, "ncclGetUniqueId")
  NNL_SYM(CommInitRank, "ncclCommInitRank")
  NNL_SYM(CommDestroy, "ncclCommDestroy")
  NNL_SYM(AllReduce, "ncclAllReduce")
  NNL_SYM(AllGather, "ncclAllGather")
  NNL_SYM(Send, "ncclSend")
  NNL_SYM(Recv, "ncclRecv")
  NNL_SYM(GroupStart, "ncclGroupStart")
  NNL_SYM(GroupEnd, "ncclGroupEnd")
  NNL_SYM(GetErrorString, "ncclGetErrorString")
#undef NNL_SYM
  g_nccl.ok = true;
}

int nccl_ready() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) return fail(NNL_ERR_UNSUPPORTED, "%s", g_nccl_why.c_str());
  return NNL_OK;
}

#define NNL_NCCL(call)                                                             \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess)                                                         \
      return ::nnl::fail(r_ == ncclSystemError || r_ == ncclRemoteError            \
                             ? NNL_ERR_COLLECTIVE_TIMEOUT : NNL_ERR_CUDA,          \
                         "%s:%d nccl: %s", __FILE__, __LINE__,                     \
                         g_nccl.GetErrorString(r_));                               \
  } while (0)

// acc[i] = ((in[0][i] + in[1][i]) + in[2][i]) + ...  (ascending rank order, f32)
__global__ void k_fold_ranks(const float* __restrict__ in, int32_t world, int64_t pitch,
                             int64_t n, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = in[i];
    for (int32_t r = 1; r < world; ++r) acc = __fadd_rn(acc, in[(int64_t)r * pitch + i]);
    out[i] = acc;
  }
}

}  // namespace
}  // namespace nnl

using namespace nnl;

struct nnl_comm {
  ncclComm_t nc;
  int world, rank, mode;
};

extern "C" {

int nnl_comm_unique_id(void* id_out) {
  if (!id_out) return fail(NNL_ERR_INVALID_ARGUMENT, "null id buffer");
  int rc = nccl_ready();
  if (rc) return rc;
  ncclUniqueId id;
  NNL_NCCL(g_nccl.GetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return NNL_OK;
}

int nnl_comm_init(nnl_comm** out, int32_t world, int32_t rank, const void* unique_id,
                  int32_t mode) {
  if (!out || !unique_id) return fail(NNL_ERR_INVALID_ARGUMENT, "null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(NNL_ERR_INVALID_ARGUMENT, "rank %d of world %d", rank, world);
  if (mode != NNL_COMM_NCCL && mode != NNL_COMM_EXACT)
    return fail(NNL_ERR_INVALID_ARGUMENT, "unknown comm mode %d", mode);
  int rc = nccl_ready();
  if (rc) return rc;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  nnl_comm* c = new nnl_comm{nullptr, world, rank, mode};
  ncclResult_t r = g_nccl.CommInitRank(&c->nc, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(NNL_ERR_COLLECTIVE_TIMEOUT, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  }
  *out = c;
  return NNL_OK;
}

int nnl_comm_destroy(nnl_comm* c) {
  if (!c) return NNL_OK;
  ncclResult_t r = g_nccl.ok ? g_nccl.CommDestroy(c->nc) : ncclSuccess;
  delete c;
  if (r != ncclSuccess) return fail(NNL_ERR_CUDA, "ncclCommDestroy: %s", g_nccl.GetErrorString(r));
  return NNL_OK;
}

int64_t nnl_comm_bucket_elems(const nnl_comm* c, int64_t n) {
  if (!c || c->mode != NNL_COMM_EXACT) return n;
  const int64_t slice = (n + c->world - 1) / c->world;
  return slice * c->world;
}

size_t nnl_comm_workspace_size(const nnl_comm* c, int64_t n) {
  if (!c || c->mode != NNL_COMM_EXACT) return 0;
  const int64_t slice = (n + c->world - 1) / c->world;
  return (size_t)slice * c->world * sizeof(float);
}

int nnl_comm_allreduce_sum_f32(nnl_comm* c, float* buf, int64_t n, void* stream) {
  if (!c) return fail(NNL_ERR_INVALID_ARGUMENT, "null comm");
  if (n <= 0) return NNL_OK;
  NNL_NCCL(g_nccl.AllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, c->nc, as_stream(stream)));
  return NNL_OK;
}

int nnl_comm_allreduce_mean(nnl_comm* c, const nnl_param_slot* slots, const nnl_chunk* chunks,
                            const int64_t* chunk_pos, int32_t n_chunks, float* bucket, int64_t n,
                            int32_t divide, int32_t* nonfinite, void* ws, size_t ws_bytes,
                            void* stream) {
  if (!c) return fail(NNL_ERR_INVALID_ARGUMENT, "null comm");
  cudaStream_t st = as_stream(stream);
  int rc = nnl_bucket_pack(slots, chunks, chunk_pos, n_chunks, bucket, stream);
  if (rc) return rc;
  const int W = c->world;
  if (W > 1 && n > 0) {
    if (c->mode == NNL_COMM_NCCL) {
      NNL_NCCL(g_nccl.AllReduce(bucket, bucket, (size_t)n, ncclFloat32, ncclSum, c->nc, st));
    } else {
      const int64_t slice = (n + W - 1) / W;
      if (ws_bytes < (size_t)slice * W * sizeof(float) || !ws)
        return fail(NNL_ERR_INVALID_ARGUMENT, "exact all-reduce workspace too small");
      float* in = static_cast<float*>(ws);  // [W][slice]: every rank's copy of my slice
      // the bucket is padded to W*slice elements (nnl_comm_bucket_elems); the
      // pad is never unpacked, so whatever it holds only flows through the pad
      NNL_NCCL(g_nccl.GroupStart());
      for (int p = 0; p < W; ++p) {
        if (p == c->rank) continue;
        NNL_NCCL(g_nccl.Send(bucket + (int64_t)p * slice, (size_t)slice, ncclFloat32, p, c->nc, st));
        NNL_NCCL(g_nccl.Recv(in + (int64_t)p * slice, (size_t)slice, ncclFloat32, p, c->nc, st));
      }
      NNL_NCCL(g_nccl.GroupEnd());
      NNL_CUDA(cudaMemcpyAsync(in + (int64_t)c->rank * slice, bucket + (int64_t)c->rank * slice,
                               slice * sizeof(float), cudaMemcpyDeviceToDevice, st));
      launch_k(k_fold_ranks, grid_for(slice, 256), 256, 0, st, in, W, slice, slice,
                                                         bucket + (int64_t)c->rank * slice);
      NNL_CHECK_LAUNCH();
      NNL_NCCL(g_nccl.AllGather(bucket + (int64_t)c->rank * slice, bucket, (size_t)slice,
                                ncclFloat32, c->nc, st));
    }
  }
  return nnl_bucket_unpack_mean(slots, chunks, chunk_pos, n_chunks, bucket, divide ? W : 1,
                                nonfinite, stream);
}

}  // extern "C"
