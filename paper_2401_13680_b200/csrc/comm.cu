// Library-owned NCCL data plane for segment-row sharding.
//
// One communicator per context (one process per GPU).  NCCL is loaded with
// dlopen at first use, so libpastila.so has no link-time dependency on it and
// shares the process's NCCL when torch already loaded one.  Bootstrap: rank 0
// creates the 128-byte ncclUniqueId (pst_comm_unique_id); the caller
// distributes it (torch.distributed object broadcast) and every rank calls
// pst_comm_init.  All collectives run on the context stream, on device
// buffers, in the order the sharded greedy needs them:
//   per step: all-gather of each rank's (area, index) best -> on-device pick ->
//             broadcast of the chosen profile from its owner;
//   attribution: all-reduce MIN of the per-window minima, then all-reduce MIN
//             of the indices of the ranks holding that minimum (lowest index);
//   profile_max: all-reduce MAX.
// The small device kernels that glue those steps (local best, pick, tie
// indices, curve update) are here too, so no host loop touches per-window data.
#include "common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <climits>

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
  api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
               api.AllGather && api.GetErrorString;
  return api;
}

#define PST_NCCL(call)                                                                 \
  do {                                                                                 \
    ncclResult_t _r = (call);                                                          \
    if (_r != ncclSuccess) {                                                           \
      pst_set_error("NCCL error at %s:%d: %s", __FILE__, __LINE__, nccl().GetErrorString(_r)); \
      return PST_ECUDA;                                                                \
    }                                                                                  \
  } while (0)

int need_nccl() {
  if (!nccl().loaded) {
    pst_set_error("NCCL (libnccl.so.2) could not be loaded");
    return PST_ESTATE;
  }
  return PST_OK;
}

int need_comm(pst_ctx* c) {
  if (!c) {
    pst_set_error("null context");
    return PST_EINVAL;
  }
  if (!c->comm) {
    pst_set_error("no communicator (call pst_comm_init)");
    return PST_ESTATE;
  }
  return PST_OK;
}

// best available local row: (area, global index), smallest area, ties -> lowest index
__global__ void k_local_best(const double* __restrict__ areas, const uint8_t* __restrict__ taken, int64_t rows,
                             int64_t base, double* out2) {
  __shared__ double bv[32];
  __shared__ long long bi[32];
  double v = PST_INF;
  long long idx = LLONG_MAX;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    if (taken[r]) continue;
    const double a = areas[r];
    if (a < v || (a == v && base + r < idx)) {
      v = a;
      idx = base + r;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(FULLMASK, v, o);
    const long long oi = __shfl_xor_sync(FULLMASK, idx, o);
    if (ov < v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = v;
    bi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int wv = 1; wv < (int)(blockDim.x >> 5); ++wv)
      if (bv[wv] < v || (bv[wv] == v && bi[wv] < idx)) {
        v = bv[wv];
        idx = bi[wv];
      }
    out2[0] = v;
    out2[1] = (double)idx;  // exact for indices < 2^53
  }
}

// global pick among the gathered [nranks][2] pairs; marks it taken when it is local
__global__ void k_pick_global(const double* __restrict__ pairs, int nranks, int64_t base, int64_t rows,
                              uint8_t* taken, double* out2) {
  if (threadIdx.x != 0) return;
  double v = PST_INF, idx = 9.0e18;
  for (int r = 0; r < nranks; ++r) {
    const double a = pairs[2 * r], i = pairs[2 * r + 1];
    if (a < v || (a == v && i < idx)) {
      v = a;
      idx = i;
    }
  }
  out2[0] = v;
  out2[1] = idx;
  const int64_t g = (int64_t)idx;
  if (g >= base && g < base + rows) taken[g - base] = 1;
}

__global__ void k_tie_index(const double* __restrict__ lmin, const double* __restrict__ gmin,
                            const int32_t* __restrict__ larg, int64_t base, int64_t N, long long* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = (lmin[j] == gmin[j]) ? (long long)larg[j] + base : LLONG_MAX;
}

__global__ void k_min_into(double* curve, const double* __restrict__ row, int64_t N, int first) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    curve[j] = first ? row[j] : fmin(curve[j], row[j]);
}

int grid_n(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : g > 148 * 16 ? 148 * 16 : g);
}

}  // namespace

extern "C" {

// 128-byte ncclUniqueId for pst_comm_init (rank 0 creates, the caller distributes it)
int pst_comm_unique_id(char* out128) {
  PST_TRY(need_nccl());
  ncclUniqueId id;
  PST_NCCL(nccl().GetUniqueId(&id));
  memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return PST_OK;
}

int pst_comm_init(pst_ctx* c, const char* id128, int nranks, int rank) {
  if (!c) {
    pst_set_error("null context");
    return PST_EINVAL;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    pst_set_error("rank %d out of range [0, %d)", rank, nranks);
    return PST_EINVAL;
  }
  PST_TRY(need_nccl());
  PST_CUDA(cudaSetDevice(c->dev));
  if (c->comm) {
    nccl().CommDestroy((ncclComm_t)c->comm);
    c->comm = nullptr;
  }
  ncclUniqueId id;
  memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm;
  PST_NCCL(nccl().CommInitRank(&comm, nranks, id, rank));
  c->comm = (void*)comm;
  c->comm_size = nranks;
  c->comm_rank = rank;
  return PST_OK;
}

int pst_comm_destroy(pst_ctx* c) {
  if (c && c->comm && nccl().loaded) nccl().CommDestroy((ncclComm_t)c->comm);
  if (c) c->comm = nullptr;
  return PST_OK;
}

// in-place all-reduce of a device buffer; dtype 0 = f64, 1 = i64, 2 = i32; op 0 = min, 1 = max, 2 = sum
int pst_comm_allreduce(pst_ctx* c, void* buf_dev, int64_t count, int dtype, int op) {
  PST_TRY(need_comm(c));
  const ncclDataType_t t = dtype == 0 ? ncclFloat64 : dtype == 1 ? ncclInt64 : ncclInt32;
  const ncclRedOp_t o = op == 0 ? ncclMin : op == 1 ? ncclMax : ncclSum;
  PST_CUDA(cudaSetDevice(c->dev));
  PST_NCCL(nccl().AllReduce(buf_dev, buf_dev, (size_t)count, t, o, (ncclComm_t)c->comm, c->st));
  return PST_OK;
}

int pst_comm_broadcast(pst_ctx* c, void* buf_dev, int64_t bytes, int root) {
  PST_TRY(need_comm(c));
  PST_CUDA(cudaSetDevice(c->dev));
  PST_NCCL(nccl().Broadcast(buf_dev, buf_dev, (size_t)bytes, ncclUint8, root, (ncclComm_t)c->comm, c->st));
  return PST_OK;
}

int pst_comm_allgather(pst_ctx* c, const void* send_dev, void* recv_dev, int64_t bytes_per_rank) {
  PST_TRY(need_comm(c));
  PST_CUDA(cudaSetDevice(c->dev));
  PST_NCCL(nccl().AllGather(send_dev, recv_dev, (size_t)bytes_per_rank, ncclUint8, (ncclComm_t)c->comm, c->st));
  return PST_OK;
}

// ---- device glue of the sharded greedy (no per-window host work) ---------
int pst_local_best_dev(pst_ctx* c, const double* areas_dev, const uint8_t* taken_dev, int64_t rows, int64_t base,
                       double* out2_dev) {
  if (!c) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  k_local_best<<<1, 1024, 0, c->st>>>(areas_dev, taken_dev, rows, base, out2_dev);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

int pst_pick_global_dev(pst_ctx* c, const double* pairs_dev, int nranks, int64_t base, int64_t rows,
                        uint8_t* taken_dev, double* out2_dev) {
  if (!c) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  k_pick_global<<<1, 32, 0, c->st>>>(pairs_dev, nranks, base, rows, taken_dev, out2_dev);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

int pst_tie_index_dev(pst_ctx* c, const double* lmin_dev, const double* gmin_dev, const int32_t* larg_dev,
                      int64_t base, int64_t N, int64_t* out_dev) {
  if (!c) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  k_tie_index<<<grid_n(N), 256, 0, c->st>>>(lmin_dev, gmin_dev, larg_dev, base, N, (long long*)out_dev);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

// curve = row (first) or min(curve, row)
int pst_curve_min_dev(pst_ctx* c, double* curve_dev, const double* row_dev, int64_t N, int first) {
  if (!c) return PST_EINVAL;
  PST_CUDA(cudaSetDevice(c->dev));
  k_min_into<<<grid_n(N), 256, 0, c->st>>>(curve_dev, row_dev, N, first);
  c->launches++;
  PST_CUDA(cudaGetLastError());
  return PST_OK;
}

}  // extern "C"
