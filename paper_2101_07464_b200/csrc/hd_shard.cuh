// Row-sharded operators: for n beyond one
// GPU's HBM every shard (rank) owns a contiguous, tile-aligned row slab of
// every panel and of x / y. The probe's kernels run unchanged on the local
// slab; after each streaming kernel ONE exchange combines what the
// single-CTA stages need:
//   [ group-reduced partial dot products | head payload | status flags ]
// summed over shards (NCCL allreduce over NVLink, or the in-process
// exchange of virtual shards). The head payload (pivot draws, the fold
// head p[0..off], the head rows of newly written panel columns) is written
// only by shard 0, whose slab holds the head rows [0, H); the other shards
// contribute zeros, so the sum is shard 0's value bit for bit, and they
// scatter it into their replica of the head rows. The single-CTA stages then
// run redundantly, with identical inputs, on every shard.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "hd_kernels.cuh"

namespace hd {

// ------------------------------------------------------------- exchange
class Exchange {
 public:
  virtual ~Exchange() = default;
  virtual int size() const = 0;
  // In-place sum over shards of buf[0:count) (device, fp64), ordered on
  // `stream` of shard `rank`. Every shard gets the identical result.
  virtual void allreduce_sum(double* buf, int64_t count, cudaStream_t stream, int rank) = 0;
};

// Shards in one process, one host thread each — virtual shards on one GPU
// (tests) or one process driving several GPUs (each shard's hd_config.device;
// peer access is enabled so the summing kernel reads the other devices'
// buffers over NVLink). Each call: sync the caller's stream, publish the
// buffer, barrier; every shard sums all published buffers in rank order into
// its scratch, barrier, then copies back. No kernel ever waits on another
// shard's kernel.
__global__ void k_sum_shards(const double* const* bufs, int nb, int64_t count, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += bufs[b][i];
    out[i] = v;
  }
}

class LocalExchange final : public Exchange {
 public:
  explicit LocalExchange(int n)
      : n_(n), bufs_(n, nullptr), scratch_(n, nullptr), cap_(n, 0), table_(n, nullptr), devs_(n, 0), peers_(n, 0) {}
  ~LocalExchange() override {
    for (auto p : scratch_) cudaFree(p);
    for (auto p : table_) cudaFree(p);
  }
  int size() const override { return n_; }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t stream, int rank) override {
    check(cudaStreamSynchronize(stream), "exchange sync");
    if (cap_[rank] < count) {
      cudaFree(scratch_[rank]);
      check(cudaMalloc(&scratch_[rank], sizeof(double) * count), "exchange scratch");
      cap_[rank] = count;
    }
    if (!table_[rank]) check(cudaMalloc(&table_[rank], sizeof(double*) * n_), "exchange table");
    bufs_[rank] = buf;
    int dev = 0;
    check(cudaGetDevice(&dev), "device");
    devs_[rank] = dev;
    barrier();
    if (!peers_[rank]) {  // first exchange: reach every other shard's device
      for (int r = 0; r < n_; ++r) {
        int ok = 0;
        if (devs_[r] != dev && cudaDeviceCanAccessPeer(&ok, dev, devs_[r]) == cudaSuccess && ok) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(devs_[r], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else check(e, "peer access");
        }
      }
      peers_[rank] = 1;
    }
    check(cudaMemcpyAsync(table_[rank], bufs_.data(), sizeof(double*) * n_, cudaMemcpyHostToDevice, stream), "table");
    k_sum_shards<<<64, 256, 0, stream>>>(table_[rank], n_, count, scratch_[rank]);
    check(cudaGetLastError(), "k_sum_shards");
    check(cudaStreamSynchronize(stream), "exchange sum");
    barrier();  // every shard has read every buffer
    check(cudaMemcpyAsync(buf, scratch_[rank], sizeof(double) * count, cudaMemcpyDeviceToDevice, stream), "copy");
    check(cudaStreamSynchronize(stream), "exchange copy");
  }

 private:
  static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("hd exchange: ") + what + ": " + cudaGetErrorString(e));
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    const uint64_t gen = gen_;
    if (++arrived_ == n_) {
      arrived_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen_ != gen; });
    }
  }
  int n_;
  std::vector<double*> bufs_, scratch_;
  std::vector<int64_t> cap_;
  std::vector<double**> table_;
  std::vector<int> devs_, peers_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t gen_ = 0;
};

// NCCL over NVLink / NVSwitch: one communicator per operator group, bound at
// run time (dlopen) to the libnccl the process already has (torch's) or the
// system one, so the library itself loads without NCCL. Types and enum values
// come from nccl.h; only the five entry points below are resolved.
class NcclExchange final : public Exchange {
 public:
  NcclExchange(const void* id, int nranks, int rank, int device) : n_(nranks) {
    load();
    cudaSetDevice(device);
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == NCCL_UNIQUE_ID_BYTES, "nccl id size");
    std::memcpy(uid.internal, id, sizeof uid.internal);
    const ncclResult_t rc = init_(&comm_, nranks, uid, rank);
    if (rc != ncclSuccess) throw std::runtime_error(std::string("hd exchange: ncclCommInitRank: ") + err(rc));
  }
  ~NcclExchange() override {
    if (comm_ && destroy_) destroy_(comm_);
  }
  int size() const override { return n_; }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t stream, int) override {
    const ncclResult_t rc = allreduce_(buf, buf, (size_t)count, ncclFloat64, ncclSum, comm_, stream);
    if (rc != ncclSuccess) throw std::runtime_error(std::string("hd exchange: ncclAllReduce: ") + err(rc));
  }
  static void unique_id(void* out) {
    load();
    ncclUniqueId id;
    const ncclResult_t rc = get_id_(&id);
    if (rc != ncclSuccess) throw std::runtime_error(std::string("hd exchange: ncclGetUniqueId: ") + err(rc));
    std::memcpy(out, id.internal, sizeof id.internal);
  }

 private:
  typedef ncclResult_t (*GetIdFn)(ncclUniqueId*);
  typedef ncclResult_t (*InitFn)(ncclComm_t*, int, ncclUniqueId, int);
  typedef ncclResult_t (*AllReduceFn)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                      cudaStream_t);
  typedef ncclResult_t (*DestroyFn)(ncclComm_t);
  typedef const char* (*ErrFn)(ncclResult_t);
  static inline void* lib_ = nullptr;
  static inline GetIdFn get_id_ = nullptr;
  static inline InitFn init_ = nullptr;
  static inline AllReduceFn allreduce_ = nullptr;
  static inline DestroyFn destroy_ = nullptr;
  static inline ErrFn errstr_ = nullptr;
  static std::string err(ncclResult_t rc) { return errstr_ ? errstr_(rc) : ("code " + std::to_string((int)rc)); }
  static void load() {
    if (lib_) return;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      lib_ = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (lib_) break;
    }
    if (!lib_) throw std::runtime_error("hd exchange: libnccl.so.2 not found");
    get_id_ = reinterpret_cast<GetIdFn>(dlsym(lib_, "ncclGetUniqueId"));
    init_ = reinterpret_cast<InitFn>(dlsym(lib_, "ncclCommInitRank"));
    allreduce_ = reinterpret_cast<AllReduceFn>(dlsym(lib_, "ncclAllReduce"));
    destroy_ = reinterpret_cast<DestroyFn>(dlsym(lib_, "ncclCommDestroy"));
    errstr_ = reinterpret_cast<ErrFn>(dlsym(lib_, "ncclGetErrorString"));
    if (!get_id_ || !init_ || !allreduce_ || !destroy_)
      throw std::runtime_error("hd exchange: libnccl lacks the required entry points");
  }
  int n_;
  ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------- shard plan
// Tile-aligned contiguous row ranges: q = ceil(tiles / count) tiles per
// shard, shard r owns rows [r q 256, min((r + 1) q 256, N)). Shard 0 must
// hold the head rows [0, head_rows) and every shard at least one tile.
inline void shard_plan(int64_t N, int count, int rank, int64_t head_rows, int64_t* begin, int64_t* end) {
  if (N < 1 || count < 1 || rank < 0 || rank >= count)
    throw std::invalid_argument("hd_shard_plan: need N >= 1 and 0 <= rank < count");
  const int64_t tiles = (N + kTile - 1) / kTile;
  const int64_t q = (tiles + count - 1) / count;
  if ((int64_t)(count - 1) * q >= tiles)
    throw std::invalid_argument("hd_shard_plan: too many shards for " + std::to_string(N) + " rows");
  if (q * kTile < head_rows)
    throw std::invalid_argument("hd_shard_plan: shard 0 cannot hold the " + std::to_string(head_rows) +
                                " head rows (fewer shards or a smaller capacity)");
  *begin = std::min<int64_t>((int64_t)rank * q * kTile, N);
  *end = std::min<int64_t>((int64_t)(rank + 1) * q * kTile, N);
}

// --------------------------------------------------- pack / unpack kernels
// Items of the head payload: a device fp64 vector (same role on every
// shard, e.g. the fold head or a pivot scalar) or the head rows of one
// panel column (tile-major, dtype T).
struct XItem {
  double* vec = nullptr;  // kind vector
  int64_t len = 0;
  void* pan = nullptr;    // kind panel column
  int64_t K = 0, col = 0;
};

constexpr int kXMaxItems = 4;

struct XArgs {
  const double* partials = nullptr;  // [nslots][ngroups]
  int nslots = 0, ngroups = 0;
  XItem item[kXMaxItems];
  int nitems = 0;
  int* status = nullptr;
  double* X = nullptr;
  int lead = 0;  // shard 0: contributes the head payload
};

__host__ __device__ inline int64_t xitem_len(const XItem& it, int64_t head_rows) {
  return it.pan ? head_rows : it.len;
}

template <typename T>
__global__ void k_xpack(const __grid_constant__ XArgs a, int64_t head_rows) {
  pdl_wait();
  pdl_launch();
  for (int s = threadIdx.x; s < a.nslots; s += blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < a.ngroups; ++g) v += a.partials[(size_t)s * a.ngroups + g];
    a.X[s] = v;
  }
  int64_t o = a.nslots;
  for (int k = 0; k < a.nitems; ++k) {
    const XItem& it = a.item[k];
    const int64_t L = xitem_len(it, head_rows);
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
      double v = 0.0;
      if (a.lead) v = it.pan ? (double)static_cast<const T*>(it.pan)[paddr(i, it.col, it.K)] : it.vec[i];
      a.X[o + i] = v;
    }
    o += L;
  }
  if (threadIdx.x < kStWords) {  // abort / bad-input flags: any shard sets them for all
    const int w = threadIdx.x;
    a.X[o + w] = (w == kStAbort || w == kStBadInput) ? (double)(a.status[w] != 0) : 0.0;
  }
}

template <typename T>
__global__ void k_xunpack(const __grid_constant__ XArgs a, int64_t head_rows) {
  pdl_wait();
  pdl_launch();
  int64_t o = a.nslots;
  for (int k = 0; k < a.nitems; ++k) {
    const XItem& it = a.item[k];
    const int64_t L = xitem_len(it, head_rows);
    if (!a.lead)
      for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
        if (it.pan) static_cast<T*>(it.pan)[paddr(i, it.col, it.K)] = (T)a.X[o + i];
        else it.vec[i] = a.X[o + i];
      }
    o += L;
  }
  if (threadIdx.x == kStAbort || threadIdx.x == kStBadInput)
    if (a.X[o + threadIdx.x] != 0.0) a.status[threadIdx.x] = 1;
}

}  // namespace hd
