// Cross-rank sums for D-sharded sessions (BASELINE configs[3]
// "independence-check microbenchmark, sharded across GPUs"). Included by
// engine.cu inside its anonymous namespace (uses Error, CU, HostBuf).
//
// A D-sharded rank holds a contiguous slice of every vector. The projection
// GEMMs then produce per-rank PARTIAL overlaps beta_p = V_p^H C_p / d and
// partial squared residual norms; their sums over ranks are the only data that
// crosses GPUs. The sum is in place and leaves identical bits on every rank,
// so every rank takes the same verdicts and issues the same sequence of
// reductions (a rank-divergent verdict would desynchronise the collective
// stream).
//
// NCCL is resolved with dlopen at first use: inside a PyTorch process the
// already-loaded libnccl.so.2 (torch's bundled build) is reused instead of
// linking a second copy next to it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

struct Reducer {
  virtual ~Reducer() = default;
  // sum `count` doubles of device memory over ranks, in place, ordered on `s`
  void sum(double* dev, int64_t count, cudaStream_t s) {
    if (count > 0) bytes += static_cast<uint64_t>(count) * sizeof(double);
    do_sum(dev, count, s);
  }
  uint64_t bytes = 0;  // payload summed so far (the bench's communication figure)

protected:
  virtual void do_sum(double* dev, int64_t count, cudaStream_t s) = 0;
};

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    // an already-resident copy first (torch's bundled build: the Python layer
    // imports torch before calling here), else the system's; local scope so
    // its symbols do not leak into later loads
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) throw Error(LIECL_B200_CUDA, std::string("cannot load libnccl.so.2: ") + dlerror());
    NcclApi a;
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) throw Error(LIECL_B200_CUDA, std::string("libnccl.so.2 lacks ") + name);
      return p;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(LIECL_B200_CUDA, std::string(what) + ": " + nccl_api().error_string(r));
}

struct NcclReducer final : Reducer {
  ncclComm_t comm = nullptr;
  NcclReducer(const uint8_t* id_bytes, int nranks, int rank) {
    ncclUniqueId id;
    static_assert(sizeof id == NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(&id, id_bytes, sizeof id);
    nccl_check(nccl_api().comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
  }
  ~NcclReducer() override {
    if (comm) nccl_api().comm_destroy(comm);
  }
  void do_sum(double* dev, int64_t count, cudaStream_t s) override {
    if (count <= 0) return;
    nccl_check(nccl_api().all_reduce(dev, dev, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, s),
               "ncclAllReduce");
  }
};

// Host-callback reduction: the caller sums over its ranks (threads or
// processes sharing one device in tests, any transport in general).
struct HostReducer final : Reducer {
  liecl_b200_reduce_fn fn;
  void* user;
  HostBuf<double> h;
  HostReducer(liecl_b200_reduce_fn f, void* u) : fn(f), user(u) {}
  void do_sum(double* dev, int64_t count, cudaStream_t s) override {
    if (count <= 0) return;
    h.ensure(static_cast<size_t>(count));
    CU(cudaMemcpyAsync(h.p, dev, static_cast<size_t>(count) * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (fn(h.p, count, user) != 0) throw Error(LIECL_B200_INTERNAL, "shard reduction callback failed");
    CU(cudaMemcpyAsync(dev, h.p, static_cast<size_t>(count) * sizeof(double), cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));  // h is rewritten by the next call
  }
};

// elements [lo, hi) of a length-D vector held by `rank` of `nranks`
inline void shard_range(int64_t D, int nranks, int rank, int64_t& lo, int64_t& hi) {
  lo = D * rank / nranks;
  hi = D * (rank + 1) / nranks;
}
