// nccl_shim.cu -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// An in-process stand-in for the NCCL subset csrc/partition.cu binds with
// dlsym (ncclGetUniqueId / CommInitRank / CommDestroy / AllReduce / AllGather
// / Send / Recv / GroupStart / GroupEnd / GetErrorString).  Every "rank" is
// a host thread of ONE process driving its own dpmrf context (own stream) on
// the same GPU, so the multi-rank NCCL schedule of the partitioned optimize
// -- grouped halo send/recv windows, the counter all-reduce, the in-place
// all-gathers, the cross-stream ordering on one communicator -- runs for
// world > 1 on a single B200 (real NCCL refuses two ranks on one device).
//
// Semantics: stream-ordered like NCCL.  Each collective / group is a host
// rendezvous of all ranks (so a rank calling a different sequence of
// operations than its peers is detected: op kinds, peers, sizes and types
// must match, else the call fails with ncclInvalidUsage); the data moves as
// cudaMemcpyAsync on the RECEIVING rank's stream after a wait on the
// sender's "ready" event, and the sender's stream then waits on the
// receiver's "done" event before it may overwrite the buffer.  All-reduce
// sums in rank order.  Load with DPMRF_NCCL_LIB=<path to this .so>.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <vector>

extern "C" {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef enum {
  ncclSuccess = 0,
  ncclUnhandledCudaError = 1,
  ncclSystemError = 2,
  ncclInternalError = 3,
  ncclInvalidArgument = 4,
  ncclInvalidUsage = 5,
} ncclResult_t;
typedef enum {
  ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclUint64 = 5,
  ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8, ncclBfloat16 = 9
} ncclDataType_t;
typedef enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3, ncclAvg = 4 } ncclRedOp_t;
}

namespace {

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

enum Kind { kSend, kRecv, kAllGather, kAllReduce };

struct Op {
  Kind kind;
  const void* send = nullptr;
  void* recv = nullptr;
  size_t count = 0;
  ncclDataType_t type = ncclUint8;
  int peer = -1;
  cudaStream_t stream = nullptr;
};

struct Shared {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int joined = 0;
  int arrived = 0;
  uint64_t gen = 0;
  bool failed = false;
  std::vector<std::vector<Op>> posted;  // per rank: the ops of the current group
  std::vector<cudaEvent_t> ready, done;
};

struct CommImpl {
  std::shared_ptr<Shared> sh;
  int rank = 0;
  void* tmp = nullptr;  // all-reduce staging (n x count)
  size_t tmp_bytes = 0;
};

std::mutex g_reg_mu;
std::map<std::string, std::shared_ptr<Shared>> g_reg;

thread_local int t_depth = 0;
thread_local std::vector<std::pair<CommImpl*, Op>> t_ops;
thread_local CommImpl* t_last = nullptr;  // this thread's communicator (empty groups)

// all ranks of the communicator; false on a 120 s timeout (a mismatched
// schedule would otherwise hang the test)
bool barrier(Shared& s) {
  std::unique_lock<std::mutex> lk(s.m);
  const uint64_t g = s.gen;
  if (++s.arrived == s.n) {
    s.arrived = 0;
    ++s.gen;
    s.cv.notify_all();
    return !s.failed;
  }
  const bool ok =
      s.cv.wait_for(lk, std::chrono::seconds(120), [&] { return s.gen != g || s.failed; });
  if (!ok) {
    s.failed = true;
    s.cv.notify_all();
    std::fprintf(stderr, "nccl_shim: rendezvous timeout (ranks disagree on the schedule)\n");
  }
  return ok && !s.failed;
}

// a rank found the schedules inconsistent: release every waiter with an error
void fail_all(Shared& s) {
  std::lock_guard<std::mutex> lk(s.m);
  s.failed = true;
  s.cv.notify_all();
}

template <class T>
__global__ void k_sum(const T* tmp, T* out, size_t count, int n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    T acc = tmp[i];
    for (int r = 1; r < n; ++r) acc = acc + tmp[r * count + i];
    out[i] = acc;
  }
}

#define CUOK(x)                                                        \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      std::fprintf(stderr, "nccl_shim: %s: %s\n", #x, cudaGetErrorString(e_)); \
      return ncclUnhandledCudaError;                                   \
    }                                                                  \
  } while (0)

// Execute one group (the calling rank's ops on one communicator).
ncclResult_t run_group(CommImpl* c, std::vector<Op>& ops) {
  Shared& s = *c->sh;
  const int me = c->rank, n = s.n;
  if (ops.empty()) {
    // a rank with nothing to exchange still takes part in the rendezvous
    // (the schedule calls the group on every rank)
    {
      std::lock_guard<std::mutex> lk(s.m);
      s.posted[me].clear();
    }
    for (int i = 0; i < 3; ++i)
      if (!barrier(s)) return ncclSystemError;
    return ncclSuccess;
  }
  cudaStream_t st = ops[0].stream;
  for (const Op& o : ops)
    if (o.stream != st) {
      std::fprintf(stderr, "nccl_shim: one group spans several streams\n");
      return ncclInvalidUsage;
    }
  CUOK(cudaEventRecord(s.ready[me], st));
  {
    std::lock_guard<std::mutex> lk(s.m);
    s.posted[me] = ops;
  }
  if (!barrier(s)) return ncclSystemError;
  // phase 1: pull what this rank receives (on its own stream)
  std::vector<int> readers;  // ranks whose copies read my buffers
  size_t k_ag = 0, k_ar = 0;
  std::map<int, size_t> nth_recv;
  for (const Op& o : ops) {
    if (o.kind == kSend) {
      readers.push_back(o.peer);
      continue;
    }
    if (o.kind == kRecv) {
      // the k-th recv from peer p matches p's k-th send to me
      const size_t k = nth_recv[o.peer]++;
      size_t seen = 0;
      const Op* src = nullptr;
      for (const Op& q : s.posted[o.peer])
        if (q.kind == kSend && q.peer == me && seen++ == k) src = &q;
      if (!src || src->count != o.count || src->type != o.type) {
        std::fprintf(stderr, "nccl_shim: rank %d recv %zu from %d unmatched\n", me, k, o.peer);
        fail_all(s);
        return ncclInvalidUsage;
      }
      CUOK(cudaStreamWaitEvent(st, s.ready[o.peer], 0));
      CUOK(cudaMemcpyAsync(o.recv, src->send, o.count * type_size(o.type),
                           cudaMemcpyDeviceToDevice, st));
      continue;
    }
    // collectives: the k-th of its kind in every rank's group
    const size_t k = o.kind == kAllGather ? k_ag++ : k_ar++;
    std::vector<const Op*> peer_ops(n);
    for (int r = 0; r < n; ++r) {
      size_t seen = 0;
      for (const Op& q : s.posted[r])
        if (q.kind == o.kind && seen++ == k) peer_ops[r] = &q;
      if (!peer_ops[r] || peer_ops[r]->count != o.count || peer_ops[r]->type != o.type) {
        std::fprintf(stderr, "nccl_shim: rank %d collective %zu mismatched at rank %d\n", me, k,
                     r);
        fail_all(s);
        return ncclInvalidUsage;
      }
    }
    const size_t bytes = o.count * type_size(o.type);
    for (int r = 0; r < n; ++r) {
      if (r == me) continue;
      readers.push_back(r);
      CUOK(cudaStreamWaitEvent(st, s.ready[r], 0));
    }
    if (o.kind == kAllGather) {
      char* dst = static_cast<char*>(o.recv);
      for (int r = 0; r < n; ++r) {
        if (dst + r * bytes == peer_ops[r]->send && r == me) continue;  // in place
        CUOK(cudaMemcpyAsync(dst + r * bytes, peer_ops[r]->send, bytes, cudaMemcpyDeviceToDevice,
                             st));
      }
    } else {
      if (c->tmp_bytes < n * bytes) {
        if (c->tmp) CUOK(cudaFree(c->tmp));
        CUOK(cudaMalloc(&c->tmp, n * bytes));
        c->tmp_bytes = n * bytes;
      }
      for (int r = 0; r < n; ++r)
        CUOK(cudaMemcpyAsync(static_cast<char*>(c->tmp) + r * bytes, peer_ops[r]->send, bytes,
                             cudaMemcpyDeviceToDevice, st));
    }
  }
  CUOK(cudaEventRecord(s.done[me], st));
  if (!barrier(s)) return ncclSystemError;
  // phase 2: my stream may overwrite my buffers only after every reader copied
  for (int r : readers) CUOK(cudaStreamWaitEvent(st, s.done[r], 0));
  // all-reduce results (after every peer has read my send buffer: in place is safe)
  k_ar = 0;
  for (const Op& o : ops) {
    if (o.kind != kAllReduce) continue;
    const size_t bytes = o.count * type_size(o.type);
    const dim3 g(static_cast<unsigned>((o.count + 255) / 256 > 1024 ? 1024 : (o.count + 255) / 256 + 0));
    switch (o.type) {
      case ncclUint32:
        k_sum<uint32_t><<<g, 256, 0, st>>>(static_cast<const uint32_t*>(c->tmp),
                                            static_cast<uint32_t*>(o.recv), o.count, n);
        break;
      case ncclInt32:
        k_sum<int32_t><<<g, 256, 0, st>>>(static_cast<const int32_t*>(c->tmp),
                                           static_cast<int32_t*>(o.recv), o.count, n);
        break;
      case ncclUint64:
        k_sum<uint64_t><<<g, 256, 0, st>>>(static_cast<const uint64_t*>(c->tmp),
                                            static_cast<uint64_t*>(o.recv), o.count, n);
        break;
      case ncclFloat64:
        k_sum<double><<<g, 256, 0, st>>>(static_cast<const double*>(c->tmp),
                                          static_cast<double*>(o.recv), o.count, n);
        break;
      default:
        std::fprintf(stderr, "nccl_shim: all-reduce type %d not supported\n", int(o.type));
        return ncclInvalidArgument;
    }
    CUOK(cudaGetLastError());
    (void)bytes;
    if (++k_ar > 1) {
      std::fprintf(stderr, "nccl_shim: one all-reduce per group supported\n");
      return ncclInvalidUsage;
    }
  }
  if (!barrier(s)) return ncclSystemError;  // posted[] may be reused after this
  return ncclSuccess;
}

ncclResult_t submit(ncclComm_t comm, Op op) {
  auto* c = reinterpret_cast<CommImpl*>(comm);
  if (!c) return ncclInvalidArgument;
  if (op.kind == kSend || op.kind == kRecv) {
    if (op.peer < 0 || op.peer >= c->sh->n || op.peer == c->rank) return ncclInvalidArgument;
  }
  if (t_depth > 0) {
    if (!t_ops.empty() && t_ops[0].first != c) {
      std::fprintf(stderr, "nccl_shim: one communicator per group supported\n");
      return ncclInvalidUsage;
    }
    t_ops.emplace_back(c, op);
    return ncclSuccess;
  }
  std::vector<Op> one{op};
  return run_group(c, one);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::random_device rd;
  for (int i = 0; i < 128; ++i) id->internal[i] = static_cast<char>(rd() & 0xFF);
  std::memcpy(id->internal, "SHIM", 4);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  const std::string key(id.internal, 128);
  std::shared_ptr<Shared> sh;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto& slot = g_reg[key];
    if (!slot) {
      slot = std::make_shared<Shared>();
      slot->n = nranks;
      slot->posted.resize(nranks);
      slot->ready.resize(nranks);
      slot->done.resize(nranks);
    }
    sh = slot;
  }
  if (sh->n != nranks) return ncclInvalidUsage;
  CUOK(cudaEventCreateWithFlags(&sh->ready[rank], cudaEventDisableTiming));
  CUOK(cudaEventCreateWithFlags(&sh->done[rank], cudaEventDisableTiming));
  auto* c = new CommImpl;
  c->sh = sh;
  c->rank = rank;
  t_last = c;
  if (!barrier(*sh)) return ncclSystemError;  // like NCCL: returns once every rank joined
  *comm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  auto* c = reinterpret_cast<CommImpl*>(comm);
  if (!c) return ncclSuccess;
  if (c->tmp) cudaFree(c->tmp);
  if (t_last == c) t_last = nullptr;
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  if (op != ncclSum) return ncclInvalidArgument;
  Op o{kAllReduce, send, recv, count, type, -1, stream};
  return submit(comm, o);
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclComm_t comm, cudaStream_t stream) {
  Op o{kAllGather, send, recv, count, type, -1, stream};
  return submit(comm, o);
}

ncclResult_t ncclSend(const void* send, size_t count, ncclDataType_t type, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
  Op o{kSend, send, nullptr, count, type, peer, stream};
  return submit(comm, o);
}

ncclResult_t ncclRecv(void* recv, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  Op o{kRecv, nullptr, recv, count, type, peer, stream};
  return submit(comm, o);
}

ncclResult_t ncclGroupStart() {
  ++t_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (t_depth <= 0) return ncclInvalidUsage;
  if (--t_depth > 0) return ncclSuccess;
  std::vector<std::pair<CommImpl*, Op>> ops;
  ops.swap(t_ops);
  if (ops.empty()) {
    if (!t_last) return ncclSuccess;
    std::vector<Op> none;
    return run_group(t_last, none);
  }
  std::vector<Op> list;
  for (auto& p : ops) list.push_back(p.second);
  return run_group(ops[0].first, list);
}

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error (shim)";
    case ncclInvalidUsage: return "invalid usage (shim: ranks disagree on the schedule)";
    case ncclInvalidArgument: return "invalid argument (shim)";
    case ncclSystemError: return "system error (shim: rendezvous timeout)";
    default: return "error (shim)";
  }
}

}  // extern "C"
