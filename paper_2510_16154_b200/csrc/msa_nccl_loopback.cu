// msa_nccl_loopback.cu - an in-process stand-in for the NCCL calls the driver makes (test hook,
// environment MSA_NCCL_LOOPBACK=1). Several contexts of one process, each driven by its own host
// thread, form a "world": point-to-point messages and collectives go through host memory with
// host-side rendezvous, so the whole row-slab path (partition, halo plan and exchange on the comm
// stream, interior / boundary K1 split, all-reduced round sums, all-gathered label tables) runs
// and can be checked against a one-context run on a single GPU. Not a transport: every call
// synchronises the stream it is given. Semantics follow NCCL's: sends and receives between a pair
// of ranks match in issue order; Send/Recv inside a group complete at GroupEnd; collectives are
// called by every rank in the same order; AllReduce sums in rank order (deterministic).
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <algorithm>
#include <vector>

#include "msa_internal.h"

namespace {

constexpr char kMagic[8] = {'M', 'S', 'A', 'L', 'O', 'O', 'P', 0};

struct World {
  explicit World(int n) : size(n), coll(n) {}
  const int size;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::vector<char>>> box;  // (src, dst) -> messages
  // collective rendezvous: generation-counted barrier + per-rank host copies
  int arrived = 0;
  long gen = 0;
  std::vector<std::vector<char>> coll;

  void barrier(std::unique_lock<std::mutex>& lk) {
    const long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct Comm {
  std::shared_ptr<World> w;
  int rank;
};

std::mutex g_reg_mu;
std::map<uint64_t, std::weak_ptr<World>> g_reg;

struct P2p {
  Comm* comm;
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  cudaStream_t st;
};
thread_local int t_depth = 0;
thread_local std::vector<P2p> t_ops;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

ncclResult_t run_p2p(std::vector<P2p>& ops) {
  // every buffer is ready once the streams the ops were issued on have drained
  for (const P2p& o : ops)
    if (cudaStreamSynchronize(o.st) != cudaSuccess) return ncclUnhandledCudaError;
  for (const P2p& o : ops) {  // post all sends first (host copies: the sender may move on)
    if (!o.send) continue;
    std::vector<char> msg(o.bytes);
    if (o.bytes && cudaMemcpy(msg.data(), o.buf, o.bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      return ncclUnhandledCudaError;
    World& w = *o.comm->w;
    std::lock_guard<std::mutex> lk(w.m);
    w.box[{o.comm->rank, o.peer}].push_back(std::move(msg));
    w.cv.notify_all();
  }
  for (const P2p& o : ops) {
    if (o.send) continue;
    World& w = *o.comm->w;
    std::vector<char> msg;
    {
      std::unique_lock<std::mutex> lk(w.m);
      auto& q = w.box[{o.peer, o.comm->rank}];
      w.cv.wait(lk, [&] { return !q.empty(); });
      msg = std::move(q.front());
      q.pop_front();
    }
    if (msg.size() != o.bytes) return ncclInvalidUsage;
    if (o.bytes && cudaMemcpy(o.buf, msg.data(), o.bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  ops.clear();
  return ncclSuccess;
}

ncclResult_t lb_get_unique_id(ncclUniqueId* id) {
  memset(id, 0, sizeof(*id));
  std::random_device rd;
  const uint64_t key = ((uint64_t)rd() << 32) ^ rd();
  memcpy(id->internal, kMagic, sizeof(kMagic));
  memcpy(id->internal + sizeof(kMagic), &key, sizeof(key));
  return ncclSuccess;
}

ncclResult_t lb_comm_init_rank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (memcmp(id.internal, kMagic, sizeof(kMagic)) != 0 || nranks < 1 || rank < 0 || rank >= nranks)
    return ncclInvalidArgument;
  uint64_t key;
  memcpy(&key, id.internal + sizeof(kMagic), sizeof(key));
  std::shared_ptr<World> w;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    w = g_reg[key].lock();
    if (!w) {
      w = std::make_shared<World>(nranks);
      g_reg[key] = w;
    }
  }
  if (w->size != nranks) return ncclInvalidUsage;
  *comm = reinterpret_cast<ncclComm_t>(new Comm{w, rank});
  return ncclSuccess;
}

ncclResult_t lb_comm_destroy(ncclComm_t comm) {
  delete reinterpret_cast<Comm*>(comm);
  return ncclSuccess;
}

ncclResult_t lb_p2p(bool send, void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                    cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!type_size(t) || peer < 0 || peer >= c->w->size) return ncclInvalidArgument;
  t_ops.push_back({c, send, buf, count * type_size(t), peer, st});
  return t_depth > 0 ? ncclSuccess : run_p2p(t_ops);
}
ncclResult_t lb_send(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  return lb_p2p(true, const_cast<void*>(buf), count, t, peer, comm, st);
}
ncclResult_t lb_recv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  return lb_p2p(false, buf, count, t, peer, comm, st);
}
ncclResult_t lb_group_start() {
  ++t_depth;
  return ncclSuccess;
}
ncclResult_t lb_group_end() {
  if (t_depth <= 0) return ncclInvalidUsage;
  return --t_depth == 0 ? run_p2p(t_ops) : ncclSuccess;
}

// post this rank's send buffer, wait for all ranks, let `combine` read every rank's copy, wait
// again (so no copy is dropped while another rank still reads it), then write recvbuf
template <typename F>
ncclResult_t collective(Comm* c, const void* send, size_t send_bytes, void* recv, size_t recv_bytes, cudaStream_t st,
                        F combine) {
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  World& w = *c->w;
  std::vector<char> mine(send_bytes);
  if (send_bytes && cudaMemcpy(mine.data(), send, send_bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    return ncclUnhandledCudaError;
  std::vector<char> out(recv_bytes);
  {
    std::unique_lock<std::mutex> lk(w.m);
    w.coll[c->rank] = std::move(mine);
    w.barrier(lk);
    combine(w.coll, out);
    w.barrier(lk);
  }
  if (recv_bytes && cudaMemcpy(recv, out.data(), recv_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    return ncclUnhandledCudaError;
  return ncclSuccess;
}

template <typename T>
void sum_into(const std::vector<std::vector<char>>& in, std::vector<char>& out, size_t n) {
  T* o = reinterpret_cast<T*>(out.data());
  for (size_t i = 0; i < n; ++i) o[i] = T(0);
  for (const auto& r : in) {  // rank order
    const T* a = reinterpret_cast<const T*>(r.data());
    for (size_t i = 0; i < n; ++i) o[i] += a[i];
  }
}

ncclResult_t lb_all_reduce(const void* send, void* recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  if (op != ncclSum && !(op == ncclMin && t == ncclUint32)) return ncclInvalidArgument;
  const size_t b = count * type_size(t);
  if (!b && count) return ncclInvalidArgument;
  if (op == ncclMin)  // msa_label_margin: min of float bits as uint32
    return collective(reinterpret_cast<Comm*>(comm), send, b, recv, b, st,
                      [&](const std::vector<std::vector<char>>& in, std::vector<char>& out) {
                        for (size_t k = 0; k < count; ++k) {
                          uint32_t m = 0xffffffffu;
                          for (const auto& r : in) m = std::min(m, reinterpret_cast<const uint32_t*>(r.data())[k]);
                          reinterpret_cast<uint32_t*>(out.data())[k] = m;
                        }
                      });
  return collective(reinterpret_cast<Comm*>(comm), send, b, recv, b, st,
                    [&](const std::vector<std::vector<char>>& in, std::vector<char>& out) {
                      switch (t) {
                        case ncclFloat64: sum_into<double>(in, out, count); break;
                        case ncclFloat32: sum_into<float>(in, out, count); break;
                        case ncclInt32: sum_into<int32_t>(in, out, count); break;
                        case ncclInt64: sum_into<int64_t>(in, out, count); break;
                        case ncclUint64: sum_into<uint64_t>(in, out, count); break;
                        default: break;
                      }
                    });
}

ncclResult_t lb_all_gather(const void* send, void* recv, size_t count, ncclDataType_t t, ncclComm_t comm,
                           cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  const size_t b = count * type_size(t);
  if (!b && count) return ncclInvalidArgument;
  return collective(c, send, b, recv, b * c->w->size, st,
                    [&](const std::vector<std::vector<char>>& in, std::vector<char>& out) {
                      for (size_t r = 0; r < in.size(); ++r)
                        if (b) memcpy(out.data() + r * b, in[r].data(), b);
                    });
}

const char* lb_error_string(ncclResult_t r) { return r == ncclSuccess ? "success (loopback)" : "loopback error"; }
ncclResult_t lb_async_error(ncclComm_t, ncclResult_t* r) {
  *r = ncclSuccess;  // the in-process transport reports its errors synchronously
  return ncclSuccess;
}

}  // namespace

MsaNcclFns msa_nccl_loopback() {
  MsaNcclFns f;
  f.GetUniqueId = lb_get_unique_id;
  f.CommInitRank = lb_comm_init_rank;
  f.CommDestroy = lb_comm_destroy;
  f.Send = lb_send;
  f.Recv = lb_recv;
  f.GroupStart = lb_group_start;
  f.GroupEnd = lb_group_end;
  f.AllReduce = lb_all_reduce;
  f.AllGather = lb_all_gather;
  f.GetErrorString = lb_error_string;
  f.CommGetAsyncError = lb_async_error;
  return f;
}
