// fake_nccl.cpp -- TEST-ONLY stand-in for libnccl.so.2 (loaded by the engine through AB_NCCL_LIB)
// so that the distributed code path of the engine (ab_create_dist, ncclSend/ncclRecv halo and
// force exchange, all-reduces of flags, results and caller-order gathers) runs on ONE GPU with
// several ranks as threads of one process.
//
// (The driver API is used because the engine links its own static CUDA runtime; CUstream and
// cudaStream_t handles are interchangeable.)
// Every rendezvous happens on the HOST: a receive waits (condition variable) for the matching
// send, then copies device-to-device on the receiver's stream after an event of the sender's
// stream; the sender's stream then waits for the copy.  All-reduces synchronise the streams,
// reduce on the host and copy back.  No kernel ever waits on another rank's kernel, so the
// single-GPU constraint (no cross-rank spinning kernels) holds.  Semantics follow NCCL's:
// point-to-point messages between a pair of ranks match in issue order.
#include <cuda.h>  // driver API: one instance per process, interoperable with every runtime copy
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace {

struct Msg {
  const void* src;
  size_t bytes;
  CUevent ready;           // on the sender's stream: data valid
  CUevent done = nullptr;  // on the receiver's stream: copy finished (set by the receiver)
  bool taken = false;
};

struct World {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;  // (src, dst) FIFO
  int inits = 0;  // ncclCommInitRank calls on this id: an id is single-use, as NCCL's
  // all-reduce rendezvous
  int arrived = 0, generation = 0;
  std::vector<std::vector<unsigned char>> data;
  std::vector<unsigned char> result;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<World>> g_worlds;

struct Comm {
  std::shared_ptr<World> w;
  int rank;
};

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  Comm* comm;
  cudaStream_t st;
};
thread_local int t_group = 0;
thread_local std::vector<Op> t_ops;

size_t tsize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t run_ops(std::vector<Op>& ops) {
  // sends first (post), then receives (wait + copy), then wait for our sends to be consumed
  std::vector<std::shared_ptr<Msg>> mine;
  for (Op& o : ops)
    if (o.send) {
      auto m = std::make_shared<Msg>();
      m->src = o.buf;
      m->bytes = o.bytes;
      cuEventCreate(&m->ready, CU_EVENT_DISABLE_TIMING);
      cuEventRecord(m->ready, (CUstream)o.st);
      World& w = *o.comm->w;
      {
        std::lock_guard<std::mutex> lk(w.mu);
        w.box[{o.comm->rank, o.peer}].push_back(m);
      }
      w.cv.notify_all();
      mine.push_back(m);
    }
  for (Op& o : ops)
    if (!o.send) {
      World& w = *o.comm->w;
      std::shared_ptr<Msg> m;
      {
        std::unique_lock<std::mutex> lk(w.mu);
        auto& q = w.box[{o.peer, o.comm->rank}];
        w.cv.wait(lk, [&] { return !q.empty(); });
        m = q.front();
        q.pop_front();
      }
      if (m->bytes != o.bytes) return ncclInvalidUsage;
      cuStreamWaitEvent((CUstream)o.st, m->ready, 0);
      if (o.bytes) cuMemcpyDtoDAsync((CUdeviceptr)o.buf, (CUdeviceptr)m->src, o.bytes, (CUstream)o.st);
      CUevent d;
      cuEventCreate(&d, CU_EVENT_DISABLE_TIMING);
      cuEventRecord(d, (CUstream)o.st);
      {
        std::lock_guard<std::mutex> lk(w.mu);
        m->done = d;
        m->taken = true;
      }
      w.cv.notify_all();
    }
  for (size_t k = 0, s = 0; k < ops.size(); ++k)
    if (ops[k].send) {
      auto& m = mine[s++];
      World& w = *ops[k].comm->w;
      {
        std::unique_lock<std::mutex> lk(w.mu);
        w.cv.wait(lk, [&] { return m->taken; });
      }
      cuStreamWaitEvent((CUstream)ops[k].st, m->done, 0);  // the send buffer is free after the copy
    }
  return ncclSuccess;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static int counter = 0;
  std::memset(id, 0, sizeof(*id));
  std::lock_guard<std::mutex> lk(g_mu);
  std::snprintf(id->internal, sizeof(id->internal), "fake-nccl-%d", ++counter);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  std::string key(id.internal);
  std::shared_ptr<World> w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_worlds[key];
    if (!slot) {
      slot = std::make_shared<World>();
      slot->n = nranks;
      slot->data.resize(nranks);
    }
    if (++slot->inits > nranks) return ncclInvalidUsage;  // a reused unique id
    w = slot;
  }
  *comm = reinterpret_cast<ncclComm_t>(new Comm{w, rank});
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete reinterpret_cast<Comm*>(comm);
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++t_group;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--t_group > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return run_ops(ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  t_ops.push_back(Op{true, const_cast<void*>(buf), count * tsize(t), peer, reinterpret_cast<Comm*>(comm), st});
  if (t_group == 0) {
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_ops(ops);
  }
  return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  t_ops.push_back(Op{false, buf, count * tsize(t), peer, reinterpret_cast<Comm*>(comm), st});
  if (t_group == 0) {
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_ops(ops);
  }
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  World& w = *c->w;
  const size_t bytes = count * tsize(t);
  std::vector<unsigned char> mine(bytes);
  cuStreamSynchronize((CUstream)st);
  if (bytes) cuMemcpyDtoH(mine.data(), (CUdeviceptr)sendbuf, bytes);
  {
    std::unique_lock<std::mutex> lk(w.mu);
    int gen = w.generation;
    w.data[c->rank] = mine;
    if (++w.arrived == w.n) {  // last rank reduces in rank order
      std::vector<unsigned char> r = w.data[0];
      for (int q = 1; q < w.n; ++q)
        for (size_t k = 0; k < count; ++k) {
          if (t == ncclFloat64) {
            double a, b;
            std::memcpy(&a, &r[8 * k], 8), std::memcpy(&b, &w.data[q][8 * k], 8);
            a = op == ncclSum ? a + b : (op == ncclMax ? (a > b ? a : b) : a);
            std::memcpy(&r[8 * k], &a, 8);
          } else if (t == ncclUint64 || t == ncclInt64) {
            unsigned long long a, b;
            std::memcpy(&a, &r[8 * k], 8), std::memcpy(&b, &w.data[q][8 * k], 8);
            a = op == ncclSum ? a + b : (op == ncclMax ? (a > b ? a : b) : a);
            std::memcpy(&r[8 * k], &a, 8);
          } else {
            return ncclInvalidArgument;
          }
        }
      w.result = r;
      w.arrived = 0;
      ++w.generation;
      w.cv.notify_all();
    } else {
      w.cv.wait(lk, [&] { return w.generation != gen; });
    }
    mine = w.result;
  }
  if (bytes) cuMemcpyHtoD((CUdeviceptr)recvbuf, mine.data(), bytes);
  // every rank must have read the result before the next all-reduce overwrites it
  {
    std::unique_lock<std::mutex> lk(w.mu);
    int gen = w.generation;
    if (++w.arrived == w.n) {
      w.arrived = 0;
      ++w.generation;
      w.cv.notify_all();
    } else {
      w.cv.wait(lk, [&] { return w.generation != gen; });
    }
  }
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "fake-nccl error"; }

}  // extern "C"
