// Test double for NCCL: every rank of a communicator is a thread of ONE process driving the same
// GPU (gpurun boxes have one GPU; NCCL refuses two ranks on one device).  Loaded by libspchol.so
// in place of libnccl.so.2 when SPCHOL_NCCL_LIB points here (tests/test_gpu_parity.py), so the
// library's real multi-GPU code path — communicator splits, the grouped send/recv exchanges of the
// update blocks, the block-column broadcasts, the solve's reduces / broadcasts / all-reduce, in the
// order the library issues them — runs unchanged.  Point-to-point calls inside ncclGroupStart/End
// are deferred to ncclGroupEnd, which posts every send before it waits for any receive (the NCCL
// group semantics that make an all-to-all exchange deadlock-free).  Semantics are blocking: a call synchronizes the caller's stream, meets the other
// members of its communicator at a rendezvous keyed by (communicator, call sequence number), the
// last arrival moves the data through host memory, and everyone returns.  Calls issued in a
// different order on different ranks deadlock here exactly as they would under NCCL (the test
// runs with a timeout).  Test infrastructure only; implements the symbols libspchol.so uses.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

namespace {
struct Comm;
struct Slot {                       // one collective call of one communicator
  int arrived = 0, left = 0;
  bool done = false;
  std::vector<const void*> send;
  std::vector<void*> recv;
  std::vector<cudaStream_t> streams;
  std::vector<int> color, key;      // ncclCommSplit
  std::vector<Comm*> made;          // ncclCommSplit results, per member
};
struct Group {                      // the shared state of one communicator (all members)
  int n = 0;
  std::vector<int> world_ranks;     // member i -> rank in the root communicator
  std::map<long long, Slot> slots;  // by call sequence number
};
struct Comm {
  std::shared_ptr<Group> g;
  int rank = 0;
  long long seq = 0;
  std::map<int, long long> sseq, rseq;   // point-to-point sequence numbers per peer
};
std::mutex mu;
std::condition_variable cv;
std::map<unsigned long long, std::shared_ptr<Group>> pending_roots;   // by unique id
unsigned long long next_id = 1;

size_t type_size(int t) { return (t == 8 || t == 5 || t == 4) ? 8 : 4; }

// Meet the other members at this communicator's next call; the last arrival runs `act` with the
// lock held, then each member runs `after` (lock held) and returns.
template <class Fill, class Act, class After>
int rendezvous(Comm* c, Fill fill, Act act, After after) {
  std::unique_lock<std::mutex> lk(mu);
  Group& g = *c->g;
  const long long s = c->seq++;
  Slot& sl = g.slots[s];
  if (sl.send.empty()) {
    sl.send.assign(g.n, nullptr);
    sl.recv.assign(g.n, nullptr);
    sl.streams.assign(g.n, nullptr);
    sl.color.assign(g.n, -1);
    sl.key.assign(g.n, 0);
    sl.made.assign(g.n, nullptr);
  }
  fill(sl, c->rank);
  if (++sl.arrived == g.n) {
    act(sl);
    sl.done = true;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return sl.done; });
  }
  after(sl, c->rank);
  if (++sl.left == g.n) g.slots.erase(s);
  return 0;
}
template <class Fill, class Act>
int rendezvous(Comm* c, Fill fill, Act act) {
  return rendezvous(c, fill, act, [](Slot&, int) {});
}

int sync(cudaStream_t st) { return cudaStreamSynchronize(st) == cudaSuccess ? 0 : 1; }
// cudaMemcpy device-to-device returns before the copy has finished (it runs on the legacy default
// stream, which the library's non-blocking streams do not wait for): wait for it explicitly.
void d2d_done() { cudaStreamSynchronize(0); }

void reduce_into(Slot& sl, int n, size_t cnt, int type, int op, void* dst) {
  std::vector<double> acc(cnt, 0.0), tmp(cnt);
  std::vector<unsigned long long> accu(cnt, ~0ULL), tmpu(cnt);
  for (int i = 0; i < n; ++i) {
    if (type == 8) {
      cudaMemcpy(tmp.data(), sl.send[i], cnt * 8, cudaMemcpyDeviceToHost);
      for (size_t e = 0; e < cnt; ++e) acc[e] += tmp[e];
    } else {
      cudaMemcpy(tmpu.data(), sl.send[i], cnt * 8, cudaMemcpyDeviceToHost);
      for (size_t e = 0; e < cnt; ++e) accu[e] = op == 3 ? std::min(accu[e], tmpu[e]) : accu[e] + tmpu[e];
    }
  }
  if (type == 8) cudaMemcpy(dst, acc.data(), cnt * 8, cudaMemcpyHostToDevice);
  else cudaMemcpy(dst, accu.data(), cnt * 8, cudaMemcpyHostToDevice);
}
}  // namespace

extern "C" {
int ncclGetUniqueId(void* id) {
  std::lock_guard<std::mutex> lk(mu);
  std::memset(id, 0, 128);
  const unsigned long long v = next_id++;
  std::memcpy(id, &v, sizeof(v));
  return 0;
}

typedef struct { char internal[128]; } mockUniqueId;

int ncclCommInitRank(void** comm, int nranks, mockUniqueId id, int rank) {
  unsigned long long key;
  std::memcpy(&key, id.internal, sizeof(key));
  std::unique_lock<std::mutex> lk(mu);
  auto& g = pending_roots[key];
  if (!g) {
    g = std::make_shared<Group>();
    g->n = nranks;
    for (int i = 0; i < nranks; ++i) g->world_ranks.push_back(i);
  }
  Comm* c = new Comm{g, rank, 0};
  *comm = c;
  return 0;
}

int ncclCommSplit(void* comm, int color, int key, void** newcomm, void* /*config*/) {
  Comm* c = (Comm*)comm;
  return rendezvous(
      c, [&](Slot& sl, int r) { sl.color[r] = color; sl.key[r] = key; },
      [&](Slot& sl) {
        const int n = c->g->n;
        std::map<int, std::vector<int>> by;   // colour -> members, ordered by key (then rank)
        for (int i = 0; i < n; ++i) if (sl.color[i] >= 0) by[sl.color[i]].push_back(i);
        for (auto& kv : by) {
          auto& v = kv.second;
          std::stable_sort(v.begin(), v.end(), [&](int a, int b) { return sl.key[a] < sl.key[b]; });
          auto g = std::make_shared<Group>();
          g->n = (int)v.size();
          for (int i : v) g->world_ranks.push_back(c->g->world_ranks[i]);
          for (int j = 0; j < (int)v.size(); ++j) sl.made[v[j]] = new Comm{g, j, 0};
        }
      },
      [&](Slot& sl, int r) { *newcomm = sl.made[r]; });
}
}

extern "C" int ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, int type, int op, void* comm,
                             cudaStream_t st) {
  if (sync(st)) return 1;
  Comm* c = (Comm*)comm;
  return rendezvous(
      c, [&](Slot& sl, int r) { sl.send[r] = sendbuff; sl.recv[r] = recvbuff; },
      [&](Slot& sl) {
        const int n = c->g->n;
        // reduce into a scratch device buffer first (send and recv may alias)
        void* scratch = nullptr;
        cudaMalloc(&scratch, std::max<size_t>(1, count * type_size(type)));
        reduce_into(sl, n, count, type, op, scratch);
        for (int i = 0; i < n; ++i) cudaMemcpy(sl.recv[i], scratch, count * type_size(type), cudaMemcpyDeviceToDevice);
        d2d_done();
        cudaFree(scratch);
      });
}

extern "C" int ncclReduce(const void* sendbuff, void* recvbuff, size_t count, int type, int op, int root, void* comm,
                          cudaStream_t st) {
  if (sync(st)) return 1;
  Comm* c = (Comm*)comm;
  return rendezvous(
      c, [&](Slot& sl, int r) { sl.send[r] = sendbuff; sl.recv[r] = recvbuff; },
      [&](Slot& sl) {
        void* scratch = nullptr;
        cudaMalloc(&scratch, std::max<size_t>(1, count * type_size(type)));
        reduce_into(sl, c->g->n, count, type, op, scratch);
        cudaMemcpy(sl.recv[root], scratch, count * type_size(type), cudaMemcpyDeviceToDevice);
        d2d_done();
        cudaFree(scratch);
      });
}

extern "C" int ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count, int type, int root, void* comm,
                             cudaStream_t st) {
  if (sync(st)) return 1;
  Comm* c = (Comm*)comm;
  return rendezvous(
      c, [&](Slot& sl, int r) { sl.send[r] = sendbuff; sl.recv[r] = recvbuff; },
      [&](Slot& sl) {
        for (int i = 0; i < c->g->n; ++i)
          if (sl.recv[i] != sl.send[root])
            cudaMemcpy(sl.recv[i], sl.send[root], count * type_size(type), cudaMemcpyDeviceToDevice);
        d2d_done();
      });
}

namespace {
struct P2P { bool send; void* buf; size_t bytes; int peer; Comm* c; cudaStream_t st; };
struct Mail { const void* buf; size_t bytes; bool taken = false; };
// mailbox key: (group, src, dst, sequence number of that pair)
std::map<std::tuple<Group*, int, int, long long>, Mail> mailbox;
thread_local int group_depth = 0;
thread_local std::vector<P2P> pending_p2p;

int run_p2p(std::vector<P2P>& ops) {
  for (auto& o : ops) if (sync(o.st)) return 1;
  std::vector<std::tuple<Group*, int, int, long long>> mine;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& o : ops)
      if (o.send) {
        auto key = std::make_tuple(o.c->g.get(), o.c->rank, o.peer, o.c->sseq[o.peer]++);
        mailbox[key] = Mail{o.buf, o.bytes, false};
        mine.push_back(key);
      }
    cv.notify_all();
  }
  for (auto& o : ops) {
    if (o.send) continue;
    std::unique_lock<std::mutex> lk(mu);
    auto key = std::make_tuple(o.c->g.get(), o.peer, o.c->rank, o.c->rseq[o.peer]++);
    cv.wait(lk, [&] { return mailbox.count(key) > 0; });
    Mail& m = mailbox[key];
    if (m.bytes != o.bytes) return 2;
    lk.unlock();
    cudaMemcpy(o.buf, m.buf, o.bytes, cudaMemcpyDeviceToDevice);
        d2d_done();
    lk.lock();
    mailbox[key].taken = true;
    cv.notify_all();
  }
  std::unique_lock<std::mutex> lk(mu);
  for (auto& key : mine) {   // the send buffers stay untouched until the receivers have copied them
    cv.wait(lk, [&] { return mailbox[key].taken; });
    mailbox.erase(key);
  }
  return 0;
}
int p2p(bool send, const void* buf, size_t count, int type, int peer, void* comm, cudaStream_t st) {
  P2P o{send, const_cast<void*>(buf), count * type_size(type), peer, (Comm*)comm, st};
  if (group_depth > 0) { pending_p2p.push_back(o); return 0; }
  std::vector<P2P> one{o};
  return run_p2p(one);
}
}  // namespace

extern "C" int ncclSend(const void* buf, size_t count, int type, int peer, void* comm, cudaStream_t st) {
  return p2p(true, buf, count, type, peer, comm, st);
}
extern "C" int ncclRecv(void* buf, size_t count, int type, int peer, void* comm, cudaStream_t st) {
  return p2p(false, buf, count, type, peer, comm, st);
}
extern "C" int ncclGroupStart() { ++group_depth; return 0; }
extern "C" int ncclGroupEnd() {
  if (--group_depth > 0) return 0;
  std::vector<P2P> ops;
  ops.swap(pending_p2p);
  return ops.empty() ? 0 : run_p2p(ops);
}
// marks this library as the blocking stand-in (libspchol.so then never graph-captures NCCL calls)
extern "C" int spcholMockNcclBlocking() { return 1; }
extern "C" int ncclCommDestroy(void* comm) {
  delete (Comm*)comm;
  return 0;
}
extern "C" const char* ncclGetErrorString(int r) { return r ? "mock nccl error" : "no error"; }
