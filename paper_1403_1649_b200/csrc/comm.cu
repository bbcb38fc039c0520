// comm.cu — ThreadComm (in-process ranks) and NcclComm (one process per GPU).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "comm.cuh"

namespace aggmg_b200 {

namespace {

__global__ void k_sum_ranks_f64(const double* all, int n, int nranks, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double s = all[k];
  for (int r = 1; r < nranks; ++r) s = __dadd_rn(s, all[static_cast<int64_t>(r) * n + k]);
  out[k] = s;
}
__global__ void k_sum_ranks_i64(const int64_t* all, int n, int nranks, int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t s = 0;
  for (int r = 0; r < nranks; ++r) s += all[static_cast<int64_t>(r) * n + k];
  out[k] = s;
}

}  // namespace

// ---- helpers --------------------------------------------------------------------

void Comm::allreduce_sum(double* v, int n) {
  if (n <= 0 || size_ == 1) return;  // one rank: the sum of one partial is the partial
  DevBuf<double> all(static_cast<int64_t>(n) * size_);
  allgather(v, all.get(), sizeof(double) * n);
  AGG_LAUNCH(k_sum_ranks_f64, grid_for(n, 128), 128, 0, all.get(), n, size_, v);
}

void Comm::allreduce_sum(int64_t* v, int n) {
  if (n <= 0 || size_ == 1) return;
  DevBuf<int64_t> all(static_cast<int64_t>(n) * size_);
  allgather(v, all.get(), sizeof(int64_t) * n);
  AGG_LAUNCH(k_sum_ranks_i64, grid_for(n, 128), 128, 0, all.get(), n, size_, v);
}

std::vector<int64_t> Comm::allgather_host(const std::vector<int64_t>& mine) {
  const int64_t m = static_cast<int64_t>(mine.size());
  std::vector<int64_t> out(static_cast<size_t>(m) * size_);
  if (m == 0) return out;
  DevBuf<int64_t> in(m), all(m * size_);
  in.upload(mine.data(), m);
  allgather(in.get(), all.get(), sizeof(int64_t) * m);
  all.download(out.data(), m * size_);
  sync();
  return out;
}

int64_t Comm::allreduce_host_sum(int64_t v) {
  int64_t s = 0;
  for (int64_t x : allgather_host({v})) s += x;
  return s;
}
int64_t Comm::allreduce_host_max(int64_t v) {
  int64_t s = INT64_MIN;
  for (int64_t x : allgather_host({v})) s = std::max(s, x);
  return s;
}
void Comm::barrier() { (void)allgather_host({0}); }

// ---- ThreadComm -------------------------------------------------------------------
//
// A send posts (pointer, size, "ready" event recorded on the sender's stream) to the
// group mailbox under key (src, dst, seq); the matching recv waits for the post, makes its
// stream wait on "ready", copies device-to-device and posts a "done" event; the sender's
// stream then waits on "done" before anything it enqueues later may touch the buffer.
// Host threads only rendezvous; the GPU work of all ranks stays asynchronous.

struct ThreadGroupState {
  struct Post {
    const void* ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;
    cudaEvent_t done = nullptr;
    bool has_done = false;
  };
  explicit ThreadGroupState(int n) : size(n), send_seq(n * n, 0), recv_seq(n * n, 0) {}
  int size;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::tuple<int, int, int64_t>, Post> posts;
  std::vector<int64_t> send_seq, recv_seq;  // [src * size + dst]
  bool aborted = false;

  template <class Pred>
  void wait(std::unique_lock<std::mutex>& lk, Pred pred) {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(300);
    while (!pred()) {
      if (aborted) throw Error("distributed run aborted: another rank failed");
      if (cv.wait_until(lk, deadline) == std::cv_status::timeout && !pred())
        throw Error("distributed run: rank exchange timed out (mismatched collectives)");
    }
  }
};

std::shared_ptr<ThreadGroupState> ThreadComm::make_group(int size) {
  return std::make_shared<ThreadGroupState>(size);
}

void thread_group_abort(ThreadGroupState& g) {
  std::lock_guard<std::mutex> lk(g.m);
  g.aborted = true;
  g.cv.notify_all();
}

ThreadComm::ThreadComm(std::shared_ptr<ThreadGroupState> g, int rank, int size) : g_(std::move(g)) {
  rank_ = rank;
  size_ = size;
}

void ThreadComm::exchange(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs,
                          cudaStream_t st) {
  ThreadGroupState& g = *g_;
  if (!st) st = stream();
  const int me = rank_;
  // self messages: matched in order, plain stream-ordered copies
  std::vector<const CommMsg*> self_send, self_recv;
  for (const auto& s : sends)
    if (s.peer == me && s.bytes) self_send.push_back(&s);
  for (const auto& r : recvs)
    if (r.peer == me && r.bytes) self_recv.push_back(&r);
  require(self_send.size() == self_recv.size(), "exchange: unmatched self message");
  for (size_t k = 0; k < self_send.size(); ++k) {
    require(self_send[k]->bytes == self_recv[k]->bytes, "exchange: self message size mismatch");
    AGG_CUDA(cudaMemcpyAsync(self_recv[k]->ptr, self_send[k]->ptr, self_send[k]->bytes,
                             cudaMemcpyDeviceToDevice, st));
  }
  std::vector<std::tuple<int, int, int64_t>> my_posts;
  for (const auto& s : sends) {
    if (s.peer == me || !s.bytes) continue;
    cudaEvent_t ev;
    AGG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    AGG_CUDA(cudaEventRecord(ev, st));
    std::lock_guard<std::mutex> lk(g.m);
    const auto key = std::make_tuple(me, s.peer, g.send_seq[me * g.size + s.peer]++);
    ThreadGroupState::Post p;
    p.ptr = s.ptr;
    p.bytes = s.bytes;
    p.ready = ev;
    g.posts[key] = p;
    my_posts.push_back(key);
    g.cv.notify_all();
  }
  for (const auto& r : recvs) {
    if (r.peer == me || !r.bytes) continue;
    std::unique_lock<std::mutex> lk(g.m);
    const auto key = std::make_tuple(r.peer, me, g.recv_seq[r.peer * g.size + me]++);
    g.wait(lk, [&] { return g.posts.count(key) > 0; });
    ThreadGroupState::Post& p = g.posts[key];
    if (p.bytes != r.bytes) {
      g.aborted = true;
      g.cv.notify_all();
      throw Error("exchange: message size mismatch between ranks " + std::to_string(r.peer) +
                  " -> " + std::to_string(me));
    }
    const void* src = p.ptr;
    cudaEvent_t ready = p.ready;
    lk.unlock();
    AGG_CUDA(cudaStreamWaitEvent(st, ready, 0));
    AGG_CUDA(cudaMemcpyAsync(r.ptr, src, r.bytes, cudaMemcpyDeviceToDevice, st));
    cudaEvent_t done;
    AGG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    AGG_CUDA(cudaEventRecord(done, st));
    lk.lock();
    ThreadGroupState::Post& q = g.posts[key];
    q.done = done;
    q.has_done = true;
    g.cv.notify_all();
  }
  for (const auto& key : my_posts) {
    std::unique_lock<std::mutex> lk(g.m);
    g.wait(lk, [&] { return g.posts[key].has_done; });
    ThreadGroupState::Post p = g.posts[key];
    g.posts.erase(key);
    lk.unlock();
    AGG_CUDA(cudaStreamWaitEvent(st, p.done, 0));
    cudaEventDestroy(p.done);
    cudaEventDestroy(p.ready);
  }
}

void ThreadComm::allgather(const void* in, void* out, size_t bytes) {
  std::vector<CommMsg> s, r;
  for (int q = 0; q < size_; ++q) {
    s.push_back({q, const_cast<void*>(in), bytes});
    r.push_back({q, static_cast<char*>(out) + static_cast<size_t>(q) * bytes, bytes});
  }
  exchange(s, r);
}

// ---- NcclComm ------------------------------------------------------------------------
//
// libnccl is resolved with dlopen at first use: under torchrun the process already holds
// the NCCL torch loaded, and RTLD_NOLOAD picks that exact copy (one NCCL per process).

namespace {

typedef struct ncclComm* nccl_comm_t;
struct NcclUid {
  char internal[kNcclIdBytes];
};
enum { kNcclInt8 = 0 };
struct NcclApi {
  int (*get_unique_id)(NcclUid*) = nullptr;
  int (*comm_init_rank)(nccl_comm_t*, int, NcclUid, int) = nullptr;
  int (*comm_destroy)(nccl_comm_t) = nullptr;
  int (*send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.get_unique_id || !api.comm_init_rank || !api.send || !api.recv || !api.all_gather ||
      !api.group_start || !api.group_end)
    throw Error("NCCL (libnccl.so.2) not found: the multi-process path needs NCCL");
  return api;
}

void nccl_check(int rc, const char* what) {
  if (rc != 0) {
    const char* s = nccl().error_string ? nccl().error_string(rc) : "?";
    throw Error(std::string("NCCL ") + what + " failed: " + s);
  }
}

class NcclComm : public Comm {
 public:
  NcclComm(int rank, int size, const char id[kNcclIdBytes]) {
    rank_ = rank;
    size_ = size;
    NcclUid uid;
    std::memcpy(uid.internal, id, kNcclIdBytes);
    ensure_init();
    nccl_check(nccl().comm_init_rank(&comm_, size, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_ && nccl().comm_destroy) nccl().comm_destroy(comm_);
  }
  void exchange(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs,
                cudaStream_t st = nullptr) override {
    if (!st) st = stream();
    std::vector<const CommMsg*> self_send, self_recv;
    for (const auto& s : sends)
      if (s.peer == rank_ && s.bytes) self_send.push_back(&s);
    for (const auto& r : recvs)
      if (r.peer == rank_ && r.bytes) self_recv.push_back(&r);
    require(self_send.size() == self_recv.size(), "exchange: unmatched self message");
    for (size_t k = 0; k < self_send.size(); ++k)
      AGG_CUDA(cudaMemcpyAsync(self_recv[k]->ptr, self_send[k]->ptr, self_send[k]->bytes,
                               cudaMemcpyDeviceToDevice, st));
    nccl_check(nccl().group_start(), "ncclGroupStart");
    for (const auto& s : sends)
      if (s.peer != rank_ && s.bytes)
        nccl_check(nccl().send(s.ptr, s.bytes, kNcclInt8, s.peer, comm_, st), "ncclSend");
    for (const auto& r : recvs)
      if (r.peer != rank_ && r.bytes)
        nccl_check(nccl().recv(r.ptr, r.bytes, kNcclInt8, r.peer, comm_, st), "ncclRecv");
    nccl_check(nccl().group_end(), "ncclGroupEnd");
  }
  void allgather(const void* in, void* out, size_t bytes) override {
    if (!bytes) return;
    nccl_check(nccl().all_gather(in, out, bytes, kNcclInt8, comm_, stream()), "ncclAllGather");
  }
  const char* kind() const override { return "nccl"; }

 private:
  nccl_comm_t comm_ = nullptr;
};

}  // namespace

void nccl_unique_id(char out[kNcclIdBytes]) {
  NcclUid uid;
  nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(out, uid.internal, kNcclIdBytes);
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const char id[kNcclIdBytes]) {
  return std::make_unique<NcclComm>(rank, size, id);
}

}  // namespace aggmg_b200
