// comm.cuh — the rank-to-rank transport of the row-partitioned (multi-GPU) path.
//
// fine levels are row-partitioned across GPUs; SpMV-family kernels need a
// halo of the input vector (point-to-point), Krylov / K-cycle scalars need an allreduce,
// setup needs a few index exchanges.  Everything the distributed code does goes through
// the three stream-ordered primitives below, so the numerics are identical whichever
// transport carries the bytes:
//
//   * NcclComm   — one process per GPU (torchrun), NCCL send/recv + allgather over
//                  NVLink/NVSwitch; libnccl is resolved at run time (the copy torch loaded).
//   * ThreadComm — R ranks as R host threads of one process, each with its own stream
//                  (and device, if several are given); bytes move by device-to-device
//                  copies ordered with CUDA events.  This is how the partitioned path is
//                  exercised on a single B200 (NCCL refuses two ranks on one GPU).
//
// Deterministic reductions: allreduce is an allgather of per-rank partials followed by a
// sum in rank order on the device, so every rank sees bit-identical scalars and the K-cycle
// branches (device predicates) agree across ranks.
#pragma once

#include <memory>
#include <vector>

#include "runtime.cuh"

namespace aggmg_b200 {

struct CommMsg {
  int peer;
  void* ptr;     // device memory (send: source, recv: destination)
  size_t bytes;  // may be 0 (message still posted, keeps both sides in step)
};

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }

  // Point-to-point: every send must be matched by the peer's recv of the same size in
  // the same call order.  Stream-ordered on the calling thread's library stream; the
  // send buffers may be overwritten by later stream work.
  // st == nullptr: the calling thread's library stream.
  virtual void exchange(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs,
                        cudaStream_t st = nullptr) = 0;
  // out[r * bytes, (r+1) * bytes) = in of rank r (device buffers), stream-ordered.
  virtual void allgather(const void* in, void* out, size_t bytes) = 0;
  virtual const char* kind() const = 0;

  // ---- helpers built on the primitives ----
  // v[0..n) summed over ranks in rank order, in place (device), bit-identical on all ranks.
  void allreduce_sum(double* v, int n);
  void allreduce_sum(int64_t* v, int n);
  // host-side (synchronising) small collectives
  std::vector<int64_t> allgather_host(const std::vector<int64_t>& mine);  // size() * mine.size()
  int64_t allreduce_host_sum(int64_t v);
  int64_t allreduce_host_max(int64_t v);
  void barrier();

 protected:
  int rank_ = 0, size_ = 1;
};

// ---- in-process ranks -------------------------------------------------------------
struct ThreadGroupState;
class ThreadComm : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroupState> g, int rank, int size);
  void exchange(const std::vector<CommMsg>& sends, const std::vector<CommMsg>& recvs,
                cudaStream_t st = nullptr) override;
  void allgather(const void* in, void* out, size_t bytes) override;
  const char* kind() const override { return "threads"; }
  static std::shared_ptr<ThreadGroupState> make_group(int size);

 private:
  std::shared_ptr<ThreadGroupState> g_;
};

// Wake every rank blocked in the group with an error (a rank failed).
void thread_group_abort(ThreadGroupState& g);

// ---- one process per GPU over NCCL -------------------------------------------------
constexpr int kNcclIdBytes = 128;
void nccl_unique_id(char out[kNcclIdBytes]);
std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const char id[kNcclIdBytes]);

}  // namespace aggmg_b200
