// runtime.cuh — device context (one stream per process, stream-ordered memory pool),
// RAII device buffers, pinned scalar readback, kernel-family profiling.
#pragma once

#include <atomic>
#include <cstring>
#include <memory>
#include <utility>
#include <vector>

#include "common.cuh"

namespace aggmg_b200 {

void ensure_init();
// Host <-> device copies of pageable host memory.  Large transfers run through a pinned
// staging ring: multi-threaded memcpy into a pinned chunk overlaps the DMA of the previous
// chunk (pageable cudaMemcpy alone reaches ~11 GB/s on the B200 box).  Small ones are plain
// stream-ordered cudaMemcpyAsync.
void host_to_device(void* dst, const void* src, size_t bytes);
// fp64 arrays: large ones cross PCIe as one-byte codes per 64 K-value piece when the piece has
// <= 256 distinct values (decoded on the device, bit-identical); other pieces travel raw
void host_to_device_values(double* dst, const double* src, size_t n);
void device_to_host(void* dst, const void* src, size_t bytes);
// int64 host indices -> int32 device indices, narrowed on the host while staging (halves the
// index bytes on the wire); *first_bad = first position whose value is outside [lo, hi), or -1.
void host_to_device_narrow(int32_t* dst, const int64_t* src, size_t n, int64_t lo, int64_t hi,
                           int64_t* first_bad);
void init_device(int device);  // creates the calling thread's context on `device`
int current_device();
// One-time per-device initialisation (kernel attributes are per device): true until
// mark_device(seen) ran on the calling thread's current device.
inline bool device_pending(const std::atomic<unsigned long long>& seen) {
  return !(seen.load() & (1ull << (current_device() & 63)));
}
inline void mark_device(std::atomic<unsigned long long>& seen) {
  seen.fetch_or(1ull << (current_device() & 63));
}
cudaStream_t side_stream();  // a second stream of the calling thread (overlapped exchanges)
cudaStream_t background_stream();  // a low-priority stream of the calling thread (setup overlap)
// While alive, the calling thread's kernels and stream-ordered allocations go to `s` instead
// of its main stream (work that overlaps the main stream, e.g. the smoother's Arnoldi chains
// during setup).  Allocations made inside bypass the per-thread block cache, whose reuse rule
// assumes a single stream; the reduction scratch switches to a second set.
class StreamRedirect {
 public:
  explicit StreamRedirect(cudaStream_t s);
  ~StreamRedirect();
  StreamRedirect(const StreamRedirect&) = delete;
  StreamRedirect& operator=(const StreamRedirect&) = delete;

 private:
  cudaStream_t prev_;
};
bool stream_redirected();
void* dev_alloc(size_t bytes);
// Make sure the stream-ordered pool holds at least `bytes` of mapped memory (capped at 60% of
// what the device has left); setup calls it with its working-set estimate.
void pool_reserve(size_t bytes);
void dev_free(void* p);

// Move-only device array allocated from the stream-ordered pool.
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(int64_t n) { resize(n); }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { reset(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void resize(int64_t n) {
    reset();
    n_ = n;
    // +32 bytes of tail padding: vectorised loads may read past the end of a row block
    if (n > 0) p_ = static_cast<T*>(dev_alloc(sizeof(T) * static_cast<size_t>(n) + 32));
  }
  void reset() {
    if (p_) dev_free(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  int64_t size() const { return n_; }
  void zero() const {
    if (n_ > 0) AGG_CUDA(cudaMemsetAsync(p_, 0, sizeof(T) * n_, stream()));
  }
  void upload(const T* h, int64_t n) const {
    if (n > 0) host_to_device(p_, h, sizeof(T) * static_cast<size_t>(n));
  }
  // Large downloads complete before returning; small ones are stream-ordered (sync()).
  void download(T* h, int64_t n) const {
    if (n > 0) device_to_host(h, p_, sizeof(T) * static_cast<size_t>(n));
  }
  // device-to-device deep copy of o (stream-ordered)
  void copy_from(const DevBuf& o) {
    resize(o.n_);
    if (n_ > 0) AGG_CUDA(cudaMemcpyAsync(p_, o.p_, sizeof(T) * n_, cudaMemcpyDeviceToDevice, stream()));
  }
  std::vector<T> to_host() const {
    std::vector<T> v(n_);
    download(v.data(), n_);
    AGG_CUDA(cudaStreamSynchronize(stream()));
    return v;
  }

 private:
  T* p_ = nullptr;
  int64_t n_ = 0;
};

void sync();

// Read `count` values of type T from device memory (synchronises the stream).
template <class T>
T read_scalar(const T* dptr) {
  T v;
  AGG_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, stream()));
  AGG_CUDA(cudaStreamSynchronize(stream()));
  return v;
}

// Small pinned staging area for scalar readbacks that avoid pageable copies.
double* pinned_scratch(int n_doubles);

// Kernel-family timing (CUDA events on the library stream).
enum ProfileFamily { kProfNone = 0, kProfSmoothL0 = 1, kProfSpmvL0 = 2, kProfFamilies = 3 };
struct ProfileScope {
  ProfileScope(int family, double bytes);
  ~ProfileScope();
  int family_;
  int slot_;
};
void profile_enable(int mask);  // bit (1 << family) per timed family
void timer_start();
double timer_stop();  // ms on the library stream since timer_start()
void profile_read(int family, double* total_ms, int64_t* launches, double* bytes);
int64_t launch_count();

}  // namespace aggmg_b200
