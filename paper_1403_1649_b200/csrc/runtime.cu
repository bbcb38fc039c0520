// runtime.cu — process-wide device context for the library.
#include <atomic>
#include <mutex>
#include <vector>

#include "runtime.cuh"

namespace aggmg_b200 {

namespace {

struct Context {
  bool ready = false;
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  double* pinned = nullptr;
  int pinned_n = 0;
  ~Context() {  // rank threads exit: release their stream and staging
    if (!ready) return;
    if (stream) cudaStreamDestroy(stream);
    if (pinned) cudaFreeHost(pinned);
  }
};

// One context per host thread: the library's default user (the C-ABI caller) and every
// rank thread of an in-process distributed run (comm.cu ThreadGroup) get their own stream,
// pinned staging and reduction scratch, so ranks never share ordering state.
Context& ctx() {
  static thread_local Context c;
  return c;
}
std::mutex& ctx_mutex() {
  static std::mutex m;
  return m;
}
std::atomic<int64_t>& launches() {
  static std::atomic<int64_t> n{0};
  return n;
}

struct ProfState {
  int mask = 0;  // bit f set: family f is timed
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  std::vector<double> bytes;  // per recorded pair
  std::vector<int> family;    // per recorded pair
  int used = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
};
ProfState& prof() {
  static thread_local ProfState p;
  return p;
}

}  // namespace

void init_device(int device) {
  Context& c = ctx();
  std::lock_guard<std::mutex> lk(ctx_mutex());
  if (c.ready) return;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw CudaError("no CUDA device available: the aggmg_b200 kernels require a B200 (sm_100a)");
  AGG_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  AGG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    throw CudaError(std::string("aggmg_b200 is built for sm_100a; found ") + prop.name);
  c.device = device;
  c.sms = prop.multiProcessorCount;
  AGG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  AGG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = UINT64_MAX;  // keep freed blocks cached: setup reallocates per level
  AGG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  AGG_CUDA(cudaMallocHost(&c.pinned, 4096 * sizeof(double)));
  c.pinned_n = 4096;
  c.ready = true;
}

void ensure_init() {
  if (!ctx().ready) init_device(0);
}

cudaStream_t stream() {
  ensure_init();
  return ctx().stream;
}
int sm_count() {
  ensure_init();
  return ctx().sms;
}
int current_device() {
  ensure_init();
  return ctx().device;
}

void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  AGG_CUDA(cudaMallocAsync(&p, bytes, stream()));
  return p;
}
void dev_free(void* p) {
  if (!p) return;
  cudaFreeAsync(p, ctx().stream);
}

void sync() { AGG_CUDA(cudaStreamSynchronize(stream())); }

double* pinned_scratch(int n) {
  ensure_init();
  if (n > ctx().pinned_n) throw Error("pinned scratch too small");
  return ctx().pinned;
}

void note_launch() { launches().fetch_add(1, std::memory_order_relaxed); }
void note_launches(int64_t n) { launches().fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return launches().load(); }

void check_launch(const char* file, int line) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw CudaError(std::string("kernel launch failed: ") + cudaGetErrorString(e) + " at " + file +
                    ":" + std::to_string(line));
}

// ---- profiling -------------------------------------------------------------------

void profile_enable(int mask) {
  ProfState& p = prof();
  sync();
  p.mask = mask;
  p.used = 0;
  p.bytes.clear();
  p.family.clear();
}

ProfileScope::ProfileScope(int family, double bytes) : family_(family), slot_(-1) {
  ProfState& p = prof();
  if (family <= 0 || !(p.mask & (1 << family))) return;
  if (p.used == static_cast<int>(p.pool.size())) {
    cudaEvent_t a, b;
    AGG_CUDA(cudaEventCreate(&a));
    AGG_CUDA(cudaEventCreate(&b));
    p.pool.emplace_back(a, b);
  }
  slot_ = p.used++;
  p.bytes.push_back(bytes);
  p.family.push_back(family);
  AGG_CUDA(cudaEventRecord(p.pool[slot_].first, stream()));
}

ProfileScope::~ProfileScope() {
  if (slot_ < 0) return;
  cudaEventRecord(prof().pool[slot_].second, ctx().stream);
}

void profile_read(int family, double* total_ms, int64_t* n, double* bytes) {
  ProfState& p = prof();
  sync();
  double ms = 0.0, by = 0.0;
  int64_t cnt = 0;
  for (int i = 0; i < p.used; ++i) {
    if (p.family[i] != family) continue;
    float t = 0.f;
    AGG_CUDA(cudaEventElapsedTime(&t, p.pool[i].first, p.pool[i].second));
    ms += t;
    by += p.bytes[i];
    ++cnt;
  }
  if (total_ms) *total_ms = ms;
  if (n) *n = cnt;
  if (bytes) *bytes = by;
}

void timer_start() {
  ProfState& p = prof();
  if (!p.t0) {
    AGG_CUDA(cudaEventCreate(&p.t0));
    AGG_CUDA(cudaEventCreate(&p.t1));
  }
  AGG_CUDA(cudaEventRecord(p.t0, stream()));
}

double timer_stop() {
  ProfState& p = prof();
  AGG_CUDA(cudaEventRecord(p.t1, stream()));
  AGG_CUDA(cudaEventSynchronize(p.t1));
  float ms = 0.f;
  AGG_CUDA(cudaEventElapsedTime(&ms, p.t0, p.t1));
  return ms;
}

}  // namespace aggmg_b200
