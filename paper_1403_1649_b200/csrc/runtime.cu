// runtime.cu — process-wide device context for the library.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <cstring>
#include <list>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "runtime.cuh"

namespace aggmg_b200 {

namespace {

struct Context {
  bool ready = false;
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // halo exchanges that overlap interior rows (dist path)
  cudaStream_t background = nullptr;  // lowest priority: setup's Arnoldi chains under the coarsening
  int prio_main = 0, prio_side = 0;
  double* pinned = nullptr;
  int pinned_n = 0;
  // pinned staging ring for large host <-> device copies
  static constexpr int kStages = 4;
  static constexpr size_t kStageBytes = size_t{32} << 20;
  char* stage[kStages] = {};
  cudaEvent_t stage_ev[kStages] = {};
  char* dstage[kStages] = {};  // device-side landing buffers of the coded value transfers
  ~Context() {  // rank threads exit: release their stream and staging
    if (!ready) return;
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (background) cudaStreamDestroy(background);
    if (pinned) cudaFreeHost(pinned);
    for (int b = 0; b < kStages; ++b) {
      if (stage[b]) cudaFreeHost(stage[b]);
      if (stage_ev[b]) cudaEventDestroy(stage_ev[b]);
      if (dstage[b]) cudaFree(dstage[b]);
    }
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

// Stream-ordered pool growth maps physical memory on demand, and a hierarchy's setup + solve
// allocates tens of GB in hundreds of blocks of many sizes: measured on B200, on-demand
// growth cost up to 0.8 s per c4 step and 0.5 s per c3 step.  pool_reserve(bytes) maps one
// block of that size into the pool (which keeps freed memory: release threshold = max) the
// first time a caller needs more than the pool has ever reserved, so the pool sub-allocates
// instead of growing block by block.  AGGMG_POOL_RESERVE_GB reserves up front at init.
void pool_reserve(size_t bytes) {
  ensure_init();
  static std::mutex m;
  static size_t reserved = 0, requested = 0;
  std::lock_guard<std::mutex> lk(m);
  if (bytes <= requested) return;  // (cudaMemGetInfo stalls now and then: ask only when growing)
  requested = bytes;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return;
  bytes = std::min(bytes, static_cast<size_t>(0.6 * static_cast<double>(fr + reserved)));
  if (bytes <= reserved) return;
  void* p = nullptr;
  cudaStream_t st = ctx().stream;
  if (cudaMallocAsync(&p, bytes, st) == cudaSuccess) {
    cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    reserved = bytes;
  }
  cudaGetLastError();
}

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
  // the main stream at the highest priority, the side stream (setup's Arnoldi chains) at the
  // lowest: the block scheduler then hands freed SMs to the coarsening first
  // (AGGMG_STREAM_PRIO=0: both at the default priority)
  static const bool prio = [] {
    const char* e = std::getenv("AGGMG_STREAM_PRIO");
    return !(e && e[0] == '0');
  }();
  int least = 0, greatest = 0;
  AGG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  c.prio_main = prio ? greatest : 0;
  c.prio_side = prio ? least : 0;
  AGG_CUDA(cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking, c.prio_main));
  cudaMemPool_t pool;
  AGG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = UINT64_MAX;  // keep freed blocks cached: setup reallocates per level
  AGG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  if (const char* r = std::getenv("AGGMG_POOL_RESERVE_GB")) {
    void* p = nullptr;
    const size_t bytes = static_cast<size_t>(std::atof(r) * double(size_t{1} << 30));
    if (bytes && cudaMallocAsync(&p, bytes, c.stream) == cudaSuccess) {
      cudaFreeAsync(p, c.stream);
      cudaStreamSynchronize(c.stream);
    }
    cudaGetLastError();
  }
  AGG_CUDA(cudaMallocHost(&c.pinned, 4096 * sizeof(double)));
  c.pinned_n = 4096;
  c.ready = true;
}

void ensure_init() {
  if (!ctx().ready) init_device(0);
}

namespace {
thread_local cudaStream_t g_redirect = nullptr;
}
StreamRedirect::StreamRedirect(cudaStream_t s) : prev_(g_redirect) { g_redirect = s; }
StreamRedirect::~StreamRedirect() { g_redirect = prev_; }
bool stream_redirected() { return g_redirect != nullptr; }

cudaStream_t stream() {
  ensure_init();
  return g_redirect ? g_redirect : ctx().stream;
}
int sm_count() {
  ensure_init();
  return ctx().sms;
}
cudaStream_t side_stream() {
  ensure_init();
  Context& c = ctx();
  if (!c.side) AGG_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
  return c.side;
}
cudaStream_t background_stream() {
  ensure_init();
  Context& c = ctx();
  if (!c.background)
    AGG_CUDA(cudaStreamCreateWithPriority(&c.background, cudaStreamNonBlocking, c.prio_side));
  return c.background;
}
int current_device() {
  ensure_init();
  return ctx().device;
}

// Large device buffers are recycled per thread context by exact size class.  Setup repeats
// the same allocation pattern every level and every hierarchy, and a stream-ordered
// cudaMallocAsync of a 134 MB block took ~0.8 ms of host time on the B200 box (occasionally
// far more) while the GPU idled behind setup's scalar readbacks.  A recycled block is reused
// on the same stream it was freed on, so stream order keeps every earlier user ahead of the
// new one; blocks freed by another thread go back to the CUDA pool.
namespace {
constexpr size_t kCacheMin = size_t{1} << 20;  // smaller buffers: the CUDA pool is fast enough
struct BlockCache {
  // free blocks by size class, plus their age order: when caching a block would pass the
  // limit the oldest cached blocks are released first, so the cache follows the current
  // working set (setup's many sizes, then a Krylov solve's many equal vectors) instead of
  // pinning whatever filled it first
  std::unordered_map<size_t, std::vector<void*>> free_by_size;
  std::list<std::pair<void*, size_t>> lru;  // oldest first
  std::unordered_map<void*, std::list<std::pair<void*, size_t>>::iterator> where;
  std::unordered_map<void*, size_t> live;  // blocks handed out by this context
  size_t cached = 0;
  size_t limit = 0;
  bool enabled = true;
  BlockCache() {
    const char* e = std::getenv("AGGMG_ALLOC_CACHE");
    enabled = !(e && e[0] == '0');
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) limit = tot / 4;
    if (const char* l = std::getenv("AGGMG_CACHE_LIMIT_MB")) limit = size_t(std::atoll(l)) << 20;
    if (const char* m = std::getenv("AGGMG_CACHE_MAX_BLOCK_MB")) max_block = size_t(std::atoll(m)) << 20;
  }
  size_t max_block = ~size_t{0};
  ~BlockCache() {  // a rank thread exits: hand the cached blocks back
    for (auto& kv : free_by_size)
      for (void* p : kv.second) cudaFree(p);
  }
  void* take(size_t sc) {
    auto it = free_by_size.find(sc);
    if (it == free_by_size.end() || it->second.empty()) return nullptr;
    void* p = it->second.back();
    it->second.pop_back();
    auto w = where.find(p);
    lru.erase(w->second);
    where.erase(w);
    cached -= sc;
    return p;
  }
  void put(void* p, size_t sc) {
    free_by_size[sc].push_back(p);
    lru.emplace_back(p, sc);
    where[p] = std::prev(lru.end());
    cached += sc;
  }
  void evict_oldest(cudaStream_t st) {
    const auto [p, sc] = lru.front();
    lru.pop_front();
    where.erase(p);
    auto& v = free_by_size[sc];
    v.erase(std::find(v.begin(), v.end(), p));
    cached -= sc;
    cudaFreeAsync(p, st);
  }
  void release_all(cudaStream_t st) {
    while (!lru.empty()) evict_oldest(st);
  }
};
BlockCache& bcache() {
  static thread_local BlockCache c;
  return c;
}
size_t size_class(size_t b) {  // 1 MB granularity keeps near-equal requests in one class
  return (b + kCacheMin - 1) / kCacheMin * kCacheMin;
}
}  // namespace

namespace {
// stream-ordered allocation; on failure the cached blocks are handed back and it is retried
void* pool_alloc(size_t bytes, BlockCache& c) {
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, stream());
  if (e == cudaErrorMemoryAllocation && c.cached > 0) {
    cudaGetLastError();
    c.release_all(ctx().stream);
    AGG_CUDA(cudaStreamSynchronize(ctx().stream));
    e = cudaMallocAsync(&p, bytes, stream());
  }
  if (e != cudaSuccess) AGG_CUDA(e);
  return p;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  ensure_init();
  BlockCache& c = bcache();
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream(), &cap);  // a captured allocation must stay a graph node
  if (c.enabled && bytes >= kCacheMin && bytes <= c.max_block && cap == cudaStreamCaptureStatusNone &&
      !g_redirect) {
    const size_t sc = size_class(bytes);
    void* p = c.take(sc);
    if (!p) p = pool_alloc(sc, c);
    c.live[p] = sc;
    return p;
  }
  return pool_alloc(bytes, c);
}
void dev_free(void* p) {
  if (!p) return;
  BlockCache& c = bcache();
  auto it = c.live.find(p);
  if (g_redirect) {  // stream-ordered release on the redirected stream, never re-cached
    if (it != c.live.end()) c.live.erase(it);
    cudaFreeAsync(p, g_redirect);
    return;
  }
  if (it == c.live.end()) {  // small block, or one handed out by another thread
    cudaFreeAsync(p, ctx().stream);
    return;
  }
  const size_t sc = it->second;
  c.live.erase(it);
  if (sc > c.limit) {  // larger than the whole cache: release
    cudaFreeAsync(p, ctx().stream);
    return;
  }
  while (c.cached + sc > c.limit) c.evict_oldest(ctx().stream);
  c.put(p, sc);
}

void sync() { AGG_CUDA(cudaStreamSynchronize(stream())); }

namespace {

constexpr size_t kStagedMin = size_t{8} << 20;  // below this a pageable copy is as fast

// Persistent host worker pool for the staging copies (spawning threads per 32 MB chunk
// costs more than the copy).  run(n, f) calls f(0..n-1) on the workers and the caller.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  template <class F>
  void run(int n, F&& f) {
    if (n <= 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::lock_guard<std::mutex> serial(run_mutex_);  // one parallel region at a time
    std::function<void(int)> job(std::ref(f));
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &job;
      n_ = n;
      next_.store(0);
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m_);
    job_ = nullptr;  // late wakers see no job; workers still inside drain() are counted
    done_cv_.wait(lk, [&] { return pending_ == 0 && active_ == 0; });
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }

 private:
  HostPool() {
    const unsigned hc = std::max(2u, std::thread::hardware_concurrency());
    const int nw = static_cast<int>(std::min(16u, hc)) - 1;
    for (int t = 0; t < nw; ++t)
      workers_.emplace_back([this] {
        uint64_t seen = 0;
        while (true) {
          {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
          }
          drain();
        }
      });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void drain() {
    std::function<void(int)>* job;
    int n;
    {
      std::lock_guard<std::mutex> lk(m_);
      job = job_;
      n = n_;
      if (!job) return;
      ++active_;
    }
    int done = 0;
    for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) {
      (*job)(i);
      ++done;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      pending_ -= done;
      --active_;
      if (pending_ == 0 && active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, run_mutex_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)>* job_ = nullptr;
  int n_ = 0, pending_ = 0, active_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// memcpy over the pool in 1 MB pieces (large pageable sources are bandwidth-bound per core)
void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = size_t{1} << 20;
  const int pieces = static_cast<int>((bytes + kPiece - 1) / kPiece);
  HostPool::get().run(pieces, [&](int p) {
    const size_t lo = kPiece * p, hi = std::min(bytes, lo + kPiece);
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  });
}

Context& staged() {
  Context& c = ctx();
  if (!c.stage[0])
    for (int b = 0; b < Context::kStages; ++b) {
      AGG_CUDA(cudaMallocHost(&c.stage[b], Context::kStageBytes));
      AGG_CUDA(cudaEventCreateWithFlags(&c.stage_ev[b], cudaEventDisableTiming));
      AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));
    }
  return c;
}

}  // namespace

void host_to_device(void* dst, const void* src, size_t bytes) {
  ensure_init();
  if (bytes < kStagedMin) {
    AGG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream()));
    return;
  }
  Context& c = staged();
  size_t off = 0;
  for (int k = 0; off < bytes; ++k) {
    const int b = k % Context::kStages;
    const size_t len = std::min(Context::kStageBytes, bytes - off);
    AGG_CUDA(cudaEventSynchronize(c.stage_ev[b]));  // the DMA that last read this stage is done
    par_memcpy(c.stage[b], static_cast<const char*>(src) + off, len);
    AGG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, c.stage[b], len, cudaMemcpyHostToDevice,
                             c.stream));
    AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));
    off += len;
  }
}

void host_to_device_narrow(int32_t* dst, const int64_t* src, size_t n, int64_t lo, int64_t hi,
                           int64_t* first_bad) {
  ensure_init();
  std::atomic<int64_t> bad{INT64_MAX};
  // narrow [a, b) of src into out over the pool; remember the first index outside [lo, hi)
  auto narrow = [&](int32_t* out, size_t a, size_t b) {
    constexpr size_t kPiece = size_t{1} << 18;
    const int pieces = static_cast<int>((b - a + kPiece - 1) / kPiece);
    HostPool::get().run(pieces, [&](int p) {
      const size_t s0 = a + kPiece * p, s1 = std::min(b, s0 + kPiece);
      bool any_bad = false;
      for (size_t k = s0; k < s1; ++k) {
        const int64_t v = src[k];
        any_bad |= (v < lo) | (v >= hi);
        out[k - a] = static_cast<int32_t>(v);
      }
      if (any_bad) {
        int64_t fb = INT64_MAX;
        for (size_t k = s0; k < s1 && fb == INT64_MAX; ++k)
          if (src[k] < lo || src[k] >= hi) fb = static_cast<int64_t>(k);
        int64_t cur = bad.load();
        while (fb < cur && !bad.compare_exchange_weak(cur, fb)) {
        }
      }
    });
  };
  if (n * sizeof(int32_t) < kStagedMin) {
    std::vector<int32_t> tmp(n);
    narrow(tmp.data(), 0, n);
    if (n) {
      AGG_CUDA(cudaMemcpyAsync(dst, tmp.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, stream()));
      AGG_CUDA(cudaStreamSynchronize(stream()));  // tmp dies here
    }
  } else {
    Context& c = staged();
    const size_t per_chunk = Context::kStageBytes / sizeof(int32_t);
    size_t off = 0;
    for (int k = 0; off < n; ++k) {
      const int b = k % Context::kStages;
      const size_t len = std::min(per_chunk, n - off);
      AGG_CUDA(cudaEventSynchronize(c.stage_ev[b]));
      narrow(reinterpret_cast<int32_t*>(c.stage[b]), off, off + len);
      AGG_CUDA(cudaMemcpyAsync(dst + off, c.stage[b], len * sizeof(int32_t), cudaMemcpyHostToDevice,
                               c.stream));
      AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));
      off += len;
    }
  }
  *first_bad = bad.load() == INT64_MAX ? -1 : bad.load();
}

// ---- fp64 arrays over PCIe as one-byte codes -----------------------------------------------
// A stencil operator's values (and a constant right-hand side) hold a handful of distinct
// doubles.  Each 64 K-value piece is coded on the host while staging — a one-byte code per
// value into the piece's own table of <= 256 distinct bit patterns — and decoded on the device
// into the destination: 8x fewer bytes written into pinned memory and sent over PCIe, the same
// doubles bit for bit.  Pieces with more distinct values travel raw; once most pieces of an
// array fail to code, the rest of the array takes the plain staging path.
namespace {
constexpr int kCodePiece = 1 << 16;  // values per piece
constexpr int kCodePieces = static_cast<int>(Context::kStageBytes / (sizeof(double) * kCodePiece));
struct CodeHeader {
  int32_t coded;  // 1: table + codes in the piece's slot; 0: raw doubles at raw_off
  int32_t ntab;
  int64_t raw_off;
};
constexpr size_t kCodeHdrBytes = sizeof(CodeHeader) * kCodePieces;
constexpr size_t kCodeSlot = 256 * sizeof(double) + kCodePiece;  // table + codes
constexpr size_t kCodeRawBase = kCodeHdrBytes + kCodePieces * kCodeSlot;

__global__ void k_decode_values(const char* stage, int64_t n, double* dst) {
  __shared__ double tab[256];
  const int p = blockIdx.x;
  const CodeHeader h = reinterpret_cast<const CodeHeader*>(stage)[p];
  const int64_t base = static_cast<int64_t>(p) * kCodePiece;
  const int len = static_cast<int>(min(static_cast<int64_t>(kCodePiece), n - base));
  if (h.coded) {
    const double* t = reinterpret_cast<const double*>(stage + kCodeHdrBytes + p * kCodeSlot);
    for (int i = threadIdx.x; i < h.ntab; i += blockDim.x) tab[i] = t[i];
    __syncthreads();
    const unsigned char* codes = reinterpret_cast<const unsigned char*>(t + 256);
    for (int i = threadIdx.x; i < len; i += blockDim.x) dst[base + i] = tab[codes[i]];
  } else {
    const double* raw = reinterpret_cast<const double*>(stage + h.raw_off);
    for (int i = threadIdx.x; i < len; i += blockDim.x) dst[base + i] = raw[i];
  }
}

// one piece: table + codes into slot; false when it holds more than 256 distinct patterns
bool code_piece(const double* src, int len, char* slot, int32_t* ntab_out) {
  double* tab = reinterpret_cast<double*>(slot);
  unsigned char* codes = reinterpret_cast<unsigned char*>(slot + 256 * sizeof(double));
  constexpr int kSlots = 1024;
  uint64_t keys[kSlots];
  unsigned char code_of[kSlots];
  bool used[kSlots] = {};
  int ntab = 0;
  uint64_t last = 0;
  unsigned char last_code = 0;
  bool have_last = false;
  for (int i = 0; i < len; ++i) {
    uint64_t k;
    std::memcpy(&k, src + i, sizeof k);
    if (have_last && k == last) {
      codes[i] = last_code;
      continue;
    }
    unsigned h = static_cast<unsigned>(((k ^ (k >> 29)) * 0x9e3779b97f4a7c15ull) >> 54) & (kSlots - 1);
    while (used[h] && keys[h] != k) h = (h + 1) & (kSlots - 1);
    if (!used[h]) {
      if (ntab == 256) return false;
      used[h] = true;
      keys[h] = k;
      code_of[h] = static_cast<unsigned char>(ntab);
      std::memcpy(tab + ntab, &k, sizeof k);
      ++ntab;
    }
    codes[i] = code_of[h];
    last = k;
    last_code = code_of[h];
    have_last = true;
  }
  *ntab_out = ntab;
  return true;
}
}  // namespace

void host_to_device_values(double* dst, const double* src, size_t n) {
  ensure_init();
  if (n * sizeof(double) < kStagedMin) {
    host_to_device(dst, src, n * sizeof(double));
    return;
  }
  Context& c = staged();
  for (int b = 0; b < Context::kStages; ++b)
    if (!c.dstage[b]) AGG_CUDA(cudaMalloc(&c.dstage[b], Context::kStageBytes));
  const size_t per_chunk = static_cast<size_t>(kCodePieces) * kCodePiece;
  size_t off = 0;
  int64_t raw_pieces = 0, pieces_seen = 0;
  for (int k = 0; off < n; ++k) {
    const int b = k % Context::kStages;
    const size_t len = std::min(per_chunk, n - off);
    const int np = static_cast<int>((len + kCodePiece - 1) / kCodePiece);
    AGG_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    char* st = c.stage[b];
    CodeHeader* hdr = reinterpret_cast<CodeHeader*>(st);
    std::atomic<int64_t> raw_used{0};
    HostPool::get().run(np, [&](int p) {
      const size_t p0 = static_cast<size_t>(p) * kCodePiece;
      const int plen = static_cast<int>(std::min<size_t>(kCodePiece, len - p0));
      int32_t ntab = 0;
      if (code_piece(src + off + p0, plen, st + kCodeHdrBytes + p * kCodeSlot, &ntab)) {
        hdr[p] = CodeHeader{1, ntab, 0};
        return;
      }
      const int64_t at = static_cast<int64_t>(kCodeRawBase) + raw_used.fetch_add(int64_t{8} * plen);
      if (at + int64_t{8} * plen <= static_cast<int64_t>(Context::kStageBytes))
        std::memcpy(st + at, src + off + p0, sizeof(double) * plen);
      hdr[p] = CodeHeader{0, 0, at};
    });
    for (int p = 0; p < np; ++p) raw_pieces += hdr[p].coded ? 0 : 1;
    pieces_seen += np;
    const size_t used = kCodeRawBase + static_cast<size_t>(raw_used.load());
    if (used > Context::kStageBytes) {  // too many raw pieces for one stage: the rest plain
      host_to_device(dst + off, src + off, (n - off) * sizeof(double));
      return;
    }
    AGG_CUDA(cudaMemcpyAsync(c.dstage[b], st, used, cudaMemcpyHostToDevice, c.stream));
    AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));
    k_decode_values<<<np, 256, 0, c.stream>>>(c.dstage[b], static_cast<int64_t>(len), dst + off);
    note_launch();
    check_launch(__FILE__, __LINE__);
    off += len;
    if (pieces_seen >= kCodePieces && 2 * raw_pieces > pieces_seen && off < n) {
      host_to_device(dst + off, src + off, (n - off) * sizeof(double));  // general values
      return;
    }
  }
}

void device_to_host(void* dst, const void* src, size_t bytes) {
  ensure_init();
  if (bytes < kStagedMin) {
    AGG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream()));
    return;
  }
  Context& c = staged();
  // issue the DMAs of the first stages, then drain in order while refilling
  const size_t nchunks = (bytes + Context::kStageBytes - 1) / Context::kStageBytes;
  auto issue = [&](size_t k) {
    const int b = static_cast<int>(k % Context::kStages);
    const size_t off = k * Context::kStageBytes, len = std::min(Context::kStageBytes, bytes - off);
    AGG_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    AGG_CUDA(cudaMemcpyAsync(c.stage[b], static_cast<const char*>(src) + off, len,
                             cudaMemcpyDeviceToHost, c.stream));
    AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));
  };
  size_t issued = 0;
  for (; issued < nchunks && issued < static_cast<size_t>(Context::kStages); ++issued) issue(issued);
  for (size_t k = 0; k < nchunks; ++k) {
    const int b = static_cast<int>(k % Context::kStages);
    const size_t off = k * Context::kStageBytes, len = std::min(Context::kStageBytes, bytes - off);
    AGG_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    par_memcpy(static_cast<char*>(dst) + off, c.stage[b], len);
    AGG_CUDA(cudaEventRecord(c.stage_ev[b], c.stream));  // stage free again (host done with it)
    if (issued < nchunks) issue(issued++);
  }
}

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
