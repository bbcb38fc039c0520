// common.cuh — shared device/host definitions for the B200-native aggmg library.
//
// Device storage: int32 row offsets / column indices, fp64 values.
// The host API keeps the reference's int64 indices (reference types.hpp:12).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace aggmg_b200 {

using idx = int32_t;  // device index type (rows, columns, nnz positions)

// aggmg::Error equivalent (reference error.hpp:14-17): message text is surfaced
// through aggmg_last_error() by the C-ABI layer.
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw Error(msg);
}
inline void require(bool cond, const char* msg) {
  if (!cond) throw Error(msg);
}

#define AGG_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::aggmg_b200::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                    " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Launch bookkeeping: every kernel goes through AGG_LAUNCH so the library can
// report how many of its own kernels ran (bench.py "gpu_launches").
void note_launch();
void note_launches(int64_t n);  // graph replays: n kernels launched by one cudaGraphLaunch
void check_launch(const char* file, int line);

#define AGG_LAUNCH(kernel, grid, block, smem, ...)                                   \
  do {                                                                               \
    kernel<<<(grid), (block), (smem), ::aggmg_b200::stream()>>>(__VA_ARGS__);        \
    ::aggmg_b200::note_launch();                                                     \
    ::aggmg_b200::check_launch(__FILE__, __LINE__);                                  \
  } while (0)

cudaStream_t stream();
int sm_count();

inline unsigned grid_for(int64_t n, int block, int64_t cap = 0) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (cap > 0 && g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---- counter-based RNG, bit-identical to reference rng.hpp:14-34 ----------------
__host__ __device__ inline uint64_t hash_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t keyed_bits(uint64_t seed, uint64_t counter) {
  return hash_mix(hash_mix(seed) ^ counter);
}
// (bits>>11 + 0.5) * 2^-53, evaluated with explicit round-to-nearest ops so no
// contraction can change the result (reference rng.hpp:26-29).
__host__ __device__ inline double uniform_open01(uint64_t seed, uint64_t counter) {
  const uint64_t bits = keyed_bits(seed, counter) >> 11;
#ifdef __CUDA_ARCH__
  return __dmul_rn(__dadd_rn(static_cast<double>(bits), 0.5), 0x1.0p-53);
#else
  return (static_cast<double>(bits) + 0.5) * 0x1.0p-53;
#endif
}
__host__ __device__ inline double uniform_sym(uint64_t seed, uint64_t counter) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(__dmul_rn(2.0, uniform_open01(seed, counter)), 1.0);
#else
  return 2.0 * uniform_open01(seed, counter) - 1.0;
#endif
}

// per-level seed (reference hierarchy.cpp:25-30)
inline uint64_t level_seed(uint64_t seed, int64_t level, uint64_t tag) {
  return hash_mix(hash_mix(seed ^ tag) ^ static_cast<uint64_t>(level));
}
constexpr uint64_t kMisTag = 0x6d697332;       // hierarchy.cpp:29
constexpr uint64_t kSmootherTag = 0x736d6f6f;  // hierarchy.cpp:30

}  // namespace aggmg_b200
