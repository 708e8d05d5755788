// spex_hd.h — portability macros for code compiled both by nvcc (the product,
// sm_100a device code) and by g++ (the test-only host emulation build used to
// check control logic on a CPU-only box).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define SPEX_HD __host__ __device__ __forceinline__
#define SPEX_HDNI __host__ __device__ __noinline__ inline
#define SPEX_D __device__ __forceinline__
#else
#define SPEX_HD inline
#define SPEX_HDNI inline
#define SPEX_D inline
#endif

#if defined(__CUDA_ARCH__)
#define SPEX_DEVICE_PASS 1
#else
#define SPEX_DEVICE_PASS 0
#endif

namespace spex {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = long long;

}  // namespace spex
