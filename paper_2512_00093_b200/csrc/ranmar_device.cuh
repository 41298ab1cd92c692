// Device-side constants and helpers shared by the sm_100a kernels.
//
// The generator is the reference's 24-bit integer RANMAR (arXiv 2512.00093,
// Algorithm 2; /root/reference/proj/include/ranmar/core.hpp:17-66):
//   Fibonacci part  x_n = x_{n-97} - x_{n-33}   (mod 2^24)
//   arithmetic part v_n = v_{n-1} + (m - d)      (mod m = 2^24 - 3)
//   output          (x_n - v_n) mod 2^24
//
// Conventions used by every kernel:
//  * Lanes are carried UNMASKED in 32-bit registers and reduced only when a
//    value leaves the kernel: subtraction mod 2^32 preserves residues mod 2^24
//    (the same argument as core.hpp:52-53 and polyring.hpp:62).
//  * "x_n" indexes the Fibonacci sequence of a state so that x_0 is the next
//    value step() produces; for n in [-97, -1], x_n = lane[(i - n) mod 97]
//    (canonicalize, jump.hpp:32-37, with u[k] = x_{k-97}).
#pragma once

#include <atomic>
#include <cstdint>

#include "ranmar_b200.h"

namespace rb {

constexpr int kLongLag = 97;                      // core.hpp:17
constexpr int kShortLag = 33;                     // core.hpp:18
constexpr uint32_t kMask = 0x00FFFFFFu;           // core.hpp:20
constexpr uint32_t kMod = 16777213u;              // core.hpp:22
constexpr uint32_t kDelta = 7654321u;             // core.hpp:23
constexpr uint32_t kStart = 362436u;              // core.hpp:24
constexpr uint32_t kStepA = kMod - kDelta;        // per-step increment of v (core.hpp:61)

// Launch counter behind ranmar_kernel_launches() (incremented by every launcher).
void count_launch(int n = 1);

// Raises a kernel's dynamic shared-memory limit once per device: the attribute
// belongs to the device context, and one process may drive several devices.
template <class Kernel>
inline cudaError_t ensure_smem(Kernel* kernel, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
    if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_relaxed);
    return e;
}

// Status bits OR-ed into the library's device status word.
constexpr uint32_t kStatusBadState = 1u;          // cursor separation / range violated
constexpr uint32_t kStatusInternal = 2u;          // an internal invariant failed (bug)
constexpr uint32_t kStatusBadType = 4u;           // langevin: an atom type outside [0, n_types]

static_assert(sizeof(ranmar_state) == 400, "ranmar_state must match ranmar::RanmarState");

// (v + a) mod m for v, a < m: branch-free as min(t, t - m) on u32.
__device__ __forceinline__ uint32_t add_mod_m(uint32_t v, uint32_t a) {
    const uint32_t t = v + a;
    return min(t, t - kMod);
}

// (v + n * (m - d)) mod m: the arithmetic component after n steps.
__host__ __device__ __forceinline__ uint32_t arith_advance(uint32_t v, uint64_t n) {
    const uint64_t nm = n % kMod;
    return static_cast<uint32_t>((v + nm * kStepA) % kMod);
}

__device__ __forceinline__ bool state_ok(int i, int j, uint32_t v) {
    return static_cast<unsigned>(i) < 97u && static_cast<unsigned>(j) < 97u &&
           (i - j + 97) % 97 == 64 && v < kMod;
}

// Streaming (evict-first) global stores: outputs are written once and are far
// larger than L2, so they should not displace anything.
__device__ __forceinline__ void st_cs(uint32_t* p, uint32_t x) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ void st_cs(float* p, float x) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(x) : "memory");
}
__device__ __forceinline__ void st_cs(double* p, double x) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(x) : "memory");
}

}  // namespace rb
