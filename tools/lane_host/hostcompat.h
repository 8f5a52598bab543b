// hostcompat.h — compiles the lane engine's per-lane code (csrc/tengine.cuh) as plain host C++
// for the CPU test harness (tools/lane_host/lane_host.cpp).  CUDA qualifiers vanish, the
// round-to-nearest intrinsics become plain IEEE operations (the harness is built with
// -ffp-contract=off, so nothing is fused), and warp-level intrinsics, which the per-lane code
// does not use, abort if reached.  Test infrastructure only.
#pragma once
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define __host__
#define __device__
#define __global__
#define __forceinline__ inline
#define __noinline__ __attribute__((noinline))
#define __launch_bounds__(...)
#define __grid_constant__
#define __shared__ static

struct HostDim3 { unsigned x, y, z; };
static HostDim3 threadIdx = {0, 0, 0}, blockIdx = {0, 0, 0}, blockDim = {32, 1, 1};

static inline double __dadd_rn(double a, double b) { return a + b; }
static inline double __dsub_rn(double a, double b) { return a - b; }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline double __ddiv_rn(double a, double b) { return a / b; }
static inline double __ddiv_rz(double a, double b) {
    // only used as a quotient estimate that is corrected exactly (numerics.cuh ceil_muldiv)
    return a / b;
}
static inline long long __double2ll_rn(double x) { return (long long)rint(x); }
static inline long long __double_as_longlong(double x) { long long r; memcpy(&r, &x, 8); return r; }
static inline double __longlong_as_double(long long x) { double r; memcpy(&r, &x, 8); return r; }
static inline uint64_t __umul64hi(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }
static inline int __clz(int x) { return x ? __builtin_clz((unsigned)x) : 32; }
static inline int __clzll(long long x) { return x ? __builtin_clzll((unsigned long long)x) : 64; }
static inline int __ffs(int x) { return __builtin_ffs(x); }
static inline int __ffsll(long long x) { return __builtin_ffsll(x); }
static inline int __popc(unsigned x) { return __builtin_popcount(x); }
template <class T> static inline T min(T a, T b) { return a < b ? a : b; }
template <class T> static inline T max(T a, T b) { return a > b ? a : b; }

[[noreturn]] static inline void hc_no_warp() { abort(); }
static inline unsigned __ballot_sync(unsigned, int) { hc_no_warp(); }
template <class T> static inline T __shfl_sync(unsigned, T, int) { hc_no_warp(); }
template <class T> static inline T __shfl_xor_sync(unsigned, T, int) { hc_no_warp(); }
static inline void __syncwarp(unsigned = 0xffffffffu) {}
static inline unsigned __activemask() { return 1u; }
static inline unsigned long long atomicAdd(unsigned long long* p, unsigned long long v) {
    unsigned long long o = *p; *p += v; return o;
}
template <class T> static inline T __shfl_up_sync(unsigned, T, int) { hc_no_warp(); }
static inline int __reduce_min_sync(unsigned, int) { hc_no_warp(); }
static inline int __all_sync(unsigned, int) { hc_no_warp(); }
static inline int __any_sync(unsigned, int) { hc_no_warp(); }

// CUDA's vector types (the lane engine's active-set entries)
struct alignas(16) int4 { int x, y, z, w; };
struct alignas(8) int2 { int x, y; };
static inline int4 make_int4(int x, int y, int z, int w) { return int4{x, y, z, w}; }
static inline int2 make_int2(int x, int y) { return int2{x, y}; }
