// engine_lat.cu — the latency build of the engine for small batches.
//
// The same engine (engine.cuh) compiled for one 4-warp block per SM: with no
// occupancy to protect, ptxas may use up to 255 registers, which removes every
// spill from the event loop.  A batch with at most one block per SM (configs 1
// and 2: a dozen instances, or one 100k-request instance per policy pair) runs
// a lone, latency-bound event loop per warp, and this build shortens that
// loop's dependency chain (config 2: 7.26 s -> 6.73 s).  Decisions are
// identical; only register allocation differs.  The engine is compiled in its
// own namespace so its out-of-line device functions do not collide with the
// throughput build's (capi.cu); the kernel context has the same layout.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#define SLOSIM_MIN_BLOCKS 1
#define SLOSIM_ENGINE_ONLY
#define slosim slosim_lat
#include "engine.cuh"
#undef slosim

// `cx` points to a slosim::Ctx (identical layout to slosim_lat::Ctx).
cudaError_t slosim_launch_latency_engine(int grid, const void* cx, char* ws, size_t stride, int64_t cap,
                                         unsigned long long* work, cudaStream_t st) {
    slosim_lat::Ctx c;
    memcpy(&c, cx, sizeof(c));
    slosim_lat::sim_kernel<<<grid, 128, 0, st>>>(c, ws, stride, cap, work);
    return cudaGetLastError();
}

#ifdef SLOSIM_PROF
// Section-profile counters of the latency build (summed with the throughput build's by slosim_prof_read).
cudaError_t slosim_lat_prof_read(unsigned long long* out16, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out16, slosim_lat::g_prof, 16 * sizeof(unsigned long long));
    if (e == cudaSuccess && reset) {
        unsigned long long z[16] = {0};
        e = cudaMemcpyToSymbol(slosim_lat::g_prof, z, sizeof(z));
    }
    return e;
}
#endif
