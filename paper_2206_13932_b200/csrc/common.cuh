// common.cuh -- small device helpers shared by the DMS kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dms {

constexpr int kBlock = 256;  // threads per CTA for the streaming kernels

// Order-preserving uint32 image of a float for the vertex order K (PAPER.md 1368-1372):
// -0 is mapped to +0 so that IEEE equality decides ties (reading Z3), then the usual
// sign-flip trick makes unsigned comparison agree with float comparison.
__device__ __forceinline__ uint32_t ord_of(float v) {
    uint32_t u = __float_as_uint(v);
    if ((u << 1) == 0u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ bool is_nan_bits(float v) { return v != v; }

// K(u) < K(v) from ordered values and vertex ids
__device__ __forceinline__ bool k_less(uint32_t ou, int64_t u, uint32_t ov, int64_t v) {
    return ou < ov || (ou == ov && u < v);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Volatile 64-bit load / store used by the decoupled look-back scans.
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Decoupled look-back (single value) executed by one full warp: returns the exclusive
// prefix of tile `tile` and publishes its inclusive prefix. `status` has one word per
// tile, zero-initialised before the launch.  Tiles must be numbered in launch order
// (dynamic tile ids) so predecessors always make progress.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* status, long long tile,
                                                            unsigned long long agg, int lane) {
    if (tile == 0) {
        if (lane == 0) st_volatile(&status[0], kFlagPre | agg);
        return 0ull;
    }
    if (lane == 0) st_volatile(&status[tile], kFlagAgg | agg);
    unsigned long long excl = 0;
    long long j = tile - 1;
    while (true) {
        long long t = j - lane;
        unsigned long long w = (t >= 0) ? ld_volatile(&status[t]) : (kFlagPre | 0ull);
        while (__any_sync(0xffffffffu, (w >> 62) == 0ull)) {
            if ((w >> 62) == 0ull) w = ld_volatile(&status[t]);
        }
        unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2ull);
        int first = pre ? (__ffs(pre) - 1) : 32;
        unsigned long long val = (lane <= first) ? (w & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (pre) break;
        j -= 32;
    }
    if (lane == 0) st_volatile(&status[tile], kFlagPre | (excl + agg));
    return excl;
}

// Block-wide exclusive sum of one uint32 per thread (kBlock threads). Returns the
// exclusive prefix; *total receives the block sum.
template <int NW>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t* smem_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) smem_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NW ? smem_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < NW) smem_warp[lane] = wi - w;
        if (lane == NW - 1) smem_warp[NW] = wi;
    }
    __syncthreads();
    uint32_t r = smem_warp[warp] + inc - x;
    *total = smem_warp[NW];
    __syncthreads();
    return r;
}

}  // namespace dms
