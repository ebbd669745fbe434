// onesweep.cuh -- the global vertex order as an LSD radix sort in "one sweep" form
// (sm_100a): one pass reads f and builds the digit histograms of all four passes, then
// every digit pass ranks its tile, finds its global digit offsets by a decoupled
// look-back over the preceding tiles and scatters -- no per-pass histogram read and no
// per-pass scan.  rank(v) = #{u : K(u) < K(v)}, K(v) = (f(v), v) (PAPER.md 1368-1372,
// readings Z2/Z3): the keys are the order-preserving uint32 images of f, the values the
// vertex ids; stable passes over an index-ordered input break ties by index.
//
// The last pass knows every element's sorted position p and writes rank[v] = p:
//   small N: directly;
//   large N: (v, p) pairs into the bucket of v's window (2^kWinBits vertices; window w's
//            bucket is wbuf[w << kWinBits ..], filled through one global cursor per
//            window, one atomic per (tile, window)), then k_os_rank writes each window's
//            ranks -- the stores of a window stay within 8 MB, so L2 merges their sectors
//            instead of a DRAM read-modify-write per 4-byte store.
// Traffic ~ 4 (histograms) + 12 + 16 + 16 + 16 (passes) + 12 (ranks) = 76 B/vertex.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace dms {

#ifndef DMS_OS_ITEMS
#define DMS_OS_ITEMS 15
#endif
#ifndef DMS_OS_MINB
#define DMS_OS_MINB 3
#endif
constexpr int kOsT = 256;
constexpr int kOsItems = DMS_OS_ITEMS;
constexpr int kOsTile = kOsT * kOsItems;  // keys per tile
constexpr int kOsWarps = kOsT / 32;
constexpr int kOsWinMax = 1024;           // windows of 2^kWinBits vertices (N < 2^31)

// status word of (tile, digit): epoch << 48 | flag << 32 | value; flag 1 = tile
// aggregate, 2 = inclusive prefix; another epoch = not written yet (no reset per pass)
__device__ __forceinline__ unsigned long long os_word(uint32_t epoch, uint32_t flag, uint32_t v) {
    return ((unsigned long long)epoch << 48) | ((unsigned long long)flag << 32) | v;
}

// the digit histograms of all four passes in one read of f, with the NaN flag and the
// K-highest vertex (f*, Sec. 6) fused
__global__ void __launch_bounds__(kOsT) k_os_hist(const float* __restrict__ f, int64_t n, uint32_t* __restrict__ hist,
                                                  int* err, unsigned long long* kmax) {
    __shared__ uint32_t h[4 * 256];
    for (int i = threadIdx.x; i < 4 * 256; i += kOsT) h[i] = 0;
    __syncthreads();
    unsigned long long m = 0;
    bool nan = false;
    const int64_t stride = (int64_t)gridDim.x * kOsT;
    for (int64_t i = (int64_t)blockIdx.x * kOsT + threadIdx.x; i < n; i += stride) {
        const float x = __ldg(f + i);
        nan |= is_nan_bits(x);
        const uint32_t o = ord_of(x);
        const unsigned long long km = ((unsigned long long)o << 32) | (unsigned long long)i;
        m = km > m ? km : m;
        atomicAdd(&h[o & 255u], 1u);
        atomicAdd(&h[256 + ((o >> 8) & 255u)], 1u);
        atomicAdd(&h[512 + ((o >> 16) & 255u)], 1u);
        atomicAdd(&h[768 + (o >> 24)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += kOsT)
        if (h[i]) atomicAdd(hist + i, h[i]);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
        m = y > m ? y : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(kmax, m);
    if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// exclusive scans of the four 256-bin histograms (one block per pass) and the window
// cursors (window w starts at w << kWinBits)
__global__ void k_os_scan(uint32_t* hist, uint32_t* wcur, int nwin) {
    __shared__ uint32_t sw[kOsWarps + 1];
    const int p = blockIdx.x;
    const uint32_t x = hist[p * 256 + threadIdx.x];
    uint32_t tot;
    const uint32_t e = block_excl_sum<kOsWarps>(x, sw, &tot);
    hist[p * 256 + threadIdx.x] = e;
    if (p == 0 && wcur)
        for (int w = threadIdx.x; w < nwin; w += kOsT) wcur[w] = (uint32_t)w << kWinBits;
}

// One digit pass.  MODE 0: write the (key, value) arrays; 1: last pass, rank[v] = p;
// 2: last pass, (v, p) into v's window bucket.  FIRST: keys / values from f.
// (Measured variants: publishing the tile counts before the ranking,
// ballot-built peer masks, one combined staging offset / 8-byte staging stores -- none
// faster.)
// LB: look-back words in flight per thread (4 on the full grid: c5b order 6.09 -> 5.70 ms,
// c5a 4.52 -> 4.40; 1 on the small grid beside the 3D gradient, where 4 cost c4 0.3 ms).
template <bool FIRST, int MODE, int LB>
__global__ void __launch_bounds__(kOsT, DMS_OS_MINB) k_os_pass(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                     const float* __restrict__ f, uint32_t* __restrict__ kout,
                                                     uint32_t* __restrict__ vout, int32_t* __restrict__ rank_out,
                                                     uint2* __restrict__ wbuf, uint32_t* __restrict__ wcur, int64_t n,
                                                     int shift, const uint32_t* __restrict__ dbase,
                                                     unsigned long long* status, uint32_t epoch, int* tile_ctr,
                                                     int64_t ntiles) {
    __shared__ uint32_t wcnt[kOsWarps][256];
    __shared__ uint32_t tstart[256];
    __shared__ uint32_t gofs[256];
    __shared__ uint32_t sw[kOsWarps + 1];
    __shared__ uint32_t sk[kOsTile];
    __shared__ uint32_t sv[kOsTile];
    // MODE 2: the per-window counts / bases alias wcnt (free once the tile is staged)
    uint32_t* winc = &wcnt[0][0];
    uint32_t* winb = &wcnt[kOsWarps / 2][0];
    static_assert(kOsWarps * 256 >= 2 * kOsWinMax, "window counters alias the warp counters");
    __shared__ int s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1);  // launch-order tiles: look-back progresses
#pragma unroll
        for (int w = 0; w < kOsWarps; w++) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) return;
        const int64_t tile0 = tile * kOsTile;
        const int64_t seg = tile0 + (int64_t)warp * (32 * kOsItems);
        uint32_t k[kOsItems], v[kOsItems], dg[kOsItems];
#pragma unroll
        for (int i = 0; i < kOsItems; i++) {
            const int64_t idx = seg + i * 32 + lane;
            if (idx < n) {
                if (FIRST) {
                    k[i] = ord_of(__ldg(f + idx));
                    v[i] = (uint32_t)idx;
                } else {
                    k[i] = __ldg(kin + idx);
                    v[i] = __ldg(vin + idx);
                }
                dg[i] = (k[i] >> shift) & 255u;
            } else {
                k[i] = 0;
                v[i] = 0;
                dg[i] = 256u;  // sentinel: never counted, never written
            }
        }
        // warp ranking: all matches first (independent, they pipeline), then the
        // per-warp digit counters, updated by the highest peer lane
        uint32_t pm[kOsItems];
#pragma unroll
        for (int i = 0; i < kOsItems; i++) pm[i] = __match_any_sync(0xffffffffu, dg[i]);
        uint32_t pos[kOsItems];
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int i = 0; i < kOsItems; i++) {
            const uint32_t d = dg[i];
            const int leader = 31 - __clz(pm[i]);
            uint32_t b = 0;
            if (lane == leader && d < 256u) {
                b = wcnt[warp][d];
                wcnt[warp][d] = b + __popc(pm[i]);
            }
            b = __shfl_sync(0xffffffffu, b, leader);
            pos[i] = b + __popc(pm[i] & lt);
            __syncwarp();
        }
        __syncthreads();
        // thread d: the warps' offsets for digit d, the tile's count, its global offset
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kOsWarps; w++) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = run;
            run += c;
        }
        unsigned long long* st = status + (size_t)tile * 256 + d;
        uint32_t excl = 0;
        if (tile == 0) {
            st_volatile(st, os_word(epoch, 2u, run));
        } else {
            st_volatile(st, os_word(epoch, 1u, run));
            // look back LB tiles at a time (independent loads in flight, consumed in order; a
            // word of another epoch is not written yet: resume from that tile)
            int64_t t = tile - 1;
            bool done = false;
            while (!done) {
                unsigned long long w[LB];
#pragma unroll
                for (int j = 0; j < LB; j++)
                    w[j] = t - j >= 0 ? ld_volatile(status + (size_t)(t - j) * 256 + d) : os_word(epoch, 2u, 0u);
                int used = 0;
#pragma unroll
                for (int j = 0; j < LB; j++) {
                    if (done || used != j) continue;
                    if ((uint32_t)(w[j] >> 48) != epoch) continue;  // not written yet
                    excl += (uint32_t)w[j];
                    used = j + 1;
                    done = ((w[j] >> 32) & 3ull) == 2ull;
                }
                t -= used;
            }
            st_volatile(st, os_word(epoch, 2u, excl + run));
        }
        gofs[d] = dbase[d] + excl;
        uint32_t tot;
        tstart[d] = block_excl_sum<kOsWarps>(run, sw, &tot);
        __syncthreads();
        // stage the tile sorted by digit (stable), then write runs per digit
#pragma unroll
        for (int i = 0; i < kOsItems; i++) {
            const uint32_t dd = dg[i];
            if (dd < 256u) {
                const uint32_t lp = tstart[dd] + wcnt[warp][dd] + pos[i];
                sk[lp] = k[i];
                sv[lp] = v[i];
            }
        }
        __syncthreads();
        const int tn = (int)((n - tile0) < (int64_t)kOsTile ? (n - tile0) : (int64_t)kOsTile);
        if (MODE == 2) {
            // per-window counts of the tile, one global cursor atomic per touched window
            for (int w = threadIdx.x; w < kOsWinMax; w += kOsT) winc[w] = 0;
            __syncthreads();
            uint32_t wl[kOsItems];
#pragma unroll
            for (int i = 0; i < kOsItems; i++) {
                const int j = threadIdx.x + i * kOsT;
                if (j < tn) wl[i] = atomicAdd(&winc[sv[j] >> kWinBits], 1u);
            }
            __syncthreads();
            for (int w = threadIdx.x; w < kOsWinMax; w += kOsT)
                if (winc[w]) winb[w] = atomicAdd(wcur + w, winc[w]);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kOsItems; i++) {
                const int j = threadIdx.x + i * kOsT;
                if (j < tn) {
                    const uint32_t kk = sk[j];
                    const uint32_t dd = (kk >> shift) & 255u;
                    const uint32_t p = gofs[dd] + (uint32_t)j - tstart[dd];
                    const uint32_t vv = sv[j];
                    wbuf[winb[vv >> kWinBits] + wl[i]] = make_uint2(vv, p);
                }
            }
        } else {
            for (int j = threadIdx.x; j < tn; j += kOsT) {
                const uint32_t kk = sk[j];
                const uint32_t dd = (kk >> shift) & 255u;
                const uint32_t p = gofs[dd] + (uint32_t)j - tstart[dd];
                if (MODE == 1) {
                    rank_out[sv[j]] = (int32_t)p;
                } else {
                    kout[p] = kk;
                    vout[p] = sv[j];
                }
            }
        }
        __syncthreads();
    }
}

__global__ void k_os_rank(const uint2* __restrict__ wbuf, int64_t n, int32_t* __restrict__ rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const uint2 e = wbuf[i];
        rank[e.x] = (int32_t)e.y;
    }
}

}  // namespace dms
