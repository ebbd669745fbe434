// sort.cuh -- hand-written stable LSD radix sort (8-bit digits) for sm_100a.
//
// Used for the global vertex order (a key-value sort of (value, index), PAPER.md
// 1069-1071 / 1121 "parallel sort") and for sorting the critical simplices by their
// lexicographic keys (Alg. 2 l. 13, PAPER.md 357-359).
//
// Per pass: k_hist (per-tile digit histogram, digit-major counts), k_scan_excl
// (single-pass decoupled look-back scan of the counts), k_scatter (stable in-tile
// ranking with warp match + per-warp digit counters, then scatter).  The last pass of
// the vertex order writes rank[value] = position directly.
#pragma once
#include "common.cuh"

namespace dms {

constexpr int kRadix = 256;

template <typename Key>
__device__ __forceinline__ uint32_t digit_of(Key k, int shift) {
    return (uint32_t)((k >> shift) & (Key)0xff);
}

template <typename Key, int ITEMS, bool FROM_F>
__global__ void __launch_bounds__(kBlock) k_hist(const Key* __restrict__ keys, const float* __restrict__ fin,
                                                 int64_t n, int shift, uint32_t* __restrict__ counts, int64_t ntiles,
                                                 int* err, unsigned long long* kmax) {
    __shared__ uint32_t h[kRadix];
    unsigned long long m = 0;
    bool nan = false;
    // tile-strided (a small persistent grid leaves room beside the gradient kernel)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = tile * (kBlock * ITEMS);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        int64_t idx = base + (int64_t)i * kBlock + threadIdx.x;
        if (idx < n) {
            Key kk;
            if (FROM_F) {
                const float x = fin[idx];
                nan |= is_nan_bits(x);
                const uint32_t o = ord_of(x);
                kk = (Key)o;
                const unsigned long long km = ((unsigned long long)o << 32) | (unsigned long long)idx;
                m = km > m ? km : m;
            } else {
                kk = keys[idx];
            }
            atomicAdd(&h[digit_of(kk, shift)], 1u);
        }
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + tile] = h[threadIdx.x];
    __syncthreads();
    }
    if (FROM_F) {  // fused: NaN detection and the highest vertex (f*) for Sec. 6
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
            m = y > m ? y : m;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(kmax, m);
        if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
    }
}

// Exclusive scan of n uint32 (single pass, decoupled look-back). status[ntiles] and
// *tile_ctr must be zero before the launch.
constexpr int kScanItems = 16;
__global__ void __launch_bounds__(kBlock) k_scan_excl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                      int64_t n, unsigned long long* status, int* tile_ctr) {
    __shared__ uint32_t sw[kBlock / 32 + 1];
    __shared__ long long s_tile;
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1);
    __syncthreads();
    const long long tile = s_tile;
    const int64_t base = tile * (kBlock * kScanItems) + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        v[j] = (base + j < n) ? in[base + j] : 0u;
        sum += v[j];
    }
    uint32_t total;
    uint32_t excl = block_excl_sum<kBlock / 32>(sum, sw, &total);
    if (threadIdx.x < 32) {
        unsigned long long e = lookback_warp(status, tile, total, threadIdx.x);
        if (threadIdx.x == 0) s_excl = e;
    }
    __syncthreads();
    uint32_t run = (uint32_t)s_excl + excl;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
}

// Stable scatter of one LSD pass.
//   FROM_F:   the keys are ord_of(f[i]) and the values the indices i (first pass of the
//             vertex order: no separate key-extraction pass).
//   RANK_OUT: write rank_out[val] = position instead of (key, val) (last pass).
// The tile is ranked in shared memory (warp match + per-warp digit counters, stable),
// staged digit-sorted in shared memory, and written out as per-digit runs so that
// consecutive threads store to consecutive global addresses.
template <typename Key, typename Val, int ITEMS, bool RANK_OUT, bool FROM_F>
#ifndef DMS_SCATTER_MINB
#define DMS_SCATTER_MINB 4  // 4 CTAs x 8 warps per SM (measured: order c4 9.6 -> 9.4 ms, c5b 6.0 -> 5.4)
#endif
__global__ void __launch_bounds__(kBlock, DMS_SCATTER_MINB) k_scatter(const Key* __restrict__ kin, const Val* __restrict__ vin,
                                                    const float* __restrict__ fin, Key* __restrict__ kout,
                                                    Val* __restrict__ vout, int32_t* __restrict__ rank_out, int64_t n,
                                                    int shift, const uint32_t* __restrict__ counts_scanned,
                                                    int64_t ntiles) {
    constexpr int NW = kBlock / 32;
    constexpr int TILE = kBlock * ITEMS;
    __shared__ uint32_t wcnt[NW][kRadix];
    __shared__ uint32_t gbase[kRadix];
    __shared__ uint32_t tstart[kRadix];
    __shared__ uint32_t sw[NW + 1];
    extern __shared__ __align__(16) unsigned char dyn[];
    Key* sk = reinterpret_cast<Key*>(dyn);
    Val* sv = reinterpret_cast<Val*>(dyn + sizeof(Key) * TILE);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // tile-strided (see k_hist)
#pragma unroll
    for (int w = 0; w < NW; w++) wcnt[w][threadIdx.x] = 0;
    gbase[threadIdx.x] = counts_scanned[(int64_t)threadIdx.x * ntiles + tile];
    __syncthreads();
    const int64_t tile0 = tile * TILE;
    const int64_t seg = tile0 + (int64_t)warp * (32 * ITEMS);
    Key k[ITEMS];
    Val v[ITEMS];
    uint32_t pos[ITEMS];
    uint32_t dg[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int64_t idx = seg + i * 32 + lane;
        if (idx < n) {
            if (FROM_F) {
                k[i] = (Key)ord_of(fin[idx]);
                v[i] = (Val)idx;
            } else {
                k[i] = kin[idx];
                v[i] = vin[idx];
            }
            dg[i] = digit_of(k[i], shift);
        } else {
            dg[i] = kRadix;  // sentinel, never written
        }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const uint32_t d = dg[i];
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t r = __popc(peers & lanemask_lt());
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (d < kRadix) b = wcnt[warp][d];
        __syncwarp();
        if (d < kRadix && lane == leader) wcnt[warp][d] = b + __popc(peers);
        __syncwarp();
        pos[i] = b + r;
    }
    __syncthreads();
    uint32_t dtot;
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) {
            const uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = run;
            run += c;
        }
        dtot = run;
    }
    uint32_t tot;
    const uint32_t ts = block_excl_sum<NW>(dtot, sw, &tot);  // start of digit threadIdx.x in the tile
    tstart[threadIdx.x] = ts;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const uint32_t d = dg[i];
        if (d < kRadix) {
            const uint32_t lp = tstart[d] + wcnt[warp][d] + pos[i];
            sk[lp] = k[i];
            sv[lp] = v[i];
        }
    }
    __syncthreads();
    const int tn = (int)((n - tile0) < (int64_t)TILE ? (n - tile0) : (int64_t)TILE);
    for (int j = threadIdx.x; j < tn; j += kBlock) {
        const Key kk = sk[j];
        const uint32_t d = digit_of(kk, shift);
        const uint32_t p = gbase[d] + (uint32_t)j - tstart[d];
        if (RANK_OUT) {
            rank_out[sv[j]] = (int32_t)p;
        } else {
            if (kout) kout[p] = kk;  // (null: the last pass of the windowed rank inversion)
            vout[p] = sv[j];
        }
    }
    __syncthreads();
    }
}

// ---- windowed rank inversion (the vertex order's last step).  rank[v] = p for the
// sorted vertices ord[p] is a random permutation: 4-byte stores straight into the
// 537 MB rank array (c4) cost a DRAM read-modify-write of a 32-byte sector each (ncu:
// 4.1 GB written + 4.2 GB read for 0.54 GB of ranks).  Instead the (v, p) pairs are
// bucketed by the window v >> kWinBits (2^21 vertices = 8 MB of ranks) with coalesced
// runs, then stored window by window, so the sectors a window touches stay in L2 until
// they are complete.
constexpr int kWinBits = 21;
constexpr int kWinItems = 16;
constexpr int kWinTile = kBlock * kWinItems;
constexpr int kWinMax = 1024;  // windows (N < 2^31)

__global__ void __launch_bounds__(kBlock) k_win_hist(const uint32_t* __restrict__ ord, int64_t n, int nwin,
                                                     uint32_t* __restrict__ counts, int64_t ntiles) {
    __shared__ uint32_t h[kWinMax];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int i = threadIdx.x; i < nwin; i += kBlock) h[i] = 0;
        __syncthreads();
        const int64_t base = tile * kWinTile;
#pragma unroll
        for (int i = 0; i < kWinItems; i++) {
            const int64_t idx = base + (int64_t)i * kBlock + threadIdx.x;
            if (idx < n) atomicAdd(&h[ord[idx] >> kWinBits], 1u);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nwin; i += kBlock) counts[(int64_t)i * ntiles + tile] = h[i];
        __syncthreads();
    }
}

// pairs (v, p) of a tile to their windows: staged window by window in shared memory (the
// order inside a window is irrelevant), written as runs
__global__ void __launch_bounds__(kBlock) k_win_scatter(const uint32_t* __restrict__ ord, int64_t n, int nwin,
                                                        const uint32_t* __restrict__ scanned, int64_t ntiles,
                                                        uint32_t* __restrict__ pv, uint32_t* __restrict__ pp) {
    __shared__ uint32_t cur[kWinMax], start[kWinMax], gb[kWinMax];
    __shared__ uint32_t sv[kWinTile], sp[kWinTile];
    __shared__ uint32_t sw[kBlock / 32 + 1];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int i = threadIdx.x; i < nwin; i += kBlock) {
            cur[i] = 0;
            gb[i] = scanned[(int64_t)i * ntiles + tile];
        }
        __syncthreads();
        const int64_t base = tile * kWinTile;
        uint32_t v[kWinItems], lp[kWinItems];
#pragma unroll
        for (int i = 0; i < kWinItems; i++) {
            const int64_t idx = base + (int64_t)i * kBlock + threadIdx.x;
            v[i] = idx < n ? ord[idx] : 0xffffffffu;
            lp[i] = idx < n ? atomicAdd(&cur[v[i] >> kWinBits], 1u) : 0u;
        }
        __syncthreads();
        // tile-local window starts: exclusive scan of cur (nwin <= kWinMax = 4 x kBlock)
        uint32_t c4[kWinMax / kBlock], sum = 0;
#pragma unroll
        for (int j = 0; j < kWinMax / kBlock; j++) {
            const int w = threadIdx.x * (kWinMax / kBlock) + j;
            c4[j] = w < nwin ? cur[w] : 0u;
            sum += c4[j];
        }
        uint32_t tot;
        uint32_t run = block_excl_sum<kBlock / 32>(sum, sw, &tot);
#pragma unroll
        for (int j = 0; j < kWinMax / kBlock; j++) {
            const int w = threadIdx.x * (kWinMax / kBlock) + j;
            if (w < nwin) start[w] = run;
            run += c4[j];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kWinItems; i++) {
            const int64_t idx = base + (int64_t)i * kBlock + threadIdx.x;
            if (idx < n) {
                const uint32_t at = start[v[i] >> kWinBits] + lp[i];
                sv[at] = v[i];
                sp[at] = (uint32_t)idx;  // the rank
            }
        }
        __syncthreads();
        const int tn = (int)((n - base) < (int64_t)kWinTile ? (n - base) : (int64_t)kWinTile);
        for (int j = threadIdx.x; j < tn; j += kBlock) {
            const uint32_t w = sv[j] >> kWinBits;
            const uint32_t p = gb[w] + (uint32_t)j - start[w];
            pv[p] = sv[j];
            pp[p] = sp[j];
        }
        __syncthreads();
    }
}

__global__ void k_win_rank(const uint32_t* __restrict__ pv, const uint32_t* __restrict__ pp, int64_t n,
                           int32_t* __restrict__ rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rank[pv[i]] = (int32_t)pp[i];
}

struct SortScratch {
    uint32_t* counts = nullptr;       // kRadix * max tiles
    uint32_t* counts_scan = nullptr;  // same
    unsigned long long* status = nullptr;
    int* tile_ctr = nullptr;
    int64_t max_tiles = 0;
    int64_t max_scan_tiles = 0;
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaError_t scan_excl(const uint32_t* in, uint32_t* out, int64_t n, SortScratch& s, cudaStream_t st,
                             int64_t* launches) {
    int64_t tiles = ceil_div(n, (int64_t)kBlock * kScanItems);
    cudaMemsetAsync(s.status, 0, tiles * sizeof(unsigned long long), st);
    cudaMemsetAsync(s.tile_ctr, 0, sizeof(int), st);
    k_scan_excl<<<(unsigned)tiles, kBlock, 0, st>>>(in, out, n, s.status, s.tile_ctr);
    *launches += 1;
    return cudaGetLastError();
}

// Sort (keys, vals) by bits [bit0, bit1) of the key.  Buffers a -> b -> a ...; returns
// 0 if the result is in (ka, va), 1 if in (kb, vb).  With rank_out != nullptr the last
// pass writes rank_out[val] = position and the return value is meaningless.  With
// f != nullptr the first pass reads the keys as ord_of(f[i]) and the values as i.
template <typename Key, typename Val, int ITEMS>
inline int radix_sort(Key* ka, Val* va, Key* kb, Val* vb, int64_t n, int bit0, int bit1, SortScratch& s,
                      cudaStream_t st, int64_t* launches, int32_t* rank_out = nullptr, const float* f = nullptr,
                      int* err = nullptr, unsigned long long* kmax = nullptr, int64_t grid_cap = 0) {
    if (n <= 0) return 0;
    constexpr int TILE = kBlock * ITEMS;
    constexpr size_t smem = (sizeof(Key) + sizeof(Val)) * TILE;
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_scatter<Key, Val, ITEMS, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_scatter<Key, Val, ITEMS, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_scatter<Key, Val, ITEMS, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_scatter<Key, Val, ITEMS, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_done = true;
    }
    const int64_t tiles = ceil_div(n, (int64_t)TILE);
    // grid_cap > 0: a small tile-strided grid (leaves SM room for a concurrent kernel)
    const unsigned grid = (unsigned)(grid_cap > 0 ? std::min<int64_t>(tiles, grid_cap) : tiles);
    int cur = 0;
    // windowed rank inversion for large orders (see k_win_scatter); DMS_RANK_WIN overrides
    // the size threshold (0: always direct stores)
    static const long long win_env = getenv("DMS_RANK_WIN") ? atoll(getenv("DMS_RANK_WIN")) : -1;
    bool windowed = false;
    if constexpr (sizeof(Key) == 4 && sizeof(Val) == 4)
        windowed = rank_out && (win_env < 0 ? n >= (int64_t(1) << 23) : (win_env > 0 && n >= win_env));
    for (int shift = bit0; shift < bit1; shift += 8) {
        const bool first = shift == bit0 && f != nullptr;
        const bool last = shift + 8 >= bit1;
        Key* ki = cur ? kb : ka;
        Val* vi = cur ? vb : va;
        Key* ko = cur ? ka : kb;
        Val* vo = cur ? va : vb;
        if (first) k_hist<Key, ITEMS, true><<<grid, kBlock, 0, st>>>(ki, f, n, shift, s.counts, tiles, err, kmax);
        else k_hist<Key, ITEMS, false><<<grid, kBlock, 0, st>>>(ki, f, n, shift, s.counts, tiles, err, kmax);
        *launches += 1;
        scan_excl(s.counts, s.counts_scan, tiles * kRadix, s, st, launches);
        const bool ro = last && rank_out && !windowed;
        Key* kout = (last && windowed) ? nullptr : ko;  // windowed: the sorted vertex ids only
#define DMS_SCATTER(RO, FF)                                                                               \
    k_scatter<Key, Val, ITEMS, RO, FF><<<grid, kBlock, smem, st>>>(ki, vi, f, kout, vo, rank_out, n, shift, \
                                                                          s.counts_scan, tiles)
        if (ro && first) DMS_SCATTER(true, true);
        else if (ro) DMS_SCATTER(true, false);
        else if (first) DMS_SCATTER(false, true);
        else DMS_SCATTER(false, false);
#undef DMS_SCATTER
        *launches += 1;
        if (last && windowed) {
            if constexpr (sizeof(Key) == 4 && sizeof(Val) == 4) {
                const uint32_t* ord = reinterpret_cast<const uint32_t*>(vo);
                uint32_t* pv = reinterpret_cast<uint32_t*>(ki);  // free now: the last pass's input
                uint32_t* pp = reinterpret_cast<uint32_t*>(vi);
                const int nwin = (int)((n + (int64_t(1) << kWinBits) - 1) >> kWinBits);
                const int64_t wt = ceil_div(n, (int64_t)kWinTile);
                const unsigned wg = (unsigned)(grid_cap > 0 ? std::min<int64_t>(wt, grid_cap) : wt);
                k_win_hist<<<wg, kBlock, 0, st>>>(ord, n, nwin, s.counts, wt);
                scan_excl(s.counts, s.counts_scan, wt * nwin, s, st, launches);
                k_win_scatter<<<wg, kBlock, 0, st>>>(ord, n, nwin, s.counts_scan, wt, pv, pp);
                k_win_rank<<<(unsigned)ceil_div(n, (int64_t)kBlock), kBlock, 0, st>>>(pv, pp, n, rank_out);
                *launches += 3;
            }
        }
        cur ^= 1;
    }
    return cur;
}

}  // namespace dms
