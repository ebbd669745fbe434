// order.cuh -- the global vertex order by sample sort (sm_100a).
//
// rank(v) = #{u : K(u) < K(v)}, K(v) = (f(v), v) with the index tie-break (PAPER.md
// 1368-1372, reading Z2/Z3), as the unique 64-bit key ord(f(v)) << 32 | v.  The paper
// uses a parallel sort (PAPER.md 1069-1071, 1121); this is a sample sort shaped for
// HBM (SURVEY 8(a) "Rank kernels"), replacing four LSD radix passes (~70 B/vertex) by:
//   k_ord_sample + radix sort of 64 keys per bucket + k_ord_splitters
//                    B - 1 splitters (unique 64-bit keys, so ties cannot unbalance them)
//   k_ord_count      read f once: bucket of every key by binary search over the splitters
//                    in shared memory, per-CTA bucket histograms, the 2-byte bucket id,
//                    fused NaN detection and f* (the K-highest vertex, Sec. 6)
//   scan             (bucket, CTA) offsets
//   k_ord_scatter    read f again, write the 8-byte keys bucket by bucket
//   k_ord_bucket     one CTA per bucket: the keys in registers, LSD passes through shared
//                    memory over the bytes that vary inside the bucket, rank[v] written
// ~4 + 2 + 4 + 2 + 8 + 8 + 4 = 32 B/vertex of DRAM traffic plus the scattered rank
// writes.  A bucket larger than the shared-memory capacity (vanishingly unlikely with 64
// samples per bucket: DESIGN.md) is sorted in place in global memory by its CTA.
#pragma once
#include "common.cuh"
#include "sort.cuh"

namespace dms {

constexpr int kOrdT = 1024;                   // threads per CTA
constexpr int kOrdItems = 16;                 // keys per thread in k_ord_bucket
constexpr int kOrdCap = kOrdT * kOrdItems;    // 16384 keys: largest bucket sorted in shared memory
constexpr int kOrdMaxB = 16384;               // buckets (64-bit splitters in shared memory: 128 KB)
constexpr int kOrdOversample = 64;            // samples per bucket
constexpr int kOrdMeanMax = 8192;             // the sample sort is used while N / B <= this
constexpr int kOrdWcStride = 33;              // [digit][warp] counters, padded (conflict free)
constexpr int kOrdBucketSmem = kOrdCap * 8 + 256 * kOrdWcStride * 4;  // dynamic shared memory of k_ord_bucket

__device__ __forceinline__ uint32_t ord_hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// one sample key per stratum [i N / S, (i+1) N / S), at a hashed position inside it
__global__ void k_ord_sample(const float* __restrict__ f, int64_t N, int S, uint64_t* __restrict__ skeys,
                             uint32_t* __restrict__ svals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int64_t lo = (int64_t)i * N / S, hi = (int64_t)(i + 1) * N / S;
    const int64_t v = lo + (hi > lo ? (int64_t)(ord_hash32((uint32_t)i) % (uint32_t)(hi - lo)) : 0);
    skeys[i] = ((uint64_t)ord_of(f[v]) << 32) | (uint64_t)v;
    svals[i] = (uint32_t)i;
}

// splitter j = the ((j+1) S/B - 1)-th smallest sample; the last slot is +inf (never
// compared, see ord_bucket)
__global__ void k_ord_splitters(const uint64_t* __restrict__ sorted, int S, int B, uint64_t* __restrict__ spl) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= B) return;
    spl[j] = j < B - 1 ? sorted[(int64_t)(j + 1) * (S / B) - 1] : ~0ull;
}

// bucket of k = #{j < B-1 : spl[j] < k} (B a power of two; branch-free binary search)
__device__ __forceinline__ int ord_bucket(const uint64_t* sp, int B, uint64_t k) {
    int b = 0;
    for (int step = B >> 1; step > 0; step >>= 1) b += (sp[b + step - 1] < k) ? step : 0;
    return b;
}

__device__ __forceinline__ void ord_range(int64_t N, int64_t* v0, int64_t* v1) {
    *v0 = (int64_t)blockIdx.x * N / gridDim.x;
    *v1 = (int64_t)(blockIdx.x + 1) * N / gridDim.x;
}

__global__ void __launch_bounds__(kOrdT, 1) k_ord_count(const float* __restrict__ f, int64_t N, int B,
                                                        const uint64_t* __restrict__ spl, uint16_t* __restrict__ bid,
                                                        uint32_t* __restrict__ counts, int* err,
                                                        unsigned long long* kmax) {
    extern __shared__ __align__(16) unsigned char dyn[];
    uint64_t* sp = reinterpret_cast<uint64_t*>(dyn);
    uint32_t* hist = reinterpret_cast<uint32_t*>(dyn + (size_t)B * 8);
    for (int i = threadIdx.x; i < B; i += kOrdT) {
        sp[i] = spl[i];
        hist[i] = 0;
    }
    __syncthreads();
    int64_t v0, v1;
    ord_range(N, &v0, &v1);
    unsigned long long m = 0;
    bool nan = false;
    int64_t v = v0 + threadIdx.x;
    for (; v + kOrdT < v1; v += 2 * kOrdT) {  // two keys per iteration (independent searches)
        const float x0 = f[v], x1 = f[v + kOrdT];
        nan |= is_nan_bits(x0) | is_nan_bits(x1);
        const uint64_t k0 = ((uint64_t)ord_of(x0) << 32) | (uint64_t)v;
        const uint64_t k1 = ((uint64_t)ord_of(x1) << 32) | (uint64_t)(v + kOrdT);
        m = k1 > m ? k1 : m;  // (k1 > k0: same value order, larger index, or a larger value)
        m = k0 > m ? k0 : m;
        const int b0 = ord_bucket(sp, B, k0), b1 = ord_bucket(sp, B, k1);
        bid[v] = (uint16_t)b0;
        bid[v + kOrdT] = (uint16_t)b1;
        atomicAdd(&hist[b0], 1u);
        atomicAdd(&hist[b1], 1u);
    }
    if (v < v1) {
        const float x = f[v];
        nan |= is_nan_bits(x);
        const uint64_t k = ((uint64_t)ord_of(x) << 32) | (uint64_t)v;
        m = k > m ? k : m;
        const int b = ord_bucket(sp, B, k);
        bid[v] = (uint16_t)b;
        atomicAdd(&hist[b], 1u);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
        m = y > m ? y : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(kmax, m);
    if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += kOrdT) counts[(int64_t)i * gridDim.x + blockIdx.x] = hist[i];
}

// keys of the CTA's range to their buckets: position = the (bucket, CTA) offset + a
// shared-memory cursor (the order inside a bucket is irrelevant: k_ord_bucket sorts by
// the whole unique key)
__global__ void __launch_bounds__(kOrdT, 1) k_ord_scatter(const float* __restrict__ f, int64_t N, int B,
                                                          const uint16_t* __restrict__ bid,
                                                          const uint32_t* __restrict__ offs,
                                                          uint64_t* __restrict__ keys) {
    extern __shared__ __align__(16) unsigned char dyn[];
    uint32_t* cur = reinterpret_cast<uint32_t*>(dyn);
    for (int i = threadIdx.x; i < B; i += kOrdT) cur[i] = offs[(int64_t)i * gridDim.x + blockIdx.x];
    __syncthreads();
    int64_t v0, v1;
    ord_range(N, &v0, &v1);
    for (int64_t v = v0 + threadIdx.x; v < v1; v += kOrdT) {
        const uint64_t k = ((uint64_t)ord_of(f[v]) << 32) | (uint64_t)v;
        const uint32_t p = atomicAdd(&cur[bid[v]], 1u);
        keys[p] = k;
    }
}

// in-place sort of keys[0, m) in global memory by one CTA (bitonic network in the
// all-ascending form, positions >= m acting as +inf): the fallback for a bucket larger
// than kOrdCap
__device__ void ord_bitonic_global(uint64_t* keys, int m) {
    int p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k; j >= 2; j >>= 1) {
            const bool flip = j == k;
            const int h = j >> 1;
            for (int i = threadIdx.x; i < (p2 >> 1); i += blockDim.x) {
                const int blk = i / h, off = i % h;
                const int a = blk * j + off;
                const int b = flip ? blk * j + j - 1 - off : a + h;
                if (b < m) {
                    const uint64_t x = keys[a], y = keys[b];
                    if (y < x) {
                        keys[a] = y;
                        keys[b] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// one CTA per bucket: rank[v] = bucket start + position of v's key inside the bucket
__global__ void __launch_bounds__(kOrdT, 1) k_ord_bucket(uint64_t* __restrict__ keys, int64_t N, int B,
                                                         int G, const uint32_t* __restrict__ offs,
                                                         int32_t* __restrict__ rank, int cap) {
    extern __shared__ __align__(16) unsigned char dyn[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(dyn);                             // kOrdCap keys
    uint32_t* wc = reinterpret_cast<uint32_t*>(dyn + (size_t)kOrdCap * 8);        // [256][33]
    __shared__ uint32_t dtot[256];
    __shared__ unsigned long long s_or[32], s_and[32];
    const int b = blockIdx.x;
    const int64_t s0 = offs[(int64_t)b * G];
    const int64_t s1 = b + 1 < B ? (int64_t)offs[(int64_t)(b + 1) * G] : N;
    const int m = (int)(s1 - s0);
    if (m <= 0) return;
    uint64_t* bk = keys + s0;
    if (m > cap) {
        ord_bitonic_global(bk, m);
        for (int i = threadIdx.x; i < m; i += kOrdT) rank[(uint32_t)bk[i]] = (int32_t)(s0 + i);
        return;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // warp-contiguous layout: element e = w * 512 + i * 32 + lane; padding (e >= m) is
    // all-ones, larger than every key, and stays last (stable passes)
    uint64_t k[kOrdItems];
    unsigned long long o = 0, a = ~0ull;
#pragma unroll
    for (int i = 0; i < kOrdItems; i++) {
        const int e = w * (32 * kOrdItems) + i * 32 + lane;
        k[i] = e < m ? bk[e] : ~0ull;
        if (e < m) {
            o |= k[i];
            a &= k[i];
        }
    }
    for (int s = 16; s > 0; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if (lane == 0) {
        s_or[w] = o;
        s_and[w] = a;
    }
    __syncthreads();
    unsigned long long vary = 0;
    {
        unsigned long long oo = 0, aa = ~0ull;
        for (int j = 0; j < 32; j++) {
            oo |= s_or[j];
            aa &= s_and[j];
        }
        vary = oo ^ aa;  // bits that differ between keys of this bucket
    }
    const uint32_t lt = lanemask_lt();
    for (int shift = 0; shift < 64; shift += 8) {
        if (((vary >> shift) & 0xffull) == 0) continue;  // (uniform over the CTA)
        for (int j = threadIdx.x; j < 256 * kOrdWcStride; j += kOrdT) wc[j] = 0;
        __syncthreads();
        uint32_t pos2[kOrdItems / 2];  // rank inside (warp, digit) < 512: two per register
#pragma unroll
        for (int i = 0; i < kOrdItems; i++) {
            const uint32_t d = (uint32_t)(k[i] >> shift) & 0xffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t c = wc[d * kOrdWcStride + w];
            __syncwarp();
            if (lane == __ffs(peers) - 1) wc[d * kOrdWcStride + w] = c + __popc(peers);
            __syncwarp();
            const uint32_t p = c + __popc(peers & lt);
            if (i & 1) pos2[i >> 1] |= p << 16;
            else pos2[i >> 1] = p;
        }
        __syncthreads();
        // per digit: exclusive scan over the 32 warps (warp w' scans digits w', w'+32, ..)
        for (int d = w; d < 256; d += 32) {
            const uint32_t x = wc[d * kOrdWcStride + lane];
            uint32_t inc = x;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, s);
                if (lane >= s) inc += y;
            }
            wc[d * kOrdWcStride + lane] = inc - x;
            if (lane == 31) dtot[d] = inc;
        }
        __syncthreads();
        if (w == 0) {  // exclusive scan of the 256 digit totals (8 per lane)
            uint32_t v8[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                v8[j] = dtot[lane * 8 + j];
                sum += v8[j];
            }
            uint32_t inc = sum;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, s);
                if (lane >= s) inc += y;
            }
            uint32_t run = inc - sum;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                dtot[lane * 8 + j] = run;
                run += v8[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kOrdItems; i++) {
            const uint32_t d = (uint32_t)(k[i] >> shift) & 0xffu;
            const uint32_t p = (i & 1) ? (pos2[i >> 1] >> 16) : (pos2[i >> 1] & 0xffffu);
            sk[dtot[d] + wc[d * kOrdWcStride + w] + p] = k[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kOrdItems; i++) k[i] = sk[w * (32 * kOrdItems) + i * 32 + lane];
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kOrdItems; i++) {
        const int e = w * (32 * kOrdItems) + i * 32 + lane;
        if (e < m) rank[(uint32_t)k[i]] = (int32_t)(s0 + e);
    }
}

}  // namespace dms
