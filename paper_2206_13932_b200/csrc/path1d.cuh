// path1d.cuh -- the elder-rule union-find of a 1D field's diagrams on its path graph
// (sm_100a).
//
// In 1D the graphs of Sec. 5 are paths: G_D0 (PAPER.md 2494-2685) alternates minima
// (nodes) and critical edges (arcs) along the line; G_D_{d-1} (PAPER.md 2728-2825)
// alternates maxima (nodes) and minima (arcs) with the virtual maximum at both ends.
// On a path the Union-Find of Sec. 5.1(c,d) has a closed form: arcs enter in processing
// order, so a node i (older = smaller age) is the oldest node of its component until the
// component reaches a node older than i; that happens first through the nearest older
// node on the left or on the right, at the moment the LAST arc between them enters, so
//     i dies at   min( max key of the arcs between NOL(i) and i,
//                      max key of the arcs between i and NOR(i) )
// (NOL / NOR = nearest older node to the left / right, infinity if none), and the arc
// reaching that maximum is the one that kills i (the elder rule, PAPER.md 1641-1664).
// The globally oldest node (and the virtual maximum, age 0 at both ends) never dies; an
// arc killing no node is unpaired (on the ring of D_{d-1}: the last arc).
//
// Kernels: k_path_local -- one thread per block of kPB nodes runs the sequential stack
// sweep (NOL/NOR inside the block, walls as running maxima of packed (key, arc)); the
// nodes whose nearest older node lies outside the block are the block's prefix / suffix
// minima, kept as sorted lists.  k_path_sparse -- sparse tables over the blocks (oldest
// age, largest arc).  k_path_resolve -- the cross-block walls of those nodes by binary
// lifting over the blocks plus a binary search in the older block's list.
// k_path_emit -- the dying node of every arc, in the emission-order layout the rest of
// the diagram pipeline reads (u.out).
#pragma once
#include "common.cuh"

namespace dms {

constexpr int kPB = 64;           // nodes per block (one thread each)
constexpr int kPLog = 24;         // sparse-table levels (blocks < 2^24)
constexpr unsigned long long kPInf = ~0ull;

struct PathArgs {
    int64_t P;                          // nodes on the path (arcs: P - 1)
    int64_t nb;                         // blocks
    // spatial -> emission maps: node s is node_em(s), arc s (between nodes s, s+1) arc_em(s)
    const int64_t* node_map;            // emission index of the s-th spatial entry
    const int64_t* arc_map;
    int64_t node_off;                   // node_em(s) = node_map[s - node_off] (virtual ends: -1)
    int32_t virt;                       // emission index of the virtual node (Dtop), -1: none
    const uint32_t* key;                // per arc (emission order): processing index
    const int32_t* age;                 // per node (emission order): smaller = older
    const int32_t* arc_a;               // traced arcs (emission order), for the structure check
    const int32_t* arc_b;
    int* bad;                           // set if the traced arcs are not this path
    // scratch
    uint32_t* sage;                     // [P] ages in spatial order
    unsigned long long* sarc;           // [P] packed (key << 32 | s) of arc s, spatial order
    unsigned long long* lw;             // [P] left wall (resolved, or partial from block start)
    unsigned long long* rw;             // [P] right wall (resolved, or partial to block end)
    uint8_t* unres;                     // [P] bit 0: left unresolved, bit 1: right unresolved
    int32_t* pre;                       // [P] per block: prefix minima (node indices)
    int32_t* suf;                       // [P] per block: suffix minima
    int32_t* npre;                      // [nb]
    int32_t* nsuf;                      // [nb]
    unsigned long long* bnd;            // [nb] the arc after the block's last node
    uint32_t* tmin;                     // [kPLog][nb] oldest age over [b, b + 2^k)
    unsigned long long* tspan;          // [kPLog][nb] largest arc over blocks [b, b + 2^k), incl. their next arc
    unsigned long long* dw;             // [P] the arc killing the node (packed), kPInf: never
    int levels;                         // sparse-table levels built
    int32_t* out;                       // [arcs] emission order: dying node, -1 unpaired
};

__device__ __forceinline__ int64_t path_node_em(const PathArgs& A, int64_t s) {
    const int64_t j = s - A.node_off;
    return (j < 0 || j >= A.P - 2 * A.node_off) ? (int64_t)A.virt : A.node_map[j];
}
__device__ __forceinline__ unsigned long long path_arc(const PathArgs& A, int64_t s) {
    const int64_t e = A.arc_map[s];
    return ((unsigned long long)A.key[e] << 32) | (unsigned long long)s;
}

// the traced arcs must be exactly the path (structure check) + ages in spatial order
__global__ void k_path_check(PathArgs A) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= A.P) return;
    const int64_t ne = path_node_em(A, s);
    A.sage[s] = (uint32_t)A.age[ne];
    if (s + 1 < A.P) {
        const int64_t e = A.arc_map[s];
        A.sarc[s] = ((unsigned long long)A.key[e] << 32) | (unsigned long long)s;
        const int64_t l = ne, r = path_node_em(A, s + 1);
        const int64_t a = A.arc_a[e], b = A.arc_b[e];
        if (!((a == l && b == r) || (a == r && b == l))) atomicOr(A.bad, 1);
    }
}

// one thread per block of kPB nodes; a CTA of kPT threads stages its kPT blocks' ages
// and arcs in shared memory (coalesced), then every thread sweeps its block
constexpr int kPT = 32;
__global__ void __launch_bounds__(kPT) k_path_local(PathArgs A) {
    __shared__ uint32_t sa[kPT * kPB];
    __shared__ unsigned long long sr[kPT * kPB];
    // the stacks in shared memory too ([slot][thread], conflict free): local memory would
    // live in the L1 that the staging already fills
    __shared__ unsigned long long sws[kPB * kPT];
    __shared__ uint8_t sts[kPB * kPT];
    const int64_t base = (int64_t)blockIdx.x * kPT * kPB;
    for (int i = threadIdx.x; i < kPT * kPB; i += kPT) {
        const int64_t s = base + i;
        sa[i] = s < A.P ? A.sage[s] : 0u;
        sr[i] = s + 1 < A.P ? A.sarc[s] : 0ull;
    }
    __syncthreads();
    const int64_t b = (int64_t)blockIdx.x * kPT + threadIdx.x;
    if (b >= A.nb) return;
    const int64_t s0 = b * kPB, s1 = min(s0 + kPB, A.P);
    const int l0 = threadIdx.x * kPB;  // the block's offset in shared memory
    uint8_t* stk = sts + threadIdx.x;
    unsigned long long* sw = sws + threadIdx.x;
#define STK(i) stk[(i) * kPT]
#define SW(i) sw[(i) * kPT]
    int top = -1, np = 0;
    unsigned long long pm = 0;  // largest arc from the block start
    uint32_t amin = 0xffffffffu;
    for (int64_t s = s0; s < s1; s++) {
        const int l = l0 + (int)(s - s0);
        const uint32_t a = sa[l];
        amin = min(amin, a);
        if (s > s0) {
            const unsigned long long w = sr[l - 1];
            pm = max(pm, w);
            SW(top) = max(SW(top), w);
        }
        uint8_t fl = 0;
        while (top >= 0 && sa[l0 + STK(top)] > a) {  // stk[top] is younger: its NOR is s
            A.rw[s0 + STK(top)] = SW(top);
            if (top > 0) SW(top - 1) = max(SW(top - 1), SW(top));
            top--;
        }
        if (top >= 0) {
            A.lw[s] = SW(top);  // NOL(s) = stk[top], the arcs between them
        } else {
            A.lw[s] = pm;       // partial: from the block start
            fl |= 1;
            A.pre[s0 + np++] = (int32_t)s;
        }
        A.unres[s] = fl;
        ++top;
        STK(top) = (uint8_t)(s - s0);
        SW(top) = 0;
    }
    // the stack now holds the suffix minima (no older node to their right in the block)
    unsigned long long acc = 0;
    for (int t = top; t >= 0; t--) {
        acc = max(acc, SW(t));
        const int64_t i = s0 + STK(t);
        A.rw[i] = acc;  // partial: to the block end
        A.unres[i] |= 2;
        A.suf[s0 + t] = (int32_t)i;
    }
    A.npre[b] = np;
    A.nsuf[b] = top + 1;
    A.bnd[b] = s1 < A.P ? sr[l0 + (int)(s1 - 1 - s0)] : 0ull;
    A.tmin[b] = amin;
    A.tspan[b] = max(pm, A.bnd[b]);
#undef STK
#undef SW
}

// level k of the sparse tables from level k - 1
__global__ void k_path_sparse(PathArgs A, int k) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= A.nb) return;
    const int64_t h = int64_t(1) << (k - 1);
    const uint32_t* m0 = A.tmin + (size_t)(k - 1) * A.nb;
    const unsigned long long* s0 = A.tspan + (size_t)(k - 1) * A.nb;
    uint32_t m = m0[b];
    unsigned long long w = s0[b];
    if (b + h < A.nb) {
        m = min(m, m0[b + h]);
        w = max(w, s0[b + h]);
    }
    A.tmin[(size_t)k * A.nb + b] = m;
    A.tspan[(size_t)k * A.nb + b] = w;
}

// largest arc over the blocks [lo, hi] (hi >= lo), including each block's next arc
__device__ __forceinline__ unsigned long long path_span(const PathArgs& A, int64_t lo, int64_t hi) {
    unsigned long long w = 0;
    int64_t c = lo;
    for (int k = A.levels - 1; k >= 0 && c <= hi; k--) {
        if (c + (int64_t(1) << k) - 1 <= hi) {
            w = max(w, A.tspan[(size_t)k * A.nb + c]);
            c += int64_t(1) << k;
        }
    }
    return w;
}

// the death arc of every node: the walls found inside its block, or across blocks by
// binary lifting over the blocks' oldest ages and a binary search in the older block's
// suffix / prefix list (the partial walls lw / rw are only read here)
__global__ void k_path_resolve(PathArgs A) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= A.P) return;
    const uint8_t fl = A.unres[s];
    unsigned long long L = A.lw[s], R = A.rw[s];
    const uint32_t a = A.sage[s];
    const int64_t b = s / kPB;
    const int levels = A.levels;
    if (fl & 1) {  // the nearest older node to the left lies in an earlier block
        int64_t c = b - 1;
        for (int k = levels - 1; k >= 0; k--) {
            const int64_t lo = c - (int64_t(1) << k) + 1;
            if (lo >= 0 && A.tmin[(size_t)k * A.nb + lo] >= a) c = lo - 1;
        }
        if (c < 0) {
            L = kPInf;
        } else {
            // the last suffix minimum of block c older than s (ages increase along the list)
            const int32_t* Ls = A.suf + c * kPB;
            int lo = 0, hi = A.nsuf[c] - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (A.sage[Ls[mid]] < a) lo = mid;
                else hi = mid - 1;
            }
            unsigned long long w = max(L, max(A.rw[Ls[lo]], A.bnd[c]));
            if (c + 1 <= b - 1) w = max(w, path_span(A, c + 1, b - 1));
            L = w;
        }
    }
    if (fl & 2) {  // the nearest older node to the right lies in a later block
        int64_t c = b + 1;
        for (int k = levels - 1; k >= 0; k--) {
            if (c < A.nb && c + (int64_t(1) << k) <= A.nb && A.tmin[(size_t)k * A.nb + c] >= a) c += int64_t(1) << k;
        }
        if (c >= A.nb) {
            R = kPInf;
        } else {
            // the first prefix minimum of block c older than s (ages decrease along the list)
            const int32_t* Lp = A.pre + c * kPB;
            int lo = 0, hi = A.npre[c] - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (A.sage[Lp[mid]] < a) hi = mid;
                else lo = mid + 1;
            }
            unsigned long long w = max(R, max(A.lw[Lp[lo]], A.bnd[b]));
            if (b + 1 <= c - 1) w = max(w, path_span(A, b + 1, c - 1));
            R = w;
        }
    }
    A.dw[s] = min(L, R);
}

__global__ void k_path_emit(PathArgs A) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= A.P) return;
    const unsigned long long w = A.dw[s];
    const int64_t ne = path_node_em(A, s);
    if (w == kPInf || ne == A.virt) return;  // the oldest node, the virtual maximum
    const int64_t arc = (int64_t)(w & 0xffffffffull);
    A.out[A.arc_map[arc]] = (int32_t)ne;
}

__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

// spatial order of the 1D critical records from the gradient kernel's per-CTA table:
// CTA t (vertices [1024 t, 1024 t + 1024)) wrote its cnt[k][t] records of dimension k at
// emission positions base[k][t]..; its spatial positions start at the scan of cnt[k]
__global__ void k_path_spatial(const uint32_t* __restrict__ base, const uint32_t* __restrict__ cnt,
                               const uint32_t* __restrict__ scan, int64_t ntiles, int64_t* __restrict__ map) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const uint32_t b = base[t], c = cnt[t], o = scan[t];
    for (uint32_t k = lane; k < c; k += 32) map[o + k] = (int64_t)b + k;
}

}  // namespace dms
