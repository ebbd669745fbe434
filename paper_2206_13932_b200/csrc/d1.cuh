// d1.cuh -- D1 of a 3D field by PairCriticalSimplices (Alg. 3, 364-417) on
// sm_100a, with its persistent 1-cycle generators (Sec. 9, PAPER.md 1188-1215).
//
// Inputs (the "sandwich", PAPER.md 1125-1155): the critical triangles left unpaired by
// D_2 (sigma, ascending lexicographic order) and the critical edges left unpaired by D0
// (the positive 1-saddles).  Every other simplex a propagation meets is regular and is
// crossed through its discrete vector (PAPER.md 486-490).
//
// Boundary(sigma) is held as a multiset of 64-bit edge keys  rank(hi) << 32 | rank(lo)
// (hi/lo = the edge's higher/lower vertex in the order K): key order = the
// lexicographic order of edges (PAPER.md 1380-1414), so max(Boundary) is the largest
// key.  A thread-private binary max-heap with lazy cancellation holds it (mod-2
// addition, PAPER.md 492-497: two equal keys on top cancel).  A column stored at a stop
// is written sorted descending -- a valid max-heap as it stands.
//
// Parallel form (PAPER.md 1136-1150, "temporary pair + compare-and-swap"), in rounds:
//   phase 1  every active sigma propagates (regular edges: add the boundary of the
//            paired triangle; critical edges owned by an earlier sigma': add the column
//            sigma' stopped with) until its maximum tau is a critical edge that no
//            earlier sigma owns; it stores its column and claims tau (atomicMin of a
//            round-tagged sigma index).  Between rounds the smallest claimant becomes
//            tau's owner; a displaced later owner and the losing claimants stay active.
//            The final owners are the pairs of the sequential algorithm (the pivots of
//            a left-to-right column reduction do not depend on which earlier column
//            with the same pivot is added).
//   phase 2  (generators) the columns of phase 1 may have added a column its owner
//            later changed; the earliest cycle of Sec. 9 is the column of the
//            sequential algorithm, so every sigma is propagated again from its
//            boundary with the final owners known: at a critical tau owned by an
//            earlier sigma' it adds sigma''s FINAL column once sigma' is done, and it
//            is done when it reaches the tau it owns.
// Heaps start in local memory (kD1Cap entries); a sigma whose heap would overflow is
// handed (as an unsorted bag) to k_d1_big, which continues it in a global-memory heap
// that grows by doubling.  All columns live in one append-only arena; an allocation
// that does not fit leaves the sigma unchanged and sets a flag, and the host grows the
// arena and repeats the round for it.
#pragma once
#include "common.cuh"
#include "diag.cuh"
#include "star.cuh"

namespace dms {

constexpr int kD1Cap = 96;  // local-memory heap entries per thread

enum : uint8_t { D1_STOP = 1, D1_DONE = 2, D1_WAIT = 3, D1_BIG = 4, D1_RETRY = 5, D1_ERR = 6 };

struct D1Args {
    Geo3 g;
    const int32_t* rank;
    const int32_t* order;  // order[rank[v]] = v
    const unsigned long long* hkey;  // hash of the positive 1-saddles: key -> index
    const int32_t* hval;
    uint32_t hmask;
    int32_t* owner;               // [n0] sigma index owning the edge, -1
    unsigned long long* claim;    // [n0] phase 1: (tag << 32) | sigma, atomicMin
    int32_t* stop;                // [nsig] index of the edge sigma stopped at
    int32_t* done;                // [nsig] phase 2: final column written
    long long* col_off;           // [nsig] column in the arena
    int32_t* col_len;
    uint8_t* status;              // [nsig]
    unsigned long long* arena;
    unsigned long long* arena_top;
    unsigned long long arena_cap;
    const int32_t* active;
    int32_t nactive;
    int32_t* big;  // deferred sigma indices
    int32_t* nbig;
    int32_t* grab;
    int* err;  // bit 0: arena full (retry), bits 1-4: invariant broken (which one)
    long long* dbg;  // [4] first failure: sigma, tau, j, o
    unsigned long long tag;  // phase-1 claim tag (decreasing over rounds)
    int phase;
    int lcap;  // local heap capacity used (<= kD1Cap; smaller only to exercise the global path)
};

__device__ __forceinline__ uint32_t d1_hash(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return (uint32_t)k;
}

__device__ __forceinline__ unsigned long long ekey(uint32_t ra, uint32_t rb) {
    return ra > rb ? ((unsigned long long)ra << 32 | rb) : ((unsigned long long)rb << 32 | ra);
}

// the two vertices of an anchored edge id
__device__ __forceinline__ void edge_verts(const Geo3& g, const StarTab& S, int64_t id, int64_t& p, int64_t& q) {
    const int64_t a = id / g.ncell[1];
    const int k = (int)(id % g.ncell[1]);
    p = a;
    q = a + lin_mask(g, S.chain[1][k][0]);
}

__device__ __forceinline__ int d1_lookup(const D1Args& A, unsigned long long key) {
    uint32_t h = d1_hash(key) & A.hmask;
    while (true) {
        const unsigned long long k = __ldg(A.hkey + h);
        if (k == key) return __ldg(A.hval + h);
        if (k == 0ull) return -1;
        h = (h + 1) & A.hmask;
    }
}

// slot s of the neighbour at linear offset d (slots sorted by offset)
__device__ __forceinline__ int slot_of_offset(const StarTab& S, int32_t d) {
    int s = 0;
#pragma unroll
    for (int b = 8; b > 0; b >>= 1)
        if (s + b < kMaxNE && S.lin[s + b - 1] < d) s += b;
    while (S.lin[s] != d) s++;
    return s;
}

// tau regular: the boundary of its paired triangle minus tau -> k1, k2; returns true.
// tau critical: returns false.  Edges paired with a vertex never reach here (they are
// never the highest edge of a cycle: the lowest lower neighbour of x comes last).
__device__ __forceinline__ bool d1_regular(const D1Args& A, const StarTab& S, unsigned long long tau,
                                           unsigned long long& k1, unsigned long long& k2) {
    const uint32_t rh = (uint32_t)(tau >> 32), rl = (uint32_t)tau;
    const int32_t x = __ldg(A.order + rh), y = __ldg(A.order + rl);
    const int s = slot_of_offset(S, y - x);
    const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(A.g.grad) + x);
#pragma unroll 1
    for (int i = 0; i < 6; i++) {
        const int t = S.edge_tri[s][i];
        if (t == 255) break;
        const uint32_t code = (uint32_t)((t < 32 ? (w.x >> (2 * t)) : (w.y >> (2 * (t - 32)))) & 3ull);
        const int a = S.tri_a[t], b = S.tri_b[t];
        if ((code == 1u && a == s) || (code == 2u && b == s)) {
            const int u = a == s ? b : a;
            const uint32_t rz = (uint32_t)__ldg(A.rank + x + S.lin[u]);
            k1 = (unsigned long long)rh << 32 | rz;
            k2 = ekey(rl, rz);
            return true;
        }
    }
    return false;
}

__device__ __forceinline__ bool arena_alloc(const D1Args& A, unsigned long long n, unsigned long long& off) {
    off = atomicAdd(A.arena_top, n);
    if (off + n > A.arena_cap) {
        atomicOr(A.err, 1);
        return false;
    }
    return true;
}

__device__ __noinline__ void d1_fail(const D1Args& A, int bit, int sig, unsigned long long tau, int j, int o) {
    if ((atomicOr(A.err, bit) & 30) == 0) {
        A.dbg[0] = sig;
        A.dbg[1] = (long long)tau;
        A.dbg[2] = j;
        A.dbg[3] = o;
    }
}

// binary max-heap with lazy mod-2 cancellation over a plain array
template <typename P>
struct Heap {
    P h;
    int n = 0;
    __device__ __forceinline__ void push(unsigned long long k) {
        int i = n++;
        while (i > 0) {
            const int p = (i - 1) >> 1;
            const unsigned long long hp = h[p];
            if (hp >= k) break;
            h[i] = hp;
            i = p;
        }
        h[i] = k;
    }
    __device__ __forceinline__ unsigned long long pop() {
        const unsigned long long top = h[0];
        const unsigned long long k = h[--n];
        int i = 0;
        while (true) {
            int c = 2 * i + 1;
            if (c >= n) break;
            unsigned long long hc = h[c];
            if (c + 1 < n) {
                const unsigned long long h2 = h[c + 1];
                if (h2 > hc) { hc = h2; c++; }
            }
            if (hc <= k) break;
            h[i] = hc;
            i = c;
        }
        if (n > 0) h[i] = k;
        return top;
    }
    // the maximum of the mod-2 set (0: empty)
    __device__ __forceinline__ unsigned long long popmax() {
        while (n > 0) {
            const unsigned long long t = pop();
            if (n > 0 && h[0] == t) {
                pop();
                continue;
            }
            return t;
        }
        return 0ull;
    }
};

struct LocalArr {
    unsigned long long a[kD1Cap];
    __device__ __forceinline__ unsigned long long& operator[](int i) { return a[i]; }
};
struct GlobalArr {
    unsigned long long* a;
    __device__ __forceinline__ unsigned long long& operator[](int i) { return a[i]; }
};

// room for m more entries; the global heap grows by doubling inside the arena
__device__ __forceinline__ bool heap_room(const D1Args& A, Heap<LocalArr>& H, int m) { return H.n + m <= A.lcap; }
__device__ __forceinline__ bool heap_room(const D1Args& A, Heap<GlobalArr>& H, int m, int& cap) {
    if (H.n + m <= cap) return true;
    int nc = cap;
    while (H.n + m > nc) nc *= 2;
    unsigned long long off;
    if (!arena_alloc(A, (unsigned long long)nc, off)) return false;
    for (int i = 0; i < H.n; i++) A.arena[off + i] = H.h.a[i];
    H.h.a = A.arena + off;
    cap = nc;
    return true;
}

// write the column (tau first, then the rest of the heap, sorted descending, cancelled)
template <typename P>
__device__ __forceinline__ bool d1_store(const D1Args& A, int sig, Heap<P>& H, unsigned long long tau) {
    unsigned long long off;
    if (!arena_alloc(A, (unsigned long long)H.n + 1, off)) return false;
    unsigned long long* out = A.arena + off;
    int len = 0;
    out[len++] = tau;
    while (true) {
        const unsigned long long k = H.popmax();
        if (!k) break;
        out[len++] = k;
    }
    A.col_off[sig] = (long long)off;
    A.col_len[sig] = len;
    return true;
}

// Propagate sigma from the column in H (Alg. 3 lines 5-15).  Returns the
// status; on D1_BIG the heap (tau pushed back) is the column as a multiset.
template <typename P, typename Room>
__device__ __forceinline__ uint8_t d1_propagate(const D1Args& A, const StarTab& S, int sig, Heap<P>& H, Room room,
                                                unsigned long long& tau_out, int& j_out) {
    while (true) {
        const unsigned long long tau = H.popmax();
        if (!tau) {
            d1_fail(A, 2, sig, 0ull, -1, -1);  // an empty boundary: a 2-saddle that kills no cycle (grids are balls)
            return D1_ERR;
        }
        unsigned long long k1, k2;
        if (d1_regular(A, S, tau, k1, k2)) {
            if (!room(2)) {
                H.push(tau);
                return D1_BIG;
            }
            H.push(k1);
            H.push(k2);
            continue;
        }
        const int j = d1_lookup(A, tau);
        if (j < 0) {
            d1_fail(A, 4, sig, tau, j, -1);  // a D0 death edge is never the highest edge of a cycle
            return D1_ERR;
        }
        const int o = A.owner[j];
        bool add;
        if (A.phase == 1) {
            add = o >= 0 && o < sig;
        } else {
            if (o == sig) {
                tau_out = tau;
                j_out = j;
                return D1_DONE;
            }
            if (o < 0 || o > sig) {
                d1_fail(A, 8, sig, tau, j, o);
                return D1_ERR;
            }
            add = *(volatile const int32_t*)(A.done + o) != 0;
            if (add) __threadfence();
        }
        if (add) {
            const long long off = *(volatile const long long*)(A.col_off + o);
            const int len = *(volatile const int32_t*)(A.col_len + o);
            if (!room(len - 1)) {
                H.push(tau);
                return D1_BIG;
            }
            // L2 loads: in phase 2 the column may have been written during this kernel by
            // another SM (its done flag was seen), so a stale L1 line must not serve it
            for (int i = 1; i < len; i++) H.push(__ldcg(A.arena + off + i));
            continue;
        }
        tau_out = tau;
        j_out = j;
        return A.phase == 1 ? D1_STOP : D1_WAIT;
    }
}

template <typename P>
__device__ __forceinline__ void d1_finish(const D1Args& A, int sig, Heap<P>& H, uint8_t st, unsigned long long tau, int j) {
    if (st == D1_STOP || st == D1_WAIT || st == D1_DONE) {
        if (!d1_store(A, sig, H, tau)) {
            A.status[sig] = D1_RETRY;
            return;
        }
        A.stop[sig] = j;
        if (st == D1_STOP) {
            atomicMin(A.claim + j, A.tag | (unsigned)sig);
        } else if (st == D1_DONE) {
            __threadfence();
            *(volatile int32_t*)(A.done + sig) = 1;
        }
    }
    A.status[sig] = st;
}

// one round over the active sigmas, local-memory heaps; persistent threads grab work
__global__ void __launch_bounds__(128) k_d1_round(D1Args A) {
    const StarTab& S = *A.g.tab;
    Heap<LocalArr> H;
    while (true) {
        int i;
        {
            // one atomic per warp: lanes take consecutive items
            const unsigned m = __activemask();
            const int lane = threadIdx.x & 31;
            const int leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(A.grab, __popc(m));
            base = __shfl_sync(m, base, leader);
            i = base + __popc(m & lanemask_lt());
        }
        if (i >= A.nactive) return;
        const int sig = A.active[i];
        const long long off = A.col_off[sig];
        const int len = A.col_len[sig];
        if (len > A.lcap || len < 0) {  // too large, or a bag: straight to the global path
            A.status[sig] = D1_BIG;
            A.big[atomicAdd(A.nbig, 1)] = sig;
            continue;
        }
        H.n = len;
        for (int k = 0; k < len; k++) H.h[k] = A.arena[off + k];  // sorted descending = a heap
        unsigned long long tau = 0;
        int j = -1;
        const uint8_t st = d1_propagate(A, S, sig, H, [&](int m) { return heap_room(A, H, m); }, tau, j);
        if (st == D1_BIG) {
            // hand the multiset over: the global path heapifies it
            unsigned long long o2;
            if (!arena_alloc(A, (unsigned long long)H.n, o2)) {
                A.status[sig] = D1_RETRY;
                continue;
            }
            for (int k = 0; k < H.n; k++) A.arena[o2 + k] = H.h[k];
            A.col_off[sig] = (long long)o2;
            A.col_len[sig] = -H.n;  // negative: an unsorted multiset
            A.status[sig] = D1_BIG;
            A.big[atomicAdd(A.nbig, 1)] = sig;
            continue;
        }
        d1_finish(A, sig, H, st, tau, j);
    }
}

// the deferred (large) sigmas: one thread each, heap in the arena
__global__ void k_d1_big(D1Args A) {
    const StarTab& S = *A.g.tab;
    const int nb = *A.nbig;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
        const int sig = A.big[b];
        const long long off = A.col_off[sig];
        const int len0 = A.col_len[sig];
        const int len = len0 < 0 ? -len0 : len0;
        int cap = 256;
        while (cap < 2 * len) cap *= 2;
        unsigned long long hoff;
        if (!arena_alloc(A, (unsigned long long)cap, hoff)) {
            A.status[sig] = D1_RETRY;
            continue;
        }
        Heap<GlobalArr> H;
        H.h.a = A.arena + hoff;
        H.n = 0;
        if (len0 >= 0) {
            for (int k = 0; k < len; k++) H.h.a[k] = A.arena[off + k];
            H.n = len;
        } else {
            for (int k = 0; k < len; k++) H.push(A.arena[off + k]);
        }
        unsigned long long tau = 0;
        int j = -1;
        uint8_t st = d1_propagate(A, S, sig, H, [&](int m) { return heap_room(A, H, m, cap); }, tau, j);
        if (st == D1_BIG) st = D1_RETRY;  // the arena is full; the host grows it and repeats
        if (st == D1_RETRY) {
            A.status[sig] = D1_RETRY;
            continue;
        }
        d1_finish(A, sig, H, st, tau, j);
    }
}

// phase 1, between rounds: the smallest claimant of each edge becomes its owner; the
// displaced owner, the losing claimants and the retries stay active
__global__ void k_d1_resolve(D1Args A, int32_t* next, int32_t* nnext) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nactive) return;
    const int sig = A.active[i];
    const uint8_t st = A.status[sig];
    int keep = -1, keep2 = -1;
    if (st == D1_STOP) {
        const int j = A.stop[sig];
        if (A.claim[j] == (A.tag | (unsigned)sig)) {
            const int old = A.owner[j];
            A.owner[j] = sig;
            if (old >= 0) keep2 = old;
        } else {
            keep = sig;
        }
    } else if (st == D1_WAIT || st == D1_RETRY || st == D1_BIG) {
        keep = sig;
    }
    if (keep >= 0) next[atomicAdd(nnext, 1)] = keep;
    if (keep2 >= 0) next[atomicAdd(nnext, 1)] = keep2;
}

// setup ---------------------------------------------------------------------------

__global__ void k_d1_invert(const int32_t* __restrict__ rank, int64_t n, int32_t* __restrict__ order) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) order[rank[v]] = (int32_t)v;
}

__global__ void k_d1_hash(Geo3 g, const int32_t* __restrict__ rank, const int64_t* __restrict__ un0, int64_t n0,
                          unsigned long long* hkey, int32_t* hval, uint32_t hmask) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n0) return;
    const StarTab& S = *g.tab;
    int64_t p, q;
    edge_verts(g, S, un0[j], p, q);
    const unsigned long long key = ekey((uint32_t)rank[p], (uint32_t)rank[q]);
    uint32_t h = d1_hash(key) & hmask;
    while (true) {
        const unsigned long long prev = atomicCAS(hkey + h, 0ull, key);
        if (prev == 0ull) {
            hval[h] = (int32_t)j;
            return;
        }
        h = (h + 1) & hmask;
    }
}

// the boundary of each sigma (three edge keys, sorted descending) at arena[3 i]
__global__ void k_d1_init(Geo3 g, const int32_t* __restrict__ rank, const int64_t* __restrict__ sig_ids, int64_t nsig,
                          unsigned long long* arena, long long* col_off, int32_t* col_len, int32_t* active,
                          int32_t* done) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsig) return;
    const StarTab& S = *g.tab;
    const int64_t id = sig_ids[i];
    const int64_t a = id / g.ncell[2];
    const int k = (int)(id % g.ncell[2]);
    const uint32_t r0 = (uint32_t)rank[a];
    const uint32_t r1 = (uint32_t)rank[a + lin_mask(g, S.chain[2][k][0])];
    const uint32_t r2 = (uint32_t)rank[a + lin_mask(g, S.chain[2][k][1])];
    unsigned long long e[3] = {ekey(r0, r1), ekey(r0, r2), ekey(r1, r2)};
    if (e[0] < e[1]) { unsigned long long t = e[0]; e[0] = e[1]; e[1] = t; }
    if (e[1] < e[2]) { unsigned long long t = e[1]; e[1] = e[2]; e[2] = t; }
    if (e[0] < e[1]) { unsigned long long t = e[0]; e[0] = e[1]; e[1] = t; }
    for (int q = 0; q < 3; q++) arena[3 * i + q] = e[q];
    col_off[i] = 3 * i;
    col_len[i] = 3;
    active[i] = (int32_t)i;
    done[i] = 0;
}

// outputs ---------------------------------------------------------------------------

// D1 pair of sigma i: (the edge it owns, sigma), in increasing death order (Alg. 3 l. 19)
__global__ void k_d1_emit(Geo3 g, const int32_t* __restrict__ stop, const int32_t* __restrict__ owner,
                          const int64_t* __restrict__ un0, const int64_t* __restrict__ sig_ids, int64_t nsig,
                          PairRec* pairs, int* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsig) return;
    const StarTab& S = *g.tab;
    const int j = stop[i];
    if (owner[j] != (int32_t)i) atomicOr(err, 16);
    PairRec r;
    r.birth_id = un0[j];
    const int64_t bv = max_vertex(g, S, 1, r.birth_id);
    r.birth_vertex = (int32_t)bv;
    r.birth_value = g.f[bv];
    r.death_id = sig_ids[i];
    const int64_t dv = max_vertex(g, S, 2, r.death_id);
    r.death_vertex = (int32_t)dv;
    r.death_value = g.f[dv];
    pairs[i] = r;
}

__global__ void k_d1_unowned(const int32_t* __restrict__ owner, int64_t n0, uint32_t* flags) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n0) flags[j] = owner[j] < 0 ? 1u : 0u;
}

__global__ void k_d1_emit_unowned(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ pos,
                                  const int64_t* __restrict__ un0, int64_t n0, int64_t* out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n0 && flags[j]) out[pos[j]] = un0[j];
}

__global__ void k_d1_gen_len(const int32_t* __restrict__ col_len, int64_t nsig, uint32_t* len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nsig) len[i] = (uint32_t)col_len[i];
}

// the generator of sigma i (its final column) as anchored edge ids in ascending
// lexicographic order; one warp per sigma
__global__ void k_d1_gen_emit(Geo3 g, const int32_t* __restrict__ order, const long long* __restrict__ col_off,
                              const int32_t* __restrict__ col_len, const uint32_t* __restrict__ pos, int64_t nsig,
                              const unsigned long long* __restrict__ arena, int64_t* gen_off, int64_t* gen) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nsig) return;
    const StarTab& S = *g.tab;
    const int len = col_len[i];
    const long long off = col_off[i];
    const int64_t base = pos[i];
    if (lane == 0) {
        gen_off[i] = base;
        if (i == nsig - 1) gen_off[nsig] = base + len;
    }
    for (int k = lane; k < len; k += 32) {
        const unsigned long long key = arena[off + len - 1 - k];
        const int32_t x = order[key >> 32], y = order[(uint32_t)key];
        const int s = slot_of_offset(S, y - x);
        gen[base + k] = (int64_t)g.ncell[1] * (x + (int64_t)S.e_anc[s][0] + (int64_t)g.Lx * S.e_anc[s][1] +
                                               (int64_t)g.Lx * g.Ly * S.e_anc[s][2]) +
                        S.e_k[s];
    }
}

}  // namespace dms
