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

// star tables of the propagation step (built on the host from StarTab)
struct alignas(16) D1Tab {
    int32_t lin[kMaxNE];
    uint8_t etri[kMaxNE][6];   // triangle slots containing the edge x-n_s (255: none)
    uint8_t eoth[kMaxNE][6];   // the triangle's other link vertex slot u
    uint8_t ecode[kMaxNE][6];  // the gradient code that pairs the triangle with that edge (1: tri_a, 2: tri_b)
    uint8_t sdiff[kMaxNE][kMaxNE];  // slot w with lin[w] == lin[u] - lin[s] (255: not a neighbour)
};

inline void build_d1_tab(const StarTab& S, D1Tab* T) {
    for (int a = 0; a < kMaxNE; a++) {
        T->lin[a] = a < S.ne ? S.lin[a] : 0x7fffffff;
        for (int i = 0; i < 6; i++) {
            const int t = a < S.ne ? S.edge_tri[a][i] : 255;
            T->etri[a][i] = (uint8_t)t;
            T->eoth[a][i] = t == 255 ? 0 : (S.tri_a[t] == a ? S.tri_b[t] : S.tri_a[t]);
            T->ecode[a][i] = t == 255 ? 0 : (S.tri_a[t] == a ? 1 : 2);
        }
        for (int b = 0; b < kMaxNE; b++) {
            T->sdiff[a][b] = 255;
            if (a >= S.ne || b >= S.ne) continue;
            for (int w = 0; w < S.ne; w++)
                if (S.lin[w] == S.lin[b] - S.lin[a]) T->sdiff[a][b] = (uint8_t)w;
        }
    }
}

struct D1Snap {
    int32_t sig, seq, len, pad;  // seq: owner columns added before this column was stored
    long long off;
};

enum : uint8_t { D1_STOP = 1, D1_DONE = 2, D1_WAIT = 3, D1_BIG = 4, D1_RETRY = 5, D1_ERR = 6 };

struct D1Args {
    Geo3 g;
    const D1Tab* tab;
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
    int adds;  // large-2-saddle path: owner columns up to this length are pushed, longer merged
    int4* deps;          // phase 1: (sigma, owner, edge, sigma's add number) of every column added
    int* ndeps;
    long long deps_cap;
    int32_t* nadd;       // [nsig] owner columns added so far by the stored column of sigma
    struct D1Snap* snaps;  // phase 1: every stored column (a snapshot of sigma's propagation)
    int* nsnaps;
    long long snaps_cap;
    unsigned long long* prof;  // diagnostics (DMS_D1_STATS): k_d1_bigc cycles / counts per action
    unsigned* st_steps;  // diagnostics (DMS_D1_STATS): per sigma, regular steps / column adds / pushed keys
    unsigned* st_adds;
    unsigned* st_pushed;
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
template <typename TB>
__device__ __forceinline__ int slot_of_offset(const TB& S, int32_t d) {
    int s = 0;
#pragma unroll
    for (int b = 8; b > 0; b >>= 1)
        if (s + b < kMaxNE && S.lin[s + b - 1] < d) s += b;
    while (S.lin[s] != d) s++;
    return s;
}

// One regular step's lookups for the edge (x, x + lin[s]): its gradient word and, in the
// same round of loads, the ranks of the third vertex of every triangle containing the
// edge (speculatively, clamped to the grid; only the paired one is used).  Returns the
// slot u of the paired triangle's third vertex (rz = its rank), or -1 if the edge is
// critical.  Edges paired with a vertex never get here: they are never the highest edge
// of a cycle (the lowest lower neighbour of x comes last).
__device__ __forceinline__ int d1_pair_lookup(const D1Args& A, const D1Tab& T, int32_t x, int s, uint32_t& rz) {
    const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(A.g.grad) + x);
    uint32_t r[6];
    const int64_t nmax = A.g.N - 1;
#pragma unroll
    for (int i = 0; i < 6; i++) {
        const int64_t z = (int64_t)x + T.lin[T.eoth[s][i]];
        r[i] = (uint32_t)__ldg(A.rank + (z < 0 ? 0 : (z > nmax ? nmax : z)));
    }
    // the edge slot's nibble: 1 + the slot of the paired triangle's third vertex (0: none)
    const int u = (int)((w.x >> (4 * s)) & 15ull) - 1;
#pragma unroll
    for (int i = 0; i < 6; i++)
        if (T.eoth[s][i] == u) rz = r[i];
    return u;
}

// tau regular: the boundary of its paired triangle minus tau -> k1, k2; returns true.
__device__ __forceinline__ bool d1_regular(const D1Args& A, const D1Tab& T, unsigned long long tau,
                                           unsigned long long& k1, unsigned long long& k2) {
    const uint32_t rh = (uint32_t)(tau >> 32), rl = (uint32_t)tau;
    const int32_t x = __ldg(A.order + rh), y = __ldg(A.order + rl);
    const int s = slot_of_offset(T, y - x);
    uint32_t rz;
    if (d1_pair_lookup(A, T, x, s, rz) < 0) return false;
    k1 = (unsigned long long)rh << 32 | rz;
    k2 = ekey(rl, rz);
    return true;
}

__device__ __forceinline__ bool arena_alloc(const D1Args& A, unsigned long long n, unsigned long long& off) {
    off = atomicAdd(A.arena_top, n);
    if (off + n > A.arena_cap) {
        atomicOr(A.err, 1);
        return false;
    }
    return true;
}

// phase 1: sigma added the column of owner o at edge j (its column stays the sequential
// one iff o still owns j at the end and o's own column is -- see k_d1_taint*)
__device__ __forceinline__ void d1_dep(const D1Args& A, int sig, int o, int j, int seq) {
    if (A.phase != 1 || !A.deps) return;
    const int k = atomicAdd(A.ndeps, 1);
    if (k < A.deps_cap) A.deps[k] = make_int4(sig, o, j, seq);
}

// phase 1: sigma's column was stored after `seq` owner columns: a restart point for the
// generator pass if its later additions turn out not to be the sequential algorithm's
__device__ __forceinline__ void d1_snap(const D1Args& A, int sig, int seq, long long off, int len) {
    if (A.phase != 1 || !A.snaps) return;
    const int k = atomicAdd(A.nsnaps, 1);
    if (k < A.snaps_cap) {
        D1Snap r;
        r.sig = sig;
        r.seq = seq;
        r.len = len;
        r.pad = 0;
        r.off = off;
        A.snaps[k] = r;
    }
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
__device__ __forceinline__ uint8_t d1_propagate(const D1Args& A, const D1Tab& S, int sig, Heap<P>& H, Room room,
                                                unsigned long long& tau_out, int& j_out, int& nadds) {
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
            if (A.st_steps) A.st_steps[sig]++;
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
            d1_dep(A, sig, o, j, nadds++);
            if (A.st_adds) {
                A.st_adds[sig]++;
                A.st_pushed[sig] += len - 1;
            }
            continue;
        }
        tau_out = tau;
        j_out = j;
        return A.phase == 1 ? D1_STOP : D1_WAIT;
    }
}

template <typename P>
__device__ __forceinline__ void d1_finish(const D1Args& A, int sig, Heap<P>& H, uint8_t st, unsigned long long tau, int j,
                                          int nadds) {
    if (st == D1_STOP || st == D1_WAIT || st == D1_DONE) {
        if (!d1_store(A, sig, H, tau)) {
            A.status[sig] = D1_RETRY;
            return;
        }
        A.nadd[sig] = nadds;
        d1_snap(A, sig, nadds, A.col_off[sig], A.col_len[sig]);
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
    __shared__ D1Tab S;
    for (int i = threadIdx.x; i < (int)(sizeof(D1Tab) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&S)[i] = reinterpret_cast<const uint32_t*>(A.tab)[i];
    __syncthreads();
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
        int nadds = A.nadd[sig];
        const uint8_t st = d1_propagate(A, S, sig, H, [&](int m) { return heap_room(A, H, m); }, tau, j, nadds);
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
            A.nadd[sig] = nadds;
            A.status[sig] = D1_BIG;
            A.big[atomicAdd(A.nbig, 1)] = sig;
            continue;
        }
        d1_finish(A, sig, H, st, tau, j, nadds);
    }
}

// ---------------------------------------------------------------- large sigmas
// One CTA of kBigT threads per deferred sigma (k_d1_bigc).  The boundary is split in two
// (an LSM pair): A, a sorted, duplicate-free array of keys in the arena (read through a
// prefetched ring of resolved entries), and P, a binary max-heap of 16-byte entries
// (key + both vertices, so a regular step needs no order[] lookups) in shared memory.
// Thread 0 runs the propagation serially: the maximum is the larger of A's head and P's
// top (equal keys cancel, mod 2); the pushed edges of regular steps go to P.  The whole
// CTA merges: P into A when P fills up (bitonic sort + parity dedup + merge), a long
// owner column straight into A, and the final column at a stop.  Merges cancel equal
// keys; their output is always sorted and duplicate-free, so every stored column is.

constexpr int kBigT = 128;
constexpr int kBigP = 2048;     // P capacity (entries)
constexpr int kBigRing = kBigT; // resolved A entries
constexpr int kBigAddSmall = 1024;

struct E16 {
    unsigned long long key;
    int32_t hi;    // the edge's higher vertex (in K)
    int32_t slot;  // the lower vertex's slot around hi
};

// one sorted, duplicate-free level of the large-2-saddle boundary (A: the big base, B:
// the medium one that absorbs additions and is merged into A when it grows past half A)
struct Level {
    long long off;           // the level's array in the arena
    int len, head;           // entries [head, len) are live
    int rbase, rcnt;         // ring = resolved entries [rbase, rbase + rcnt)
    long long buf[2];        // this run's reusable buffers
    int cap[2], cur;         // their capacities; which buffer holds the level (-1: the stored column)
};

struct BigSmem {
    E16 P[kBigP];                     // 32 KB
    unsigned long long S[2 * kBigP];  // 32 KB: sort buffer / staging (E16 x 2048)
    E16 ring[2][kBigRing];            // resolved heads of A and B
    int cnt[kBigT + 1];
    Level lv[2];
    // control block (written by thread 0 before a barrier)
    int action, arg, pn, j, m, status, ok, nadds;
    long long oo;                     // owner column offset
    long long o_out;                  // merge output of the current merge
    long long tbuf;                   // merge scratch (reused)
    int tcap;
    E16 tau;
};

enum : int { BA_REFILL = 1, BA_MERGEP = 2, BA_ADDS = 3, BA_ADDB = 4, BA_STOP = 5, BA_ABORT = 6 };

__device__ __forceinline__ E16 d1_resolve_key(const D1Args& A, const D1Tab& T, unsigned long long key) {
    E16 e;
    e.key = key;
    e.hi = __ldg(A.order + (key >> 32));
    e.slot = slot_of_offset(T, __ldg(A.order + (uint32_t)key) - e.hi);
    return e;
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// 4-ary max-heap over E16 entries in shared memory (half the levels of a binary heap:
// the serial thread's pops are its largest cost)
__device__ __forceinline__ void sh_push(E16* P, int& n, const E16& e) {
    int i = n++;
    while (i > 0) {
        const int p = (i - 1) >> 2;
        if (P[p].key >= e.key) break;
        P[i] = P[p];
        i = p;
    }
    P[i] = e;
}
__device__ __forceinline__ E16 sh_pop(E16* P, int& n) {
    const E16 top = P[0];
    const E16 k = P[--n];
    int i = 0;
    while (true) {
        const int c = 4 * i + 1;
        if (c >= n) break;
        int b = c;
        unsigned long long bk = P[c].key;
        if (c + 3 < n) {
            const unsigned long long k1 = P[c + 1].key, k2 = P[c + 2].key, k3 = P[c + 3].key;
            const int b01 = k1 > bk ? c + 1 : c;
            const unsigned long long m01 = k1 > bk ? k1 : bk;
            const int b23 = k3 > k2 ? c + 3 : c + 2;
            const unsigned long long m23 = k3 > k2 ? k3 : k2;
            b = m23 > m01 ? b23 : b01;
            bk = m23 > m01 ? m23 : m01;
        } else {
            for (int q = c + 1; q < n; q++) {
                const unsigned long long kq = P[q].key;
                if (kq > bk) { bk = kq; b = q; }
            }
        }
        if (bk <= k.key) break;
        P[i] = P[b];
        i = b;
    }
    if (n > 0) P[i] = k;
    return top;
}

// A few of the largest new entries in registers (sorted, descending): the serial thread
// pops and pushes them without shared-memory latency; the heap P takes the rest.
constexpr int kHot = 8;
struct Hot {
    E16 e[kHot];
    int n = 0;
};
__device__ __forceinline__ void hot_pop_front(Hot& H) {
#pragma unroll
    for (int i = 0; i < kHot - 1; i++) H.e[i] = H.e[i + 1];
    H.n--;
}
// insert x (an equal key already present cancels, mod 2); the smallest entry of a full
// buffer (or x itself) goes to P
__device__ __forceinline__ void hot_insert(Hot& H, const E16& x, E16* P, int& pn) {
    int eq = -1;
#pragma unroll
    for (int i = 0; i < kHot; i++)
        if (i < H.n && H.e[i].key == x.key) eq = i;
    if (eq >= 0) {
#pragma unroll
        for (int i = 0; i < kHot - 1; i++)
            if (i >= eq) H.e[i] = H.e[i + 1];
        H.n--;
        return;
    }
    if (H.n == kHot) {
        if (x.key < H.e[kHot - 1].key) {
            sh_push(P, pn, x);
            return;
        }
        sh_push(P, pn, H.e[kHot - 1]);
        H.n--;
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < kHot; i++) q += (i < H.n && H.e[i].key > x.key) ? 1 : 0;
#pragma unroll
    for (int i = kHot - 1; i > 0; i--)
        if (i > q && i <= H.n) H.e[i] = H.e[i - 1];
#pragma unroll
    for (int i = 0; i < kHot; i++)
        if (i == q) H.e[i] = x;
    H.n++;
}
__device__ __forceinline__ void hot_flush(Hot& H, E16* P, int& pn) {
#pragma unroll
    for (int i = 0; i < kHot; i++)
        if (i < H.n) sh_push(P, pn, H.e[i]);
    H.n = 0;
}

// regular step on an entry with known vertices (d1_regular without the order[] loads);
// the gradient word of the new entry k2's higher vertex is prefetched (k1's is x's)
__device__ __forceinline__ bool d1_regular16(const D1Args& A, const D1Tab& T, const E16& t, E16& k1, E16& k2) {
    const int32_t x = t.hi;
    const int s = t.slot;
    uint32_t rz;
    const int u = d1_pair_lookup(A, T, x, s, rz);
    if (u < 0) return false;
    const uint32_t rh = (uint32_t)(t.key >> 32), rl = (uint32_t)t.key;
    k1.key = (unsigned long long)rh << 32 | rz;
    k1.hi = x;
    k1.slot = u;
    if (rl > rz) {  // (y, z), y = x + lin[s] higher: z = y + (lin[u] - lin[s])
        k2.key = (unsigned long long)rl << 32 | rz;
        k2.hi = x + T.lin[s];
        k2.slot = T.sdiff[s][u];
    } else {        // (z, y): y = z + (lin[s] - lin[u])
        k2.key = (unsigned long long)rz << 32 | rl;
        k2.hi = x + T.lin[u];
        k2.slot = T.sdiff[u][s];
    }
    prefetch_l1(reinterpret_cast<const ulonglong2*>(A.g.grad) + k2.hi);
    return true;
}

// CTA exclusive scan of one int per thread (kBigT threads); returns the prefix, *total
__device__ __forceinline__ int cta_scan(BigSmem& sm, int v, int* total) {
    const int t = threadIdx.x;
    sm.cnt[t] = v;
    __syncthreads();
    if (t == 0) {
        int acc = 0;
        for (int i = 0; i < kBigT; i++) {
            const int c = sm.cnt[i];
            sm.cnt[i] = acc;
            acc += c;
        }
        sm.cnt[kBigT] = acc;
    }
    __syncthreads();
    const int r = sm.cnt[t];
    *total = sm.cnt[kBigT];
    __syncthreads();
    return r;
}

// merge of two sorted (descending), duplicate-free key arrays with mod-2 cancellation:
// out[0 .. result) = X xor Y, sorted descending.  tmp: scratch of nx + ny keys.
// Merge path: every thread takes one diagonal range; an equal pair straddling a
// boundary is kept on the left side so that it cancels.
template <bool YCG>
__device__ int cta_merge(BigSmem& sm, const unsigned long long* X, int nx, const unsigned long long* Yp, int ny,
                         unsigned long long* out, unsigned long long* tmp) {
    const int t = threadIdx.x;
    // Y may be a column another SM wrote during this kernel (phase 2): read it from L2
    auto Yld = [&](int i) { return YCG ? __ldcg(Yp + i) : Yp[i]; };
    const int total = nx + ny;
    const int per = (total + kBigT - 1) / kBigT;
    auto corank = [&](int k) {
        int lo = max(0, k - ny), hi = min(k, nx);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const int jj = k - mid;
            if (jj > 0 && X[mid] >= Yld(jj - 1)) lo = mid + 1;
            else hi = mid;
        }
        int i = lo, jj = k - lo;
        if (i > 0 && jj < ny && X[i - 1] == Yld(jj)) jj++;
        return make_int2(i, jj);
    };
    const int d0 = min(t * per, total), d1 = min(d0 + per, total);
    const int2 s0 = corank(d0), s1 = d1 == total ? make_int2(nx, ny) : corank(d1);
    int a = s0.x, b = s0.y;
    const int base = s0.x + s0.y;
    int c = 0;
    while (a < s1.x || b < s1.y) {
        if (b >= s1.y) tmp[base + c++] = X[a++];
        else if (a >= s1.x) tmp[base + c++] = Yld(b++);
        else {
            const unsigned long long x = X[a], y = Yld(b);
            if (x > y) { tmp[base + c++] = x; a++; }
            else if (y > x) { tmp[base + c++] = y; b++; }
            else { a++; b++; }
        }
    }
    int n;
    const int dst = cta_scan(sm, c, &n);
    for (int k = 0; k < c; k++) out[dst + k] = tmp[base + k];
    __syncthreads();
    return n;
}

// P's keys -> sm.S sorted descending with the mod-2 duplicates removed; returns the count
__device__ int cta_sort_pending(BigSmem& sm, int pn) {
    const int t = threadIdx.x;
    int p2 = 1;
    while (p2 < pn) p2 <<= 1;
    for (int i = t; i < p2; i += kBigT) sm.S[i] = i < pn ? sm.P[i].key : 0ull;
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = t; i < p2; i += kBigT) {
                const int l = i ^ jj;
                if (l > i) {
                    const unsigned long long x = sm.S[i], y = sm.S[l];
                    const bool desc = (i & k) == 0;
                    if (desc ? x < y : x > y) { sm.S[i] = y; sm.S[l] = x; }
                }
            }
            __syncthreads();
        }
    // keep the last element of each run of equal keys iff the run length is odd
    const int per = (pn + kBigT - 1) / kBigT;
    const int i0 = min(t * per, pn), i1 = min(i0 + per, pn);
    int c = 0;
    for (int i = i0; i < i1; i++) {
        const unsigned long long k = sm.S[i];
        if (i + 1 < pn && sm.S[i + 1] == k) continue;
        int r = 1;
        while (i - r >= 0 && sm.S[i - r] == k) r++;
        if (r & 1) c++;
    }
    int n;
    const int dst = cta_scan(sm, c, &n);
    // compact into the upper half of P's storage (viewed as keys), then back into S
    unsigned long long* Q = reinterpret_cast<unsigned long long*>(sm.P);
    int w = dst;
    for (int i = i0; i < i1; i++) {
        const unsigned long long k = sm.S[i];
        if (i + 1 < pn && sm.S[i + 1] == k) continue;
        int r = 1;
        while (i - r >= 0 && sm.S[i - r] == k) r++;
        if (r & 1) Q[w++] = k;
    }
    __syncthreads();
    for (int i = t; i < n; i += kBigT) sm.S[i] = Q[i];
    __syncthreads();
    return n;
}

// thread 0: an arena block for the merge of nx + ny keys into level l's other buffer
// (lead = 1: a fresh block with a leading slot for tau -- the stored column at a stop)
__device__ __forceinline__ bool big_alloc(const D1Args& A, BigSmem& sm, int l, int need, int lead) {
    unsigned long long o;
    if (sm.tcap < need) {
        const int cap = max(2 * sm.tcap, need);
        if (!arena_alloc(A, (unsigned long long)cap, o)) return false;
        sm.tbuf = (long long)o;
        sm.tcap = cap;
    }
    if (lead) {
        if (!arena_alloc(A, (unsigned long long)(need + 1), o)) return false;
        sm.o_out = (long long)o;
        return true;
    }
    Level& L = sm.lv[l];
    const int other = L.cur == 0 ? 1 : 0;
    if (L.cap[other] < need) {
        const int cap = max(2 * L.cap[other], need);
        if (!arena_alloc(A, (unsigned long long)cap, o)) return false;
        L.buf[other] = (long long)o;
        L.cap[other] = cap;
    }
    sm.o_out = L.buf[other];
    return true;
}

// the CTA merges Y (ny sorted keys, smem or global) into level l; with into_out, the
// result goes to the fresh block sm.o_out + 1 (the stored column) instead.  Returns false
// if the arena is full (the caller retries the 2-saddle next round).
template <bool YCG>
__device__ bool big_merge(const D1Args& A, BigSmem& sm, int l, const unsigned long long* Y, int ny, bool into_out) {
    const int t = threadIdx.x;
    Level& L = sm.lv[l];
    const int nx = L.len - L.head;
    const unsigned long long* X = A.arena + L.off + L.head;
    __syncthreads();
    if (t == 0) sm.ok = big_alloc(A, sm, l, nx + ny, into_out ? 1 : 0) ? 1 : 0;
    __syncthreads();
    if (!sm.ok) return false;
    const long long outoff = sm.o_out + (into_out ? 1 : 0);
    int n;
    if (ny > 0) {
        n = cta_merge<YCG>(sm, X, nx, Y, ny, A.arena + outoff, A.arena + sm.tbuf);
    } else {
        for (int k = t; k < nx; k += kBigT) A.arena[outoff + k] = X[k];
        n = nx;
        __syncthreads();
    }
    if (t == 0) {
        if (into_out) {
            sm.m = n;  // the merged length (the stop writes the column)
        } else {
            L.cur = L.cur == 0 ? 1 : 0;
            L.off = outoff;
            L.len = n;
            L.head = 0;
            L.rbase = 0;
            L.rcnt = 0;
        }
    }
    __syncthreads();
    return true;
}

// B into A once B holds more than half of A (each key is merged O(log) times)
__device__ bool big_settle(const D1Args& A, BigSmem& sm) {
    const int nb = sm.lv[1].len - sm.lv[1].head, na = sm.lv[0].len - sm.lv[0].head;
    if (nb == 0 || 2 * nb <= na) return true;
    if (!big_merge<false>(A, sm, 0, A.arena + sm.lv[1].off + sm.lv[1].head, nb, false)) return false;
    if (threadIdx.x == 0) {
        sm.lv[1].len = 0;
        sm.lv[1].head = 0;
        sm.lv[1].rbase = 0;
        sm.lv[1].rcnt = 0;
    }
    __syncthreads();
    return true;
}

__global__ void __launch_bounds__(kBigT) k_d1_bigc(D1Args A) {
    extern __shared__ __align__(16) unsigned char d1_smem[];
    BigSmem& sm = *reinterpret_cast<BigSmem*>(d1_smem);
    __shared__ D1Tab S;
    for (int i = threadIdx.x; i < (int)(sizeof(D1Tab) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&S)[i] = reinterpret_cast<const uint32_t*>(A.tab)[i];
    __syncthreads();
    const int t = threadIdx.x;
    const int nb = *A.nbig;
    for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
        const int sig = A.big[bi];
        if (t == 0) {
            const long long off = A.col_off[sig];
            const int len0 = A.col_len[sig];
            sm.pn = 0;
            sm.tcap = 0;
            for (int l = 0; l < 2; l++) {
                Level& L = sm.lv[l];
                L.off = 0;
                L.len = L.head = L.rbase = L.rcnt = 0;
                L.cap[0] = L.cap[1] = 0;
                L.cur = -1;
            }
            sm.nadds = A.nadd[sig];
            if (len0 >= 0) {  // [tau, sorted rest]: A = rest (in place), P = {tau}
                sm.lv[0].off = off + 1;
                sm.lv[0].len = len0 - 1;
                sh_push(sm.P, sm.pn, d1_resolve_key(A, S, A.arena[off]));
            } else {          // a bag from the local path: everything into P
                for (int k = 0; k < -len0; k++) sh_push(sm.P, sm.pn, d1_resolve_key(A, S, A.arena[off + k]));
            }
        }
        __syncthreads();
        Hot hot;  // thread 0's register buffer (empty at every CTA action that reads P)
        long long pc_t = clock64(), pc_cyc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int pc_last = 0, pc_n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        while (true) {
            if (t == 0 && A.prof) {
                const long long now = clock64();
                pc_cyc[pc_last] += now - pc_t;
                pc_t = now;
            }
            if (t == 0) {
                // serial propagation until the CTA is needed
                int pn = sm.pn;
                int h0 = sm.lv[0].head, h1 = sm.lv[1].head;
                const int l0 = sm.lv[0].len, l1 = sm.lv[1].len;
                const int rb0 = sm.lv[0].rbase, rc0 = sm.lv[0].rcnt, rb1 = sm.lv[1].rbase, rc1 = sm.lv[1].rcnt;
                int action = 0, arg = 0;
                while (true) {
                    if (pn > kBigP - 3 - kHot) {
                        hot_flush(hot, sm.P, pn);
                        action = BA_MERGEP;
                        break;
                    }
                    if (h0 < l0 && h0 >= rb0 + rc0) { action = BA_REFILL; arg = 0; break; }
                    if (h1 < l1 && h1 >= rb1 + rc1) { action = BA_REFILL; arg = 1; break; }
                    // the maximum of the levels' heads, P's top and the register buffer's
                    // first; equal copies cancel in pairs (mod 2)
                    const unsigned long long a0 = h0 < l0 ? sm.ring[0][h0 - rb0].key : 0ull;
                    const unsigned long long a1 = h1 < l1 ? sm.ring[1][h1 - rb1].key : 0ull;
                    const unsigned long long p = pn ? sm.P[0].key : 0ull;
                    const unsigned long long h = hot.n ? hot.e[0].key : 0ull;
                    const unsigned long long mx = max(max(h, p), max(a0, a1));
                    if (!mx) {
                        d1_fail(A, 2, sig, 0ull, -1, -1);
                        action = BA_ABORT;
                        break;
                    }
                    E16 tv;
                    int cnt = 0;
                    if (h == mx) {
                        tv = hot.e[0];
                        hot_pop_front(hot);
                        cnt++;
                    }
                    if (a0 == mx) {
                        tv = sm.ring[0][h0 - rb0];
                        h0++;
                        cnt++;
                    }
                    if (a1 == mx) {
                        tv = sm.ring[1][h1 - rb1];
                        h1++;
                        cnt++;
                    }
                    if (p == mx) {
                        tv = sh_pop(sm.P, pn);
                        cnt++;
                        while (pn && sm.P[0].key == mx) {
                            sh_pop(sm.P, pn);
                            cnt++;
                        }
                    }
                    if (!(cnt & 1)) continue;
                    E16 k1, k2;
                    if (d1_regular16(A, S, tv, k1, k2)) {
                        hot_insert(hot, k1, sm.P, pn);
                        hot_insert(hot, k2, sm.P, pn);
                        if (A.st_steps) A.st_steps[sig]++;
                        continue;
                    }
                    const int j = d1_lookup(A, tv.key);
                    if (j < 0) {
                        d1_fail(A, 4, sig, tv.key, j, -1);
                        action = BA_ABORT;
                        break;
                    }
                    const int o = A.owner[j];
                    bool add;
                    uint8_t st = A.phase == 1 ? D1_STOP : D1_WAIT;
                    if (A.phase == 1) {
                        add = o >= 0 && o < sig;
                    } else if (o == sig) {
                        add = false;
                        st = D1_DONE;
                    } else {
                        if (o < 0 || o > sig) {
                            d1_fail(A, 8, sig, tv.key, j, o);
                            action = BA_ABORT;
                            break;
                        }
                        add = *(volatile const int32_t*)(A.done + o) != 0;
                        if (add) __threadfence();
                    }
                    if (add) {
                        d1_dep(A, sig, o, j, sm.nadds++);
                        sm.oo = *(volatile const long long*)(A.col_off + o);
                        sm.m = *(volatile const int32_t*)(A.col_len + o);
                        if (A.st_adds) {
                            A.st_adds[sig]++;
                            A.st_pushed[sig] += sm.m - 1;
                        }
                        // a short column goes to P (serial pushes), a longer one is merged
                        // into level B by the CTA
                        action = (sm.m - 1 <= A.adds && pn + sm.m <= kBigP - 3 - kHot) ? BA_ADDS : BA_ADDB;
                        break;
                    }
                    hot_flush(hot, sm.P, pn);
                    sm.tau = tv;
                    sm.j = j;
                    sm.status = st;
                    action = BA_STOP;
                    break;
                }
                sm.pn = pn;
                sm.lv[0].head = h0;
                sm.lv[1].head = h1;
                sm.action = action;
                sm.arg = arg;
                if (A.prof) {
                    const long long now = clock64();
                    pc_cyc[0] += now - pc_t;  // serial propagation
                    pc_t = now;
                    pc_last = action;
                    pc_n[action]++;
                }
            }
            __syncthreads();
            const int action = sm.action;
            if (action == BA_ABORT) {
                if (t == 0) A.status[sig] = D1_ERR;
                __syncthreads();
                break;
            }
            if (action == BA_REFILL) {
                const int l = sm.arg;
                const int head = sm.lv[l].head, len = sm.lv[l].len;
                const int n = min(kBigRing, len - head);
                if (t < n) {
                    sm.ring[l][t] = d1_resolve_key(A, S, A.arena[sm.lv[l].off + head + t]);
                    prefetch_l1(reinterpret_cast<const ulonglong2*>(A.g.grad) + sm.ring[l][t].hi);
                }
                __syncthreads();
                if (t == 0) {
                    sm.lv[l].rbase = head;
                    sm.lv[l].rcnt = n;
                }
                __syncthreads();
                continue;
            }
            if (action == BA_ADDS) {
                // stage the owner column's entries (minus its tau) resolved, then push
                const int m1 = sm.m - 1;
                E16* stage = reinterpret_cast<E16*>(sm.S);
                for (int k = t; k < m1; k += kBigT) stage[k] = d1_resolve_key(A, S, __ldcg(A.arena + sm.oo + 1 + k));
                __syncthreads();
                if (t == 0) {
                    int pn = sm.pn;
                    for (int k = 0; k < m1; k++) sh_push(sm.P, pn, stage[k]);
                    sm.pn = pn;
                }
                __syncthreads();
                continue;
            }
            bool ok = true;
            if (action == BA_ADDB) {
                // the owner column (minus its tau) into B; written in an earlier kernel or
                // fenced by its done flag (phase 2: read from L2)
                const unsigned long long* Y = A.arena + sm.oo + 1;
                const int ny = sm.m - 1;
                ok = A.phase == 2 ? big_merge<true>(A, sm, 1, Y, ny, false) : big_merge<false>(A, sm, 1, Y, ny, false);
                ok = ok && big_settle(A, sm);
            } else {  // MERGEP or STOP: the pending heap (sorted, mod-2 deduplicated) into B
                if (sm.pn > 0) {
                    const int ny = cta_sort_pending(sm, sm.pn);
                    ok = big_merge<false>(A, sm, 1, sm.S, ny, false);
                    if (ok && t == 0) sm.pn = 0;
                    __syncthreads();
                }
                if (ok && action == BA_MERGEP) ok = big_settle(A, sm);
            }
            if (ok && action == BA_STOP) {
                // the stored column: [tau, A merged with B]
                const int nb1 = sm.lv[1].len - sm.lv[1].head;
                ok = big_merge<false>(A, sm, 0, A.arena + sm.lv[1].off + sm.lv[1].head, nb1, true);
                if (ok && t == 0) {
                    const long long outoff = sm.o_out;
                    A.arena[outoff] = sm.tau.key;
                    A.col_off[sig] = outoff;
                    A.col_len[sig] = sm.m + 1;
                    A.nadd[sig] = sm.nadds;
                    d1_snap(A, sig, sm.nadds, outoff, sm.m + 1);
                    A.stop[sig] = sm.j;
                    const uint8_t st = (uint8_t)sm.status;
                    if (st == D1_STOP) {
                        atomicMin(A.claim + sm.j, A.tag | (unsigned)sig);
                    } else if (st == D1_DONE) {
                        __threadfence();
                        *(volatile int32_t*)(A.done + sig) = 1;
                    }
                    A.status[sig] = st;
                }
            }
            if (!ok) {
                if (t == 0) A.status[sig] = D1_RETRY;
                __syncthreads();
                break;
            }
            __syncthreads();
            if (action == BA_STOP) break;
        }
        if (t == 0 && A.prof) {
            pc_cyc[pc_last] += clock64() - pc_t;
            for (int q = 0; q < 8; q++) {
                atomicAdd(A.prof + q, (unsigned long long)pc_cyc[q]);
                atomicAdd(A.prof + 8 + q, (unsigned long long)pc_n[q]);
            }
        }
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
                          int32_t* done, int32_t* nadd) {
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
    nadd[i] = 0;
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

__global__ void k_fill_u32(uint32_t* a, int64_t n, uint32_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

// taint (phase 1 -> phase 2): sigma's phase-1 trajectory is the sequential algorithm's up
// to its first addition of a column that is not the owner's final one -- the owner lost
// that edge later, or its own final column is tainted.  first_bad[sigma] = the number of
// that addition (0xffffffff: none, the phase-1 column is the generator).
__global__ void k_d1_taint_direct(const int4* __restrict__ deps, int64_t nd, const int32_t* __restrict__ owner,
                                  uint32_t* first_bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int4 d = deps[i];
    if (owner[d.z] != d.y) atomicMin(first_bad + d.x, (uint32_t)d.w);
}
__global__ void k_d1_taint_prop(const int4* __restrict__ deps, int64_t nd, uint32_t* first_bad, int* changed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd) return;
    const int4 d = deps[i];
    if (first_bad[d.y] != 0xffffffffu && first_bad[d.x] > (uint32_t)d.w) {
        if (atomicMin(first_bad + d.x, (uint32_t)d.w) > (uint32_t)d.w) *changed = 1;
    }
}
__global__ void k_d1_taint_flags(const uint32_t* __restrict__ first_bad, int64_t n, uint32_t* taint) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) taint[i] = first_bad[i] != 0xffffffffu ? 1u : 0u;
}
// the latest snapshot of a tainted sigma taken before its first bad addition
__global__ void k_d1_snap_pick(const D1Snap* __restrict__ snaps, int64_t ns, const uint32_t* __restrict__ first_bad,
                               unsigned long long* best) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const D1Snap r = snaps[i];
    const uint32_t fb = first_bad[r.sig];
    if (fb != 0xffffffffu && (uint32_t)r.seq <= fb)
        atomicMax(best + r.sig, ((unsigned long long)(r.seq + 1) << 32) | (unsigned long long)i);
}

// phase 2 starts with the tainted sigmas only: their boundaries at arena[base + 3 k]
__global__ void k_d1_init_tainted(Geo3 g, const int32_t* __restrict__ rank, const int64_t* __restrict__ sig_ids,
                                  int64_t nsig, const uint32_t* __restrict__ taint, const uint32_t* __restrict__ pos,
                                  unsigned long long base, unsigned long long* arena, long long* col_off,
                                  int32_t* col_len, int32_t* active, int32_t* done,
                                  const unsigned long long* __restrict__ best, const D1Snap* __restrict__ snaps) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsig) return;
    if (!taint[i]) {
        done[i] = 1;
        return;
    }
    done[i] = 0;
    active[pos[i]] = (int32_t)i;
    if (best && best[i]) {  // restart from the snapshot
        const D1Snap r = snaps[best[i] & 0xffffffffull];
        col_off[i] = r.off;
        col_len[i] = r.len;
        return;
    }
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
    const unsigned long long o = base + 3ull * pos[i];
    for (int q = 0; q < 3; q++) arena[o + q] = e[q];
    col_off[i] = (long long)o;
    col_len[i] = 3;
}

// arena compaction: the live columns (one per sigma) copied to new offsets; one warp each
__global__ void k_d1_abs_len(const int32_t* __restrict__ col_len, int64_t nsig, uint32_t* len) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nsig) len[i] = (uint32_t)abs(col_len[i]);
}
__global__ void k_d1_compact(long long* col_off, const int32_t* __restrict__ col_len, const uint32_t* __restrict__ pos,
                             int64_t nsig, const unsigned long long* __restrict__ src, unsigned long long* dst) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nsig) return;
    const int len = abs(col_len[i]);
    const long long off = col_off[i];
    const long long to = pos[i];
    for (int k = lane; k < len; k += 32) dst[to + k] = src[off + k];
    __syncwarp();
    if (lane == 0) col_off[i] = to;
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
