// diag.cuh -- extremum diagrams D0 and D_{d-1} (Sec. 5) on sm_100a.
//
// D0 (Sec. 5.1, PAPER.md 2481-2685):
//   (a)+(b) k_d0_arcs: for every critical edge (in emission order), follow the two
//           descending v-paths (vertex -> paired edge -> other vertex) from its
//           vertices to minima.  The paired edge of a vertex is its steepest-descent
//           edge, so this is root finding in the steepest-descent forest.  Arc =
//           (node of minimum a, node of minimum b); nodes = emission positions in C_0,
//           arc keys = positions in the sorted C_1, node ages = positions in sorted C_0.
//   (c)+(d) union-find over the arcs in increasing lexicographic order with the
//           Elder rule, done as parallel contraction rounds in one cooperative kernel
//           (DESIGN.md "Union-find"), finished by a sequential tail in the same kernel.
// D_{d-1} (Sec. 5.2, PAPER.md 2690-2825): the same on the dual gradient: stable sets
//   of the critical (d-1)-simplices, followed through the d-simplices (d-simplex ->
//   its paired facet -> the other cofacet of that facet), a virtual maximum on the
//   boundary (exact mode), union-find in decreasing order, the virtual maximum oldest.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "star.cuh"
#include "tet5.cuh"

namespace dms {

struct Geo3 {
    int ndim;
    int32_t Lx, Ly, Lz;
    int64_t N;
    int64_t ncell[4];
    const float* f;
    const void* grad;
    const StarTab* tab;
    const ChaseTab* ctab;  // dual-chase transitions
    const unsigned long long* cw;  // 3D, optional: chase word per vertex = tet codes | lower mask << 48
    const uint32_t* cw2;           // 2D, optional: chase word = triangle codes | lower mask << 12
    const uint8_t* vc;             // 2D / 3D, optional: vertex codes (the D0 descent), 1 byte each
    const T5Tab* t5;               // the five-tetrahedra complex (tet5.cuh), else null
};

__device__ __forceinline__ int64_t lin_mask(const Geo3& g, int m) {
    return (int64_t)(m & 1) + (int64_t)g.Lx * ((m >> 1) & 1) + (int64_t)g.Lx * g.Ly * ((m >> 2) & 1);
}

__device__ __forceinline__ bool kless_v(const Geo3& g, int64_t u, int64_t v) {
    const uint32_t ou = ord_of(__ldg(g.f + u)), ov = ord_of(__ldg(g.f + v));
    return k_less(ou, u, ov, v);
}

// vertex code of v (edge slot paired with v), -1 if v is a minimum
__device__ __forceinline__ int vcode_of(const Geo3& g, int64_t v) {
    if (g.vc) {  // compact copy: 8-16x denser than the gradient words
        const int c = (int)__ldg(g.vc + v);
        return c == (g.ndim == 3 ? 15 : 7) ? -1 : c;
    }
    if (g.ndim == 3) {
        int c = (int)((__ldg(reinterpret_cast<const uint32_t*>(g.grad) + 4 * v + 1) >> 24) & 15u);
        return c == 15 ? -1 : c;
    } else if (g.ndim == 2) {
        int c = (int)(__ldg(reinterpret_cast<const uint16_t*>(g.grad) + v) & 7u);
        return c == 7 ? -1 : c;
    }
    int c = (int)__ldg(reinterpret_cast<const uint8_t*>(g.grad) + v);
    return c == 3 ? -1 : c;
}

__device__ __forceinline__ void coords_of(const Geo3& g, int64_t v, int& x, int& y, int& z) {
    const int vv = (int)v;
    x = vv % g.Lx;
    const int t = vv / g.Lx;
    y = t % g.Ly;
    z = t / g.Ly;
}

__device__ __forceinline__ bool slot_in(const Geo3& g, const StarTab& S, int x, int y, int z, int s) {
    const int nx = x + S.off[s][0], ny = y + S.off[s][1], nz = z + S.off[s][2];
    return nx >= 0 && nx < g.Lx && ny >= 0 && ny < g.Ly && nz >= 0 && nz < g.Lz;
}

// follow the descending v-path from v to its minimum (Sec. 5.1(a))
// (K decreases along the path, so it has fewer than N steps: the bound only stops a walk over
// a gradient buffer the caller freed or overwrote from spinning on the GPU)
__device__ __forceinline__ int64_t descend(const Geo3& g, const StarTab& S, int64_t v) {
    for (int64_t steps = 0; steps < g.N; steps++) {
        const int c = vcode_of(g, v);
        if (c < 0) return v;
        const int64_t u = v + S.lin[c];
        if (u < 0 || u >= g.N) return v;
        v = u;
    }
    return v;
}

// sort key of a critical cell: x << 12 | G  ->  rank(x) << 12 | G
__global__ void k_rekey(uint64_t* __restrict__ keys, int64_t m, const int32_t* __restrict__ rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        const uint64_t k = keys[i];
        keys[i] = ((uint64_t)(uint32_t)rank[k >> 12] << 12) | (k & 0xfffull);
    }
}

// union-find inputs in emission order, scattered straight from the sort permutations
// (perm: sorted position -> emission index): arc key = processing index (rev: m-1-sorted
// position), node age = sorted position (rev: n - sorted position; the virtual node n
// gets age 0, the oldest)
__global__ void k_uf_keys(const uint32_t* __restrict__ perm, int64_t m, int rev, uint32_t* __restrict__ key) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < m) key[perm[p]] = rev ? (uint32_t)(m - 1 - p) : (uint32_t)p;
}
__global__ void k_uf_ages(const uint32_t* __restrict__ perm, int64_t n, int rev, int32_t* __restrict__ age) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) age[perm[r]] = rev ? (int32_t)(n - r) : (int32_t)r;
    if (rev && r == n) age[n] = 0;
}

// out in processing order: outp[j] = out[perm[rev ? m-1-j : j]]
__global__ void k_permute1(const int32_t* __restrict__ out, const uint32_t* __restrict__ perm, int64_t m, int rev,
                           int32_t* __restrict__ outp) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < m) outp[j] = out[perm[rev ? m - 1 - j : j]];
}

__global__ void k_gather_keys(const int32_t* __restrict__ list, int64_t n, const uint32_t* __restrict__ key,
                              uint32_t* __restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out[j] = key[list[j]];
}

// keys that sort on the rank bits alone (one cell per star): the 32-bit rank of the
// highest vertex (keys are x << 12 | G before the rekey)
__global__ void k_rekey32(const uint64_t* __restrict__ keys, int64_t m, const int32_t* __restrict__ rank,
                          uint32_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = (uint32_t)rank[keys[i] >> 12];
}

// Critical lists with one cell per star (C_0; C_1 in 1D): the sort keys are DISTINCT
// ranks, so a record's lexicographic position is the number of records of lower rank --
// a bitmap over the ranks and a prefix popcount (k_bm_set, k_bm_popc + scan, k_bm_place)
// instead of a radix sort
__global__ void k_bm_set(const uint64_t* __restrict__ keys, int64_t m, const int32_t* __restrict__ rank,
                         uint32_t* __restrict__ r_out, unsigned* __restrict__ bm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t r = (uint32_t)rank[keys[i] >> 12];
    r_out[i] = r;
    atomicOr(bm + (r >> 5), 1u << (r & 31));
}
__global__ void k_bm_popc(const unsigned* __restrict__ bm, int64_t nw, uint32_t* __restrict__ cnt) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w < nw) cnt[w] = (uint32_t)__popc(bm[w]);
}
__global__ void k_bm_place(const uint32_t* __restrict__ r, int64_t m, const unsigned* __restrict__ bm,
                           const uint32_t* __restrict__ pre, uint32_t* __restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t rr = r[i], w = rr >> 5;
    perm[pre[w] + (uint32_t)__popc(bm[w] & ((1u << (rr & 31)) - 1u))] = (uint32_t)i;
}

// Critical lists with several cells per star (C_1..C_d in 2D / 3D): lexicographic order
// = by the star's rank, then by the local key G (PAPER.md 1380-1414).  The present stars
// get consecutive indices from the rank bitmap (k_bm_set with its popcount scan), every
// record an arrival slot inside its star's run (k_ms_count), the runs are laid out by a
// scan of the star counts, and each run (<= 36 cells) is sorted by G by one thread
// (k_ms_fix) -- the result does not depend on the arrival order.
__global__ void k_ms_count(const uint32_t* __restrict__ r, int64_t m, const unsigned* __restrict__ bm,
                           const uint32_t* __restrict__ pre, uint32_t* __restrict__ sidx, uint32_t* __restrict__ scnt,
                           uint32_t* __restrict__ slot) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t rr = r[i], w = rr >> 5;
    const uint32_t s = pre[w] + (uint32_t)__popc(bm[w] & ((1u << (rr & 31)) - 1u));
    sidx[i] = s;
    slot[i] = atomicAdd(scnt + s, 1u);
}
__global__ void k_ms_place(const uint64_t* __restrict__ keys, int64_t m, const uint32_t* __restrict__ sidx,
                           const uint32_t* __restrict__ slot, const uint32_t* __restrict__ sbase,
                           unsigned long long* __restrict__ stage) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    stage[sbase[sidx[i]] + slot[i]] = ((keys[i] & 0xfffull) << 32) | (unsigned long long)i;
}
__global__ void k_ms_fix(const unsigned long long* __restrict__ stage, int64_t nstars, const uint32_t* __restrict__ sbase,
                         const uint32_t* __restrict__ scnt, uint32_t* __restrict__ perm) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nstars) return;
    const uint32_t b = sbase[s], n = scnt[s];
    unsigned long long e[40];
    const uint32_t nn = n < 40 ? n : 40;
    for (uint32_t k = 0; k < nn; k++) {
        const unsigned long long x = stage[b + k];
        uint32_t j = k;
        while (j > 0 && e[j - 1] > x) {
            e[j] = e[j - 1];
            j--;
        }
        e[j] = x;
    }
    for (uint32_t k = 0; k < nn; k++) perm[b + k] = (uint32_t)e[k];
}

__global__ void k_iota(uint32_t* __restrict__ a, int64_t m) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) a[i] = (uint32_t)i;
}

__global__ void k_gather_ids(const int64_t* __restrict__ src, const uint32_t* __restrict__ perm, int64_t m,
                             int64_t* __restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) dst[i] = src[perm[i]];
}

__global__ void k_node_map(const int64_t* __restrict__ ids, int64_t m, int32_t* __restrict__ node_of) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) node_of[ids[i]] = (int32_t)i;
}

__global__ void k_d0_arcs(Geo3 g, const int64_t* __restrict__ c1, int64_t m, const int32_t* __restrict__ node_of0,
                          int32_t* __restrict__ arc_a, int32_t* __restrict__ arc_b) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const StarTab& S = *g.tab;
    const int64_t id = c1[i];
    const int64_t a = id / g.ncell[1];
    const int k = (int)(id % g.ncell[1]);
    const int64_t b = a + lin_mask(g, S.chain[1][k][0]);
    arc_a[i] = node_of0[descend(g, S, a)];
    arc_b[i] = node_of0[descend(g, S, b)];
}

// ---------------------------------------------------------------- dual tracing

// 1D: edges (a, a+1) have id a
__device__ int32_t chase_edge1(const Geo3& g, int64_t c, const int32_t* node_of, int32_t vnode) {
    while (c >= 0) {
        const bool right_hi = kless_v(g, c, c + 1);
        const int64_t x = right_hi ? c + 1 : c;
        const int slot = right_hi ? 0 : 1;  // the edge seen from x: 0 = left, 1 = right
        const int code = vcode_of(g, x);
        if (code != slot) return node_of[c];  // not paired with its highest vertex: critical
        if (slot == 0) c = (x < g.N - 1) ? x : -1;  // x's other (right) edge
        else c = (x > 0) ? x - 1 : -1;              // x's other (left) edge
    }
    return vnode;
}

// neighbour slot s of a star is lower than its centre (ordered values, index tie-break)
__device__ __forceinline__ bool nb_lower(uint32_t on, uint32_t ox, int s, int ne) {
    return on < ox || (on == ox && s < (ne >> 1));
}

__device__ __forceinline__ bool in_grid(const Geo3& g, int x, int y, int z) {
    return x >= 0 && x < g.Lx && y >= 0 && y < g.Ly && z >= 0 && z < g.Lz;
}

// 1D: the arcs of G_{D_{d-1}} for the critical vertices ids[0..m) (the (d-1)-simplices):
// both edges of a critical vertex chase up to a critical edge (a maximum) or VIRTUAL
// (2D / 3D use the work-queue kernel below)
__global__ void k_dtop_arcs(Geo3 g, const int64_t* __restrict__ ids, int64_t m, const int32_t* __restrict__ node_of,
                            int32_t vnode, int32_t* __restrict__ arc_a, int32_t* __restrict__ arc_b) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t id = ids[j];
    arc_a[j] = chase_edge1(g, id > 0 ? id - 1 : -1, node_of, vnode);
    arc_b[j] = chase_edge1(g, id < g.N - 1 ? id : -1, node_of, vnode);
}

// Work-queue dual chases (3D / 2D): a persistent grid; every lane owns one chase (one
// side of one arc) and walks one hop per iteration, carrying (x = highest vertex, slot
// of the current top cell in x's star, ordered f(x), x's gradient word): a hop that stays
// in St^-(x) needs one f load, a hop that climbs loads the new vertex's gradient word.
// A lane whose chase ended takes the next job from a warp-private batch, so long and
// short paths do not leave lanes idle.  Jobs: 2 per critical (d-1)-simplex, ids in
// emission order; results go to out_a / out_b in the same order.
template <int D>
struct ChaseState {
    uint32_t x, ox;
    int T;       // top-cell slot in x's star
    int cx, cy, cz;
    uint64_t w;  // x's gradient word (3D: hi half; 2D: the uint16)
};

// 3D: w = the hi half of the gradient word, tet codes (bits 0-47) | lower mask (bits
// 48-61), so a hop that stays in St^-(x) reads nothing and a climb reads one 8-byte word.
// 2D: the chase word (triangle codes | lower mask << 12) if present, else the uint16.
template <int D>
__device__ __forceinline__ uint64_t load_w(const Geo3& g, uint32_t x) {
    if (D == 3) return __ldg(reinterpret_cast<const unsigned long long*>(g.grad) + 2 * (uint64_t)x + 1);
    if (g.cw2) return __ldg(g.cw2 + x);
    return __ldg(reinterpret_cast<const uint16_t*>(g.grad) + x);
}
template <int D>
__device__ __forceinline__ int top_code(const Geo3& g, uint64_t w, int T) {
    if (D == 3) return (int)((w >> (2 * T)) & 3ull);
    return (int)((w >> ((g.cw2 ? 0 : 3) + 2 * T)) & 3ull);
}
// chase word present: is neighbour slot s in the lower mask of the word's vertex
template <int D>
__device__ __forceinline__ bool has_cw(const Geo3& g) {
    return D == 3 ? true : g.cw2 != nullptr;
}
template <int D>
__device__ __forceinline__ bool cw_lower(uint64_t w, int s) {
    return (w >> ((D == 3 ? 48 : 12) + s)) & 1ull;
}

// one hop; returns -2 to continue, else the end node (a maximum's node or vnode)
template <int D>
__device__ __forceinline__ int32_t chase_step(const Geo3& g, const StarTab& S, ChaseState<D>& c,
                                              const int32_t* node_of, int32_t vnode) {
    constexpr int NE = D == 3 ? 14 : 6;
    const int T = c.T;
    const int code = top_code<D>(g, c.w, T);
    if (code == 0) {  // a critical top cell: a maximum
        int64_t id;
        if (D == 3)
            id = 6 * ((int64_t)c.x + S.q_anc[T][0] + (int64_t)g.Lx * S.q_anc[T][1] + (int64_t)g.Lx * g.Ly * S.q_anc[T][2]) +
                 S.q_k[T];
        else
            id = 2 * ((int64_t)c.x + S.t_anc[T][0] + (int64_t)g.Lx * S.t_anc[T][1]) + S.t_k[T];
        return node_of[id];
    }
    const uint32_t e = D == 3 ? g.ctab->q_next[T][code - 1] : g.ctab->t_next[T][code - 1];
    const int T2 = (int)(e & 255u);
    if (T2 == 255) return vnode;
    const int s2 = (int)((e >> 8) & 255u);
    const int nx = c.cx + S.off[s2][0], ny = c.cy + S.off[s2][1], nz = c.cz + S.off[s2][2];
    if (!in_grid(g, nx, ny, nz)) return vnode;  // s' on the boundary: the virtual maximum
    const uint32_t n2 = c.x + (uint32_t)S.lin[s2];
    bool stay;
    uint32_t on = 0;
    if (has_cw<D>(g)) {
        stay = cw_lower<D>(c.w, s2);  // s2 in x's lower mask
    } else {
        on = ord_of(__ldg(g.f + n2));
        stay = nb_lower(on, c.ox, s2, NE);
    }
    if (stay) {
        c.T = T2;  // the other cofacet of s' is still in St^-(x)
    } else {       // it climbs to n2
        c.T = (int)(e >> 16);
        c.x = n2;
        c.ox = on;
        c.cx = nx; c.cy = ny; c.cz = nz;
        c.w = load_w<D>(g, n2);
    }
    return -2;
}

// start of a job: the critical (d-1)-simplex ids[job >> 1], cofacet side job & 1.
// Returns -2 with c set, or the end node directly.
template <int D>
__device__ __forceinline__ int32_t chase_start(const Geo3& g, const StarTab& S, const int64_t* ids, int job,
                                               ChaseState<D>& c, const int32_t* node_of, int32_t vnode) {
    constexpr int NE = D == 3 ? 14 : 6;
    const int64_t id = ids[job >> 1];
    const int side = job & 1;
    const int64_t a = id / g.ncell[D - 1];
    const int k = (int)(id % g.ncell[D - 1]);
    uint32_t p[3], o[3];
    p[0] = (uint32_t)a;
#pragma unroll
    for (int q = 1; q < D; q++) p[q] = (uint32_t)(a + lin_mask(g, S.chain[D - 1][k][q - 1]));
#pragma unroll
    for (int q = 0; q < D; q++) o[q] = ord_of(__ldg(g.f + p[q]));
    int jx = 0;
#pragma unroll
    for (int q = 1; q < D; q++)
        if (o[jx] < o[q] || (o[jx] == o[q] && p[jx] < p[q])) jx = q;
    const uint32_t x = p[jx], ox = o[jx];
    int cx, cy, cz;
    coords_of(g, x, cx, cy, cz);
    int T, s3;
    if (D == 3) {
        const int t = S.t_slot[k][jx];
        T = S.tri_tet[t][side];
        if (T == 255) return vnode;
        s3 = S.tet_a[T] ^ S.tet_b[T] ^ S.tet_c[T] ^ S.tri_a[t] ^ S.tri_b[t];
    } else {
        const int e = S.e_slot[k][jx];
        T = S.edge_tri[e][side];
        if (T == 255) return vnode;
        s3 = S.tri_a[T] ^ S.tri_b[T] ^ e;
    }
    const int nx = cx + S.off[s3][0], ny = cy + S.off[s3][1], nz = cz + S.off[s3][2];
    if (!in_grid(g, nx, ny, nz)) return vnode;
    const uint32_t n3 = x + (uint32_t)S.lin[s3];
    bool stay;
    uint32_t on = 0;
    uint64_t wx = 0;
    if (has_cw<D>(g)) {
        wx = load_w<D>(g, x);
        stay = cw_lower<D>(wx, s3);
    } else {
        on = ord_of(__ldg(g.f + n3));
        stay = nb_lower(on, ox, s3, NE);
    }
    if (stay) {
        c.x = x; c.ox = ox; c.T = T; c.cx = cx; c.cy = cy; c.cz = cz;
    } else {
        int jj;
        if (D == 3) jj = S.tet_a[T] == s3 ? 0 : (S.tet_b[T] == s3 ? 1 : 2);
        else jj = S.tri_a[T] == s3 ? 0 : 1;
        c.T = D == 3 ? S.q_reslot[T][jj] : S.t_reslot[T][jj];
        c.x = n3; c.ox = on; c.cx = nx; c.cy = ny; c.cz = nz;
    }
    c.w = (has_cw<D>(g) && c.x == x) ? wx : load_w<D>(g, c.x);
    return -2;
}

#ifdef DMS_CHASE_STATS  // diagnostics build only: histogram of hops per chase (log2 bins), [63] = total
__device__ unsigned long long g_chase_hist[64];
#endif
// anchored id of the top cell in slot T of x's star
template <int D>
__device__ __forceinline__ int64_t top_id(const Geo3& g, const StarTab& S, uint32_t x, int T) {
    if (D == 3)
        return 6 * ((int64_t)x + S.q_anc[T][0] + (int64_t)g.Lx * S.q_anc[T][1] + (int64_t)g.Lx * g.Ly * S.q_anc[T][2]) +
               S.q_k[T];
    return 2 * ((int64_t)x + S.t_anc[T][0] + (int64_t)g.Lx * S.t_anc[T][1]) + S.t_k[T];
}

// Ascending dual chases, 2 jobs per critical (d-1)-simplex (one per cofacet side),
// from a work queue.  MEMO: ascending paths merge (they drain into few maxima), so
// the top cell a chase enters when it climbs to a new vertex is stamped (generation
// << 24 | job + 1); a chase that climbs into a cell stamped in this generation by
// another job stops there and records "same end as that job" (res[job] = -3 - other);
// k_resolve_joins follows these links.  Paths are acyclic, so the links are too.  Two
// merged paths climb into the same cells from then on, so stamping at climbs only
// loses at most one climb of sharing; plain loads/stores suffice (a lost race only
// loses a merge: any stamp seen is a cell that job really entered).  Without MEMO the
// ends go to out_a/out_b.
template <int D, bool MEMO>
__global__ void __launch_bounds__(kBlock) k_dtop_arcs_q(Geo3 g, const int64_t* __restrict__ ids, int njobs,
                                                       const int32_t* __restrict__ node_of, int32_t vnode,
                                                       int32_t* __restrict__ out_a, int32_t* __restrict__ out_b,
                                                       int* job_ctr, uint32_t* mark, uint32_t gen,
                                                       int32_t* __restrict__ res) {
    // star tables: shared memory in 2D, L1-cached global in 3D (measured)
    __shared__ StarTab S_sh;
    if (D == 2) {
        const int4* src = reinterpret_cast<const int4*>(g.tab);
        int4* dst = reinterpret_cast<int4*>(&S_sh);
        for (int i = threadIdx.x; i < (int)(sizeof(StarTab) / 16); i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    const StarTab& S = D == 2 ? S_sh : *g.tab;
    const int lane = threadIdx.x & 31;
    ChaseState<D> c;
    c.x = c.ox = 0; c.T = 0; c.cx = c.cy = c.cz = 0; c.w = 0;
    int job = -1;          // current job, -1: none
    bool done = false;     // the queue is exhausted for this lane
    // jobs come from the global queue in warp-private batches (one atomic per batch: a
    // per-refill atomic on the single queue counter serialises across the whole grid)
    constexpr int kBatch = 32;
    int b_next = 0, b_end = 0;  // warp-uniform: the batch's unassigned jobs [b_next, b_end)
    bool exhausted = false;
#ifdef DMS_CHASE_STATS
    int hops = 0;
#endif
    while (true) {
        const bool need = job < 0 && !done;
        const unsigned nm = __ballot_sync(0xffffffffu, need);
        if (nm) {
            if (b_next >= b_end && !exhausted) {
                int base = 0;
                if (lane == 0) base = atomicAdd(job_ctr, kBatch);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base >= njobs) exhausted = true;
                else { b_next = base; b_end = min(base + kBatch, njobs); }
            }
            if (need) {
                const int jb = b_next + __popc(nm & lanemask_lt());
                if (jb < b_end) {
                    const int32_t r = chase_start<D>(g, S, ids, jb, c, node_of, vnode);
                    if (r != -2) {
                        if (MEMO) res[jb] = r;
                        else (jb & 1 ? out_b : out_a)[jb >> 1] = r;
                    } else {
                        job = jb;
                    }
#ifdef DMS_CHASE_STATS
                    hops = 0;
#endif
                } else if (exhausted) {
                    done = true;
                }
            }
            b_next = min(b_end, b_next + __popc(nm));
        }
        if (__all_sync(0xffffffffu, done)) break;
        if (job >= 0) {
            const uint32_t x0 = c.x;
            int32_t r = chase_step<D>(g, S, c, node_of, vnode);
            if (MEMO && r == -2 && c.x != x0) {  // stamps at climbs only (see above)
                uint32_t* mp = mark + top_id<D>(g, S, c.x, c.T);
                const uint32_t old = __ldcg(mp);
                if ((old >> 24) == gen) r = -3 - (int32_t)((old & 0xffffffu) - 1u);  // joins that job
                else __stcg(mp, (gen << 24) | (uint32_t)(job + 1));
            }
#ifdef DMS_CHASE_STATS
            hops++;
#endif
            if (r != -2) {
                if (MEMO) res[job] = r;
                else (job & 1 ? out_b : out_a)[job >> 1] = r;
                job = -1;
#ifdef DMS_CHASE_STATS
                atomicAdd(&g_chase_hist[min(62, 31 - __clz(hops))], 1ull);
                atomicAdd(&g_chase_hist[63], (unsigned long long)hops);
#endif
            }
        }
    }
}

// ends of the memoised chases: follow the join links to a job that reached an end
__global__ void k_resolve_joins(const int32_t* __restrict__ res, int njobs, int32_t* __restrict__ out_a,
                                int32_t* __restrict__ out_b) {
    const int jb = blockIdx.x * blockDim.x + threadIdx.x;
    if (jb >= njobs) return;
    int32_t v = res[jb];
    while (v < 0) v = __ldg(res + (-3 - v));
    (jb & 1 ? out_b : out_a)[jb >> 1] = v;
}

// ---------------------------------------------------------------- union-find
// Arcs and nodes are stored in emission order (spatially coherent, so the rounds hit
// nearby nodes); every arc carries its key (its processing index: ascending lex order for
// D0, descending for D_{d-1}) and every node its age (smaller = older; for D_{d-1} the
// virtual node is the oldest).  Hooks always go younger -> older, so a root is its
// component's oldest node.
// out[i]: -2 undecided, -1 unpaired (cycle), >= 0 the node that dies at arc i.
//
// A round: every live arc finds its two roots; every root
// takes the minimum index m(R) of its live outgoing arcs.  Then for an arc e = m(A)
// joining roots A and B:
//   * e == m(B) (mutual): the younger of A, B dies at e  (both sides are exactly the
//     Kruskal components at e);
//   * else, if A is younger than B: A dies at e  (A is exactly its Kruskal component
//     at e, and B's Kruskal component at e already holds B's oldest node);
//   * else the arc waits.
// Both rules keep the invariant "for every outgoing arc of a component, its Kruskal
// component at that arc's key contains the component's oldest node", so every
// decision equals the sequential elder-rule union-find's.

__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t a) {
    while (true) {
        const int32_t p = parent[a];
        if (p == a) return a;
        const int32_t gp = parent[p];
        if (gp != p) parent[a] = gp;  // path halving (only ever points to an ancestor)
        a = gp;
    }
}

// parent/best for the nodes; out = -2 (undecided) and the first live list of arc
// records {endpoint a, endpoint b, key, arc} for the arcs
__global__ void k_uf_init(int32_t* parent, unsigned long long* best, int64_t n, const int32_t* arc_a,
                          const int32_t* arc_b, const uint32_t* key, int64_t m, int32_t* out, int4* rec) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { parent[i] = (int32_t)i; best[i] = ~0ull; }
    if (i < m) {
        out[i] = -2;
        rec[i] = make_int4(arc_a[i], arc_b[i], (int)key[i], (int)i);
    }
}

// "ignore" boundary mode (PAPER.md 2822-2825, App. A; reading Z7): the arcs of the exact
// mode with every end at the virtual maximum `virt` replaced by the other end -- a
// self-loop, which the union-find leaves unpaired (the half-arc is dropped)
__global__ void k_arcs_drop_virtual(const int32_t* __restrict__ a_in, const int32_t* __restrict__ b_in,
                                    const uint32_t* __restrict__ key_in, int64_t m, int32_t virt,
                                    const int32_t* __restrict__ age_in, int64_t nodes, int32_t* a_out,
                                    int32_t* b_out, uint32_t* key_out, int32_t* age_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        int32_t a = a_in[i], b = b_in[i];
        if (a == virt) a = b;
        if (b == virt) b = a;
        a_out[i] = a;
        b_out[i] = b;
        key_out[i] = key_in[i];
    }
    if (i < nodes) age_out[i] = age_in[i];
}

// the arc records in processing (key) order for the batched rounds: src[j] = the arc
// with key j (perm: processing index -> emission index; rev: D_{d-1}'s descending order)
__global__ void k_uf_src(const int32_t* __restrict__ arc_a, const int32_t* __restrict__ arc_b,
                         const uint32_t* __restrict__ perm, int64_t m, int rev, int4* __restrict__ src) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t i = perm[rev ? m - 1 - j : j];
    src[j] = make_int4(arc_a[i], arc_b[i], (int)j, (int)i);
}

__global__ void k_flag_undecided(const int32_t* out, int64_t m, uint32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flags[i] = out[i] == -2 ? 1u : 0u;
}

__global__ void k_gather_undecided(const int32_t* out, int64_t m, const uint32_t* pos, int32_t* list) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m && out[i] == -2) list[pos[i]] = (int32_t)i;
}

// All union-find rounds in one cooperative launch (grid-wide barriers between the
// phases, no host round trip), then block 0 sorts the (few) undecided arcs and runs
// the sequential elder-rule union-find over them in processing order.
#ifndef DMS_UFTAIL
#define DMS_UFTAIL 128  // sequential-tail threshold (sweep 2048..64: smaller is slightly faster; 1D most)
#endif
constexpr int kUFTail = DMS_UFTAIL;
constexpr int kUFTile = 1024;  // records per CTA tile in pass A (its 16 KB also hold the tail's sort list)
static_assert(kUFTail * 8 <= kUFTile * 16, "the tail's sort list aliases the pass-A staging");

struct UFArgs {
    const uint32_t* key;  // per arc: its processing index (the arc order of the union-find)
    const int32_t* age;   // per node: smaller = older
    int32_t* parent;
    unsigned long long* best;  // per root: round tag << 32 | lightest arc key (see best_tag)
    int32_t* out;
    int4* rec0;   // live arc records {a, b, key, arc}; a, b = roots as of the last find
    int4* rec1;
    int* nlive;   // [2]
    int* status;  // [1]: -1 finished, else the number of undecided arcs left
    int* cur_out; // [1]
    int* trace;   // [64]: live arcs of each round; [63] = rounds run; [128..]: 64 u64 timestamps
    int max_rounds;
    int agg;
    // batches (dense graphs): src = all arc records in processing (key) order; the rounds
    // start with an empty live list and reveal `batch` more records of src whenever the
    // live list has shrunk to batch / 4 or less.  Every arc is still decided only after all
    // lighter arcs are present, so the decisions are the sequential ones;
    // cycle arcs die in the first round after their batch is revealed instead of riding
    // along through every round.  batch = 0: everything is live from the start.
    const int4* src;
    int nsrc;
    int batch;
};

__device__ __forceinline__ int ld_cg_int(const int* p) { return __ldcg(p); }
// The lightest outgoing arc of every root, per round: best[r] = tag(round) << 32 | key
// with tags decreasing over the rounds, so a value left from an earlier round is always
// larger than any of this round's (no reset pass).  All lanes of the warp call it
// (active or not): lanes hitting the same root pre-reduce with match/redux and only
// the leader touches memory, and only if the stored value is larger -- the roots of
// the big components otherwise take one same-address atomic per incident arc.
__device__ __forceinline__ unsigned long long best_tag(int round) {
    return (unsigned long long)(0x7fffffffu - (uint32_t)round) << 32;
}
__device__ __forceinline__ void best_min(unsigned long long* best, int32_t r, uint32_t key, unsigned long long tag,
                                         bool active, int agg) {
    if (agg == 0) {
        if (active) atomicMin(best + r, tag | key);
        return;
    }
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const unsigned peers = __match_any_sync(act, r);
    const uint32_t kmin = __reduce_min_sync(peers, key);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
        const unsigned long long v = tag | kmin;
        if (agg == 1 || __ldcg(best + r) > v) atomicMin(best + r, v);
    }
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kBlock) k_uf_coop(UFArgs U) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int4 s_rec[kUFTile];  // pass A staging; the tail's sort list after the rounds
    __shared__ int s_cnt, s_base;
    unsigned long long* s_list = reinterpret_cast<unsigned long long*>(s_rec);
    const int stride = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int cur = 0;
    bool done = false;
    int rv = U.batch ? 0 : U.nsrc;  // records of src revealed so far
    for (int round = 0; round < U.max_rounds; round++) {
        const int4* live = cur ? U.rec1 : U.rec0;
        int4* nxt = cur ? U.rec0 : U.rec1;
        const int nl = ld_cg_int(&U.nlive[cur]);
        int add = 0;  // this round also takes src[rv .. rv + add)
        if (rv < U.nsrc && nl <= U.batch / 4) {
            add = min(U.batch, U.nsrc - rv);
        }
        const int n = nl + add;
        // pass A: roots of the arcs still undecided (records marked a = -1 were decided
        // last round), cycle arcs (same root: final, unpaired), lightest arc of every
        // root; the survivors are compacted into the next list with their roots
        const unsigned long long tag = best_tag(round);
        // tiles of kUFTile records per CTA: survivors gather in shared memory and leave
        // with one global atomic per tile (a per-warp atomic on the single list counter
        // serialises: measured 2/3 of the stall samples on 1D)
        // (a tile is K * kBlock records, K <= 4 chosen so that small rounds still spread
        // over the whole grid)
        const int K = min(kUFTile / kBlock, max(1, (n + stride - 1) / stride));
        for (int tile = blockIdx.x * K * kBlock; tile < n; tile += gridDim.x * K * kBlock) {
            if (threadIdx.x == 0) s_cnt = 0;
            __syncthreads();
            for (int k = 0; k < K; k++) {
                const int idx = tile + k * kBlock + threadIdx.x;
                int4 r = make_int4(0, 0, 0, 0);
                bool act = false;
                if (idx < n) {
                    r = idx < nl ? live[idx] : U.src[rv + (idx - nl)];
                    if (r.x >= 0) {
                        r.x = uf_find(U.parent, r.x);
                        r.y = uf_find(U.parent, r.y);
                        if (r.x == r.y) U.out[r.w] = -1;
                        else act = true;
                    }
                }
                best_min(U.best, r.x, (uint32_t)r.z, tag, act, U.agg);
                best_min(U.best, r.y, (uint32_t)r.z, tag, act, U.agg);
                const unsigned mk = __ballot_sync(0xffffffffu, act);
                int bp = 0;
                if (lane == 0 && mk) bp = atomicAdd(&s_cnt, __popc(mk));
                bp = __shfl_sync(0xffffffffu, bp, 0);
                if (act) s_rec[bp + __popc(mk & lanemask_lt())] = r;
            }
            __syncthreads();
            const int cnt = s_cnt;
            if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&U.nlive[cur ^ 1], cnt);
            __syncthreads();
            for (int j = threadIdx.x; j < cnt; j += kBlock) nxt[s_base + j] = s_rec[j];
            __syncthreads();
        }
        grid.sync();
        cur ^= 1;  // the survivors' list
        rv += add;
        const int m2 = ld_cg_int(&U.nlive[cur]);
        if (gtid == 0) {
            if (round < 63) {
                U.trace[round] = m2;
                reinterpret_cast<unsigned long long*>(U.trace + 128)[round] = globaltimer();
            }
            U.trace[63] = round;
            U.nlive[cur ^ 1] = 0;  // the list just consumed becomes the next round's output
        }
        if (m2 <= kUFTail && rv == U.nsrc) { done = true; break; }
        if (m2 == 0) {  // nothing to decide this round: reveal more next round
            grid.sync();  // (the counter reset above must land before the next appends)
            continue;
        }
        // pass B: mutual minimum, or a younger root dying at its lightest arc
        int4* sur = cur ? U.rec1 : U.rec0;
        for (int idx = gtid; idx < m2; idx += stride) {
            const int4 r = sur[idx];
            const unsigned long long kt = tag | (uint32_t)r.z;
            const bool ma = __ldcg(&U.best[r.x]) == kt, mb = __ldcg(&U.best[r.y]) == kt;
            if (!ma && !mb) continue;
            const bool a_older = U.age[r.x] < U.age[r.y];
            int32_t young = -1;
            if (ma && mb) {
                young = a_older ? r.y : r.x;
                U.parent[young] = a_older ? r.x : r.y;
            } else if (ma && !a_older) {
                young = r.x;
                U.parent[r.x] = r.y;
            } else if (mb && a_older) {
                young = r.y;
                U.parent[r.y] = r.x;
            }
            if (young >= 0) {
                U.out[r.w] = young;
                sur[idx].x = -1;
            }
        }
        grid.sync();
    }
    if (blockIdx.x != 0) return;
    const int n = ld_cg_int(&U.nlive[cur]);
    if (threadIdx.x == 0) *U.cur_out = cur;
    if (!done) {  // did not converge within max_rounds: the host finishes the tail
        if (threadIdx.x == 0) *U.status = n > 0 ? n : 1;
        return;
    }
    const int4* live = cur ? U.rec1 : U.rec0;
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int j = threadIdx.x; j < p2; j += blockDim.x)
        s_list[j] = j < n ? (((unsigned long long)(uint32_t)live[j].z << 32) | (uint32_t)j) : ~0ull;
    __syncthreads();
    // bitonic sort by key (ascending processing order)
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < p2; t += blockDim.x) {
                const int o = t ^ j;
                if (o > t) {
                    const unsigned long long x = s_list[t], y = s_list[o];
                    const bool up = (t & k) == 0;
                    if ((x > y) == up) { s_list[t] = y; s_list[o] = x; }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        for (int j = 0; j < n; j++) {
            const int4 r = live[(int)(s_list[j] & 0xffffffffull)];
            int32_t a = r.x, b = r.y;
            while (U.parent[a] != a) a = U.parent[a];
            while (U.parent[b] != b) b = U.parent[b];
            if (a == b) { U.out[r.w] = -1; continue; }
            const bool a_older = U.age[a] < U.age[b];
            const int32_t young = a_older ? b : a, old = a_older ? a : b;
            U.parent[young] = old;
            U.out[r.w] = young;
        }
        *U.status = -1;
    }
}

// sequential Kruskal over the undecided arcs in processing order (the result equals
// the full sequential union-find: DESIGN.md "Union-find")
__global__ void k_uf_tail(const int32_t* __restrict__ arc_a, const int32_t* __restrict__ arc_b, const int32_t* list,
                          int64_t n, int32_t* parent, int32_t* out, const int32_t* __restrict__ age) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int64_t j = 0; j < n; j++) {
        const int32_t i = list[j];
        int32_t a = arc_a[i], b = arc_b[i];
        while (parent[a] != a) a = parent[a];
        while (parent[b] != b) b = parent[b];
        if (a == b) { out[i] = -1; continue; }
        const bool a_older = age[a] < age[b];
        const int32_t young = a_older ? b : a, old = a_older ? a : b;
        parent[young] = old;
        out[i] = young;
    }
}

// ---------------------------------------------------------------- emission

struct alignas(16) PairRec {  // 32 B, two 16-byte stores per record
    int64_t birth_id, death_id;
    int32_t birth_vertex, death_vertex;
    float birth_value, death_value;
};

// highest vertex (in K) of an anchored simplex
__device__ __forceinline__ int64_t max_vertex(const Geo3& g, const StarTab& S, int dim, int64_t id) {
    if (dim == 0) return id;
    if (g.t5) return t5_max_vertex(g.f, g.Lx, g.Ly, g.t5, dim, id);
    const int64_t a = id / g.ncell[dim];
    const int k = (int)(id % g.ncell[dim]);
    int64_t best = a;
    for (int j = 0; j < dim; j++) {
        const int64_t p = a + lin_mask(g, S.chain[dim][k][j]);
        if (kless_v(g, best, p)) best = p;
    }
    return best;
}

__global__ void k_flag_ge0(const int32_t* out, int64_t m, uint32_t* flags, int want_unpaired) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flags[i] = want_unpaired ? (out[i] == -1 ? 1u : 0u) : (out[i] >= 0 ? 1u : 0u);
}

// D0 pairs (birth = the dying minimum, death = the critical edge), ascending arcs
// out: processing order; its values are node (minimum) emission indices into c0e
__global__ void k_emit_d0(Geo3 g, const int32_t* out, int64_t m, const uint32_t* pos, const int64_t* c0e,
                          const int64_t* c1, PairRec* pairs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || out[i] < 0) return;
    const StarTab& S = *g.tab;
    PairRec r;
    r.birth_id = c0e[out[i]];
    r.birth_vertex = (int32_t)r.birth_id;
    r.birth_value = g.f[r.birth_id];
    r.death_id = c1[i];
    const int64_t dv = max_vertex(g, S, 1, r.death_id);
    r.death_vertex = (int32_t)dv;
    r.death_value = g.f[dv];
    pairs[pos[i]] = r;
}

// D_{d-1} pairs (birth = critical (d-1)-simplex, death = the dying maximum), in
// processing (decreasing) order
__global__ void k_emit_dtop(Geo3 g, const int32_t* out, int64_t m, const uint32_t* pos, const int64_t* cdm1,
                            const int64_t* cde, PairRec* pairs) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m || out[j] < 0) return;
    const StarTab& S = *g.tab;
    const int d = g.ndim;
    PairRec r;
    r.birth_id = cdm1[m - 1 - j];
    const int64_t bv = max_vertex(g, S, d - 1, r.birth_id);
    r.birth_vertex = (int32_t)bv;
    r.birth_value = g.f[bv];
    r.death_id = cde[out[j]];
    const int64_t dv = max_vertex(g, S, d, r.death_id);
    r.death_vertex = (int32_t)dv;
    r.death_value = g.f[dv];
    pairs[pos[j]] = r;
}

// unpaired saddles, in ascending lex order.  rev: the arcs are in decreasing order.
__global__ void k_emit_unpaired(const int32_t* out, int64_t m, const uint32_t* pos, int64_t n, const int64_t* ids,
                                int64_t* list, int rev) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m || out[j] != -1) return;
    const int64_t id = rev ? ids[m - 1 - j] : ids[j];
    list[rev ? n - 1 - pos[j] : pos[j]] = id;
}

// same, with the count taken on the device (n = exclusive-scan end + last flag), so the
// host does not wait for it
__global__ void k_emit_unpaired_dev(const int32_t* out, int64_t m, const uint32_t* pos, const uint32_t* flags,
                                    const int64_t* ids, int64_t* list, int rev) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m || out[j] != -1) return;
    const int64_t n = (int64_t)__ldg(pos + m - 1) + __ldg(flags + m - 1);
    const int64_t id = rev ? ids[m - 1 - j] : ids[j];
    list[rev ? n - 1 - pos[j] : pos[j]] = id;
}

}  // namespace dms
