// tet5.cuh -- the five-tetrahedra subdivision of a 3D grid (sm_100a): SURVEY 8(f) #4.
//
// PAPER.md 662-664 (Sec. 8.1): the paper's 3D benchmark volumes are "triangulated into a
// simplicial complex by breaking up each cell into ... five tetrahedra".  Reading Z21
// (DESIGN.md): the cube with minimum corner a, parity p = (ax + ay + az) mod 2, is cut
// into the central tetrahedron on its corners c (local bit masks x=1, y=2, z=4) with
// popcount(c) + p even, and the four corner tetrahedra {o, o^1, o^2, o^4} at its other
// corners o.  The central corners are the vertices of even coordinate sum in every cube,
// so neighbouring cubes cut their common square along the same diagonal.  A vertex of
// even coordinate sum has 18 neighbours (6 axis + 12 face diagonals; 48 star triangles,
// 32 star tetrahedra), an odd one 6 (12, 8): two star classes, both tabulated here on the
// host from that rule (no table is shared with the oracle).
//
// Simplex ids (reading Z21): a k-simplex is anchored at its component-wise minimum a;
// id = C_k * vid(a) + idx, C_k = 1 / 6 / 10 / 5, idx = the position of its vertex
// offsets from a (ascending masks) among the k-simplices of the cube at a whose
// component-wise minimum is a, for a's parity, sorted ascending as tuples.
//
// Gradient layout (dms_gradient_bytes = 16 N), one byte per cell, indexed by cell id:
//   [0, N)        vertex code: star slot of the edge paired with the vertex, 0xFF minimum
//   [N, 11N)      triangle code: j < 3 -- paired with its facet edge omitting vertex j
//                 (ascending-mask order of its id entry), 0xFE -- paired with a
//                 tetrahedron (the tail of that vector), 0xFF -- critical
//   [11N, 16N)    tetrahedron code: j < 4 -- paired with its facet omitting vertex j,
//                 0xFF -- critical
// (an edge is paired with its higher vertex, with a triangle, or is critical: its pairing
// is read off the codes above).  Every byte of a cell of the complex is written by the
// thread of the cell's highest vertex (the lower star it belongs to).
#pragma once
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace dms {

constexpr int kT5NE = 18, kT5NT = 48, kT5NQ = 32;

// the star of a vertex of one parity class (0: even coordinate sum)
struct alignas(16) T5Star {
    int ne, nt, nq, nneg;  // nneg: slots before x in vertex-id order (the index tie-break)
    int8_t off[kT5NE][3];  // neighbour offsets, slots sorted by (dz, dy, dx) = vertex-id order
    uint8_t tri_a[kT5NT], tri_b[kT5NT];                  // neighbour slots, a < b
    uint8_t tet_a[kT5NQ], tet_b[kT5NQ], tet_c[kT5NQ];    // a < b < c
    uint32_t tri_emask[kT5NT];   // the triangle's two star edges (x,a), (x,b)
    uint32_t tri_qmask[kT5NT];   // star tetrahedra holding the triangle
    uint64_t tet_tmask[kT5NQ];   // the tetrahedron's three star triangles
    uint64_t edge_tmask[kT5NE];  // star triangles holding the edge
    // anchored ids of the star cells: anchor offset from x, index in the anchor's table,
    // and the positions of x, n_a (, n_b, n_c) in the cell's ascending-mask vertex list
    int8_t e_anc[kT5NE][3];
    uint8_t e_k[kT5NE];
    int8_t t_anc[kT5NT][3];
    uint8_t t_k[kT5NT], t_pos[kT5NT][3];
    int8_t q_anc[kT5NQ][3];
    uint8_t q_k[kT5NQ], q_pos[kT5NQ][4];
};

struct alignas(16) T5Tab {
    T5Star star[2];
    uint8_t ids[2][4][10][4];  // [anchor parity][k][idx] -> ascending vertex masks
    uint8_t cnt[4];            // cells per anchor: 1, 6, 10, 5
    // dual adjacency: [cube parity][tet idx][facet j (omits vertex j)] -> idx | dir << 4,
    // dir 0 = the same cube, 1..6 = the cube at -x, +x, -y, +y, -z, +z
    uint8_t tet_nbr[2][5][4];
    // cofacets of a triangle anchored at a: [parity of a][idx][side] -> idx | dir << 4
    // (dir 0: the cube at a, 1 / 3 / 5: the cube at a - e_x / e_y / e_z), 0xFF none
    uint8_t tri_cof[2][10][2];
};

// ------------------------------------------------------------------ host construction
namespace t5detail {

inline int pc3(int m) { return (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1); }

// the five tetrahedra of a cube of parity p, as local corner masks (central first)
inline std::vector<std::array<int, 4>> cube_tets(int p) {
    std::vector<std::array<int, 4>> out(1);
    int nc = 0;
    for (int c = 0; c < 8; c++) {
        if (((pc3(c) + p) & 1) == 0) out[0][nc++] = c;
        else out.push_back({c, c ^ 1, c ^ 2, c ^ 4});
    }
    return out;
}

using P3 = std::array<int, 3>;
inline P3 mask_pt(int m) { return {m & 1, (m >> 1) & 1, (m >> 2) & 1}; }

// anchor (component-wise minimum) and ascending masks of a set of lattice points
inline void anchor_masks(const std::vector<P3>& pts, P3& a, std::vector<int>& masks) {
    a = pts[0];
    for (auto& q : pts)
        for (int ax = 0; ax < 3; ax++) a[ax] = std::min(a[ax], q[ax]);
    masks.clear();
    for (auto& q : pts) {
        int m = 0;
        for (int ax = 0; ax < 3; ax++) m |= (q[ax] - a[ax]) << ax;
        masks.push_back(m);
    }
    std::sort(masks.begin(), masks.end());
}

inline int par(const P3& a) { return ((a[0] + a[1] + a[2]) % 2 + 2) % 2; }

}  // namespace t5detail

// builds every table; returns false on an inconsistency
inline bool build_t5_tables(T5Tab* T) {
    using namespace t5detail;
    std::memset(T, 0xff, sizeof(T5Tab));
    // id tables: faces of the cube's tetrahedra whose component-wise minimum is the anchor
    for (int p = 0; p < 2; p++) {
        auto tets = cube_tets(p);
        for (int k = 0; k <= 3; k++) {
            std::vector<std::vector<int>> cells;
            for (auto& t : tets)
                for (int sub = 1; sub < 16; sub++) {
                    if (__builtin_popcount(sub) != k + 1) continue;
                    std::vector<int> m;
                    int andm = 7;
                    for (int j = 0; j < 4; j++)
                        if ((sub >> j) & 1) { m.push_back(t[j]); andm &= t[j]; }
                    if (andm) continue;
                    std::sort(m.begin(), m.end());
                    if (std::find(cells.begin(), cells.end(), m) == cells.end()) cells.push_back(m);
                }
            std::sort(cells.begin(), cells.end());
            if (cells.size() > 10) return false;
            if (p == 1 && (int)cells.size() != T->cnt[k]) return false;
            T->cnt[k] = (uint8_t)cells.size();
            for (size_t i = 0; i < cells.size(); i++)
                for (int j = 0; j <= k; j++) T->ids[p][k][i][j] = (uint8_t)cells[i][j];
        }
    }
    if (T->cnt[0] != 1 || T->cnt[1] != 6 || T->cnt[2] != 10 || T->cnt[3] != 5) return false;
    // id of a cell given as lattice points relative to a vertex of parity P0: anchor + index
    auto idx_of = [&](const std::vector<P3>& pts, P3& anc, int P0) -> int {
        std::vector<int> m;
        anchor_masks(pts, anc, m);
        const int k = (int)pts.size() - 1, p = (P0 + par(anc)) & 1;
        for (int i = 0; i < T->cnt[k]; i++) {
            bool eq = true;
            for (int j = 0; j <= k; j++) eq = eq && T->ids[p][k][i][j] == m[j];
            if (eq) return i;
        }
        return -1;
    };
    // stars: the tetrahedra of the 8 cubes around x = 0 (cube min corner -b) holding x
    for (int P = 0; P < 2; P++) {
        T5Star& S = T->star[P];
        std::vector<std::array<P3, 4>> stets;
        for (int b = 0; b < 8; b++) {
            const P3 c = {-(b & 1), -((b >> 1) & 1), -((b >> 2) & 1)};
            const int cp = (P + pc3(b)) & 1;
            for (auto& t : cube_tets(cp)) {
                std::array<P3, 4> q;
                bool has0 = false;
                for (int j = 0; j < 4; j++) {
                    const P3 m = mask_pt(t[j]);
                    q[j] = {c[0] + m[0], c[1] + m[1], c[2] + m[2]};
                    has0 = has0 || (q[j] == P3{0, 0, 0});
                }
                if (has0) stets.push_back(q);
            }
        }
        // neighbours (the other vertices of the star tetrahedra), sorted by (dz, dy, dx)
        std::vector<P3> nb;
        for (auto& q : stets)
            for (auto& v : q)
                if (v != P3{0, 0, 0} && std::find(nb.begin(), nb.end(), v) == nb.end()) nb.push_back(v);
        std::sort(nb.begin(), nb.end(), [](const P3& u, const P3& v) {
            return std::make_tuple(u[2], u[1], u[0]) < std::make_tuple(v[2], v[1], v[0]);
        });
        if ((int)nb.size() > kT5NE) return false;
        S.ne = (int)nb.size();
        S.nneg = 0;
        for (int s = 0; s < S.ne; s++) {
            for (int ax = 0; ax < 3; ax++) S.off[s][ax] = (int8_t)nb[s][ax];
            if (std::make_tuple(nb[s][2], nb[s][1], nb[s][0]) < std::make_tuple(0, 0, 0)) S.nneg++;
        }
        auto slot = [&](const P3& v) { return (int)(std::find(nb.begin(), nb.end(), v) - nb.begin()); };
        // triangles and tetrahedra of the star as slot tuples
        std::vector<std::array<int, 2>> tris;
        std::vector<std::array<int, 3>> qs;
        for (auto& q : stets) {
            std::vector<int> o;
            for (auto& v : q)
                if (v != P3{0, 0, 0}) o.push_back(slot(v));
            std::sort(o.begin(), o.end());
            qs.push_back({o[0], o[1], o[2]});
            for (int i = 0; i < 3; i++)
                for (int j = i + 1; j < 3; j++) {
                    std::array<int, 2> t = {o[i], o[j]};
                    if (std::find(tris.begin(), tris.end(), t) == tris.end()) tris.push_back(t);
                }
        }
        std::sort(tris.begin(), tris.end());
        std::sort(qs.begin(), qs.end());
        if ((int)tris.size() > kT5NT || (int)qs.size() > kT5NQ) return false;
        S.nt = (int)tris.size();
        S.nq = (int)qs.size();
        for (int s = 0; s < S.ne; s++) S.edge_tmask[s] = 0;
        for (int t = 0; t < S.nt; t++) {
            S.tri_a[t] = (uint8_t)tris[t][0];
            S.tri_b[t] = (uint8_t)tris[t][1];
            S.tri_emask[t] = (1u << tris[t][0]) | (1u << tris[t][1]);
            S.tri_qmask[t] = 0;
            S.edge_tmask[tris[t][0]] |= 1ull << t;
            S.edge_tmask[tris[t][1]] |= 1ull << t;
        }
        auto tri_slot = [&](int a, int b) {
            std::array<int, 2> t = {std::min(a, b), std::max(a, b)};
            return (int)(std::find(tris.begin(), tris.end(), t) - tris.begin());
        };
        for (int q = 0; q < S.nq; q++) {
            S.tet_a[q] = (uint8_t)qs[q][0];
            S.tet_b[q] = (uint8_t)qs[q][1];
            S.tet_c[q] = (uint8_t)qs[q][2];
            const int t0 = tri_slot(qs[q][0], qs[q][1]), t1 = tri_slot(qs[q][0], qs[q][2]),
                      t2 = tri_slot(qs[q][1], qs[q][2]);
            if (t0 >= S.nt || t1 >= S.nt || t2 >= S.nt) return false;
            S.tet_tmask[q] = (1ull << t0) | (1ull << t1) | (1ull << t2);
            S.tri_qmask[t0] |= 1u << q;
            S.tri_qmask[t1] |= 1u << q;
            S.tri_qmask[t2] |= 1u << q;
        }
        // anchored ids and vertex positions
        const P3 o = {0, 0, 0};
        auto pos_in = [&](const P3& anc, int p, int k, int idx, const P3& v) {
            int m = 0;
            for (int ax = 0; ax < 3; ax++) m |= (v[ax] - anc[ax]) << ax;
            for (int j = 0; j <= k; j++)
                if (T->ids[p][k][idx][j] == m) return j;
            return -1;
        };
        for (int s = 0; s < S.ne; s++) {
            P3 anc;
            const int i = idx_of({o, nb[s]}, anc, P);
            if (i < 0) return false;
            for (int ax = 0; ax < 3; ax++) S.e_anc[s][ax] = (int8_t)anc[ax];
            S.e_k[s] = (uint8_t)i;
        }
        for (int t = 0; t < S.nt; t++) {
            P3 anc;
            const P3 a = nb[S.tri_a[t]], b = nb[S.tri_b[t]];
            const int i = idx_of({o, a, b}, anc, P);
            if (i < 0) return false;
            for (int ax = 0; ax < 3; ax++) S.t_anc[t][ax] = (int8_t)anc[ax];
            S.t_k[t] = (uint8_t)i;
            const int p = (P + par(anc)) & 1;
            S.t_pos[t][0] = (uint8_t)pos_in(anc, p, 2, i, o);
            S.t_pos[t][1] = (uint8_t)pos_in(anc, p, 2, i, a);
            S.t_pos[t][2] = (uint8_t)pos_in(anc, p, 2, i, b);
        }
        for (int q = 0; q < S.nq; q++) {
            P3 anc;
            const P3 a = nb[S.tet_a[q]], b = nb[S.tet_b[q]], c = nb[S.tet_c[q]];
            const int i = idx_of({o, a, b, c}, anc, P);
            if (i < 0) return false;
            for (int ax = 0; ax < 3; ax++) S.q_anc[q][ax] = (int8_t)anc[ax];
            S.q_k[q] = (uint8_t)i;
            const int p = (P + par(anc)) & 1;
            S.q_pos[q][0] = (uint8_t)pos_in(anc, p, 3, i, o);
            S.q_pos[q][1] = (uint8_t)pos_in(anc, p, 3, i, a);
            S.q_pos[q][2] = (uint8_t)pos_in(anc, p, 3, i, b);
            S.q_pos[q][3] = (uint8_t)pos_in(anc, p, 3, i, c);
        }
    }
    // dual adjacency of the tetrahedra (every tetrahedron spans its cube: anchor = cube)
    for (int p = 0; p < 2; p++) {
        auto tets = cube_tets(p);
        for (int q = 0; q < 5; q++) {
            std::vector<int> qm(T->ids[p][3][q], T->ids[p][3][q] + 4);
            for (int j = 0; j < 4; j++) {
                std::vector<int> fm;
                for (int u = 0; u < 4; u++)
                    if (u != j) fm.push_back(qm[u]);
                int found = -1, dir = 0;
                for (int q2 = 0; q2 < 5 && found < 0; q2++) {
                    if (q2 == q) continue;
                    int hit = 0;
                    for (int u = 0; u < 3; u++)
                        for (int w = 0; w < 4; w++) hit += T->ids[p][3][q2][w] == fm[u];
                    if (hit == 3) found = q2;
                }
                if (found < 0) {  // on a cube face: the tetrahedron of the neighbouring cube
                    int ax = -1, v = 0;
                    for (int a = 0; a < 3 && ax < 0; a++) {
                        const int b0 = (fm[0] >> a) & 1;
                        if (((fm[1] >> a) & 1) == b0 && ((fm[2] >> a) & 1) == b0) { ax = a; v = b0; }
                    }
                    if (ax < 0) return false;
                    dir = 1 + 2 * ax + v;
                    std::vector<int> gm;
                    for (int u = 0; u < 3; u++) gm.push_back(fm[u] ^ (1 << ax));
                    for (int q2 = 0; q2 < 5 && found < 0; q2++) {
                        int hit = 0;
                        for (int u = 0; u < 3; u++)
                            for (int w = 0; w < 4; w++) hit += T->ids[p ^ 1][3][q2][w] == gm[u];
                        if (hit == 3) found = q2;
                    }
                    if (found < 0) return false;
                }
                T->tet_nbr[p][q][j] = (uint8_t)(found | (dir << 4));
            }
        }
        // cofacets of the triangles anchored at a
        for (int t = 0; t < T->cnt[2]; t++) {
            const uint8_t* tm = T->ids[p][2][t];
            int n = 0;
            for (int q = 0; q < 5; q++) {  // in the cube at a
                int hit = 0;
                for (int u = 0; u < 3; u++)
                    for (int w = 0; w < 4; w++) hit += T->ids[p][3][q][w] == tm[u];
                if (hit == 3) T->tri_cof[p][t][n++] = (uint8_t)q;
            }
            const int orm = tm[0] | tm[1] | tm[2];
            for (int ax = 0; ax < 3; ax++) {  // on the cube's lower face of axis ax
                if ((orm >> ax) & 1) continue;
                for (int q = 0; q < 5; q++) {
                    int hit = 0;
                    for (int u = 0; u < 3; u++)
                        for (int w = 0; w < 4; w++) hit += T->ids[p ^ 1][3][q][w] == (tm[u] | (1 << ax));
                    if (hit == 3) {
                        if (n >= 2) return false;
                        T->tri_cof[p][t][n++] = (uint8_t)(q | ((1 + 2 * ax) << 4));
                    }
                }
            }
            if (n != 2) return false;  // every triangle has two cofacets in the infinite grid
        }
    }
    return true;
}

// ------------------------------------------------------------------ device: geometry helpers

struct T5Geo {
    int32_t Lx, Ly, Lz;
    int64_t N;
};

__device__ __forceinline__ bool t5_cube_ok(const T5Geo& g, int cx, int cy, int cz) {
    return cx >= 0 && cy >= 0 && cz >= 0 && cx <= g.Lx - 2 && cy <= g.Ly - 2 && cz <= g.Lz - 2;
}

__device__ __forceinline__ void t5_dir(int dir, int& dx, int& dy, int& dz) {
    dx = dy = dz = 0;
    if (dir == 0) return;
    const int ax = (dir - 1) >> 1, s = ((dir - 1) & 1) ? 1 : -1;
    if (ax == 0) dx = s;
    else if (ax == 1) dy = s;
    else dz = s;
}

// G: the lexicographic key of a lower-star cell (x, n_1, n_2, n_3) (PAPER.md 1380-1414:
// decreasing vertex sequences, a face before its cofaces) from the local ranks r1 > r2 > r3
// of its other vertices among x's lower neighbours (-1 = absent), as the dense position
// among all such cells: #cells whose highest other vertex is below r1, then the edge, then
// the cells (r1, r2, ...).  < 987 for 18 neighbours, so the records keep the 12-bit G slot.
__device__ __forceinline__ uint32_t t5_key(int r1, int r2, int r3) {
    uint32_t k = (uint32_t)(r1 + r1 * (r1 - 1) / 2 + r1 * (r1 - 1) * (r1 - 2) / 6);
    if (r2 >= 0) {
        k += 1u + (uint32_t)(r2 + r2 * (r2 - 1) / 2);
        if (r3 >= 0) k += 1u + (uint32_t)r3;
    }
    return k;
}

struct T5Args {
    const float* f;
    int32_t Lx, Ly, Lz;
    int64_t N;
    int64_t v0, v1;
    const T5Tab* tab;
    uint8_t* grad;
    int64_t* crit_id[4];
    uint64_t* crit_key[4];
    int64_t cap[4];
    unsigned long long* totals;
    int* err;
};

__device__ __forceinline__ int64_t t5_warp_append(unsigned long long* total, uint32_t cnt) {
    const int lane = threadIdx.x & 31;
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(total, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31);
    return (int64_t)base + (inc - cnt);
}

constexpr int kT5Block = 128;

// ProcessLowerStars (Robins et al.; reading Z1, the oracle's O3 step by step) on the lower
// star of one vertex of the five-tetrahedra complex.  Cells are star slots: edges (x, n_s),
// triangles (x, n_a, n_b), tetrahedra (x, n_a, n_b, n_c); the queues and the
// classification are bit masks over those slots, the minimum of a queue is found by
// scanning its members' keys (t5_key).  One thread per vertex.
__global__ void __launch_bounds__(kT5Block) k_gradient_t5(T5Args A) {
    __shared__ T5Star S[2];
    // the keys of the thread's lower triangles / tetrahedra, [cell][thread] (computed once
    // per star: every queue pop scans its members' keys)
    __shared__ uint16_t s_key[(kT5NT + kT5NQ) * kT5Block];
    uint16_t* const mykey = s_key + threadIdx.x;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A.tab->star);
        uint32_t* dst = reinterpret_cast<uint32_t*>(S);
        for (int i = threadIdx.x; i < (int)(sizeof(S) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const int64_t LxLy = (int64_t)A.Lx * A.Ly;
    // consecutive vertices alternate between the 18- and the 6-neighbour class (within a row):
    // a pair of CTAs shares a window of 2 x 128 vertices, one takes its even offsets, the other
    // its odd ones, so a CTA (and each of its warps) runs one class and the short CTAs of
    // 6-neighbour stars retire early instead of idling beside the long ones
    const int64_t v = A.v0 + (int64_t)(blockIdx.x >> 1) * (2 * kT5Block) + 2 * (int64_t)threadIdx.x + (blockIdx.x & 1);
    const bool active = v < A.v1;
    uint32_t critE = 0, critQ = 0, crit_v = 0;
    uint64_t critT = 0;
    int P = 0;
    uint64_t R0 = 0, R1 = 0;  // local ranks of the lower slots, 5 bits each (slots 0-11 | 12-17)
    if (active) {
        const int x = (int)(v % A.Lx), y = (int)((v / A.Lx) % A.Ly), z = (int)(v / LxLy);
        P = (x + y + z) & 1;
        const T5Star& T = S[P];
        const float fx = __ldg(A.f + v);
        if (fx != fx) atomicOr(A.err, 1);
        const uint32_t ox = ord_of(fx);
        uint32_t on[kT5NE];
        uint32_t low = 0;
#pragma unroll
        for (int s = 0; s < kT5NE; s++) {
            on[s] = 0xffffffffu;
            if (s < T.ne) {
                const int nx = x + T.off[s][0], ny = y + T.off[s][1], nz = z + T.off[s][2];
                if (nx >= 0 && ny >= 0 && nz >= 0 && nx < A.Lx && ny < A.Ly && nz < A.Lz) {
                    on[s] = ord_of(__ldg(A.f + (v + T.off[s][0] + (int64_t)A.Lx * T.off[s][1] + LxLy * T.off[s][2])));
                    if (on[s] < ox || (on[s] == ox && s < T.nneg)) low |= 1u << s;
                }
            }
        }
        // local ranks among the lower neighbours (vertex-id order = slot order on ties)
#pragma unroll
        for (int s = 0; s < kT5NE; s++) {
            if (!((low >> s) & 1u)) continue;
            int r = 0;
#pragma unroll
            for (int t = 0; t < kT5NE; t++)
                r += ((low >> t) & 1u) && (on[t] < on[s] || (on[t] == on[s] && t < s));
            if (s < 12) R0 |= (uint64_t)r << (5 * s);
            else R1 |= (uint64_t)r << (5 * (s - 12));
        }
        auto rk = [&](int s) -> int { return (int)(((s < 12 ? R0 >> (5 * s) : R1 >> (5 * (s - 12)))) & 31ull); };
        auto keyE = [&](int s) -> uint32_t { return t5_key(rk(s), -1, -1); };
        auto keyT = [&](int t) -> uint32_t {
            const int a = rk(T.tri_a[t]), b = rk(T.tri_b[t]);
            return t5_key(max(a, b), min(a, b), -1);
        };
        auto keyQ = [&](int q) -> uint32_t {
            int a = rk(T.tet_a[q]), b = rk(T.tet_b[q]), c = rk(T.tet_c[q]);
            const int hi = max(a, max(b, c)), lo = min(a, min(b, c));
            return t5_key(hi, a + b + c - hi - lo, lo);
        };
        uint64_t lowT = 0;
        uint32_t lowQ = 0;
        for (int t = 0; t < T.nt; t++)
            if ((T.tri_emask[t] & low) == T.tri_emask[t]) lowT |= 1ull << t;
        for (int q = 0; q < T.nq; q++)
            if ((T.tet_tmask[q] & lowT) == T.tet_tmask[q]) lowQ |= 1u << q;
        for (uint64_t m = lowT; m; m &= m - 1) {
            const int t = __ffsll((long long)m) - 1;
            mykey[t * kT5Block] = (uint16_t)keyT(t);
        }
        for (uint32_t m = lowQ; m; m &= m - 1) {
            const int q = __ffs(m) - 1;
            mykey[(kT5NT + q) * kT5Block] = (uint16_t)keyQ(q);
        }
        uint64_t tc_lo = 0, tc_hi = 0;  // 2-bit triangle codes: 1 / 2 paired with edge a / b, 3 tail, 0 critical
        uint64_t qc = 0;                // 2-bit tetrahedron codes: 1..3 paired with triangle 0..2 (ab, ac, bc), 0 critical
        int vcode = 0xff;
        if (low == 0) {
            crit_v = 1;
        } else {
            uint32_t cE = 0, cQ = 0, zE = 0, zQ = 0, oQ = 0;
            uint64_t cT = 0, zT = 0, oT = 0;
            // delta: the lowest lower neighbour (local rank 0)
            int delta = 0;
            for (int s = 0; s < T.ne; s++)
                if (((low >> s) & 1u) && rk(s) == 0) delta = s;
            vcode = delta;
            cE = 1u << delta;
            zE = low & ~cE;
            {
                const uint64_t mm = T.edge_tmask[delta] & lowT;
#pragma unroll
                for (int h = 0; h < 2; h++)
                    for (uint32_t m = h ? (uint32_t)(mm >> 32) : (uint32_t)mm; m; m &= m - 1) {
                        const int t = __ffs(m) - 1 + 32 * h;
                        if (__popc(T.tri_emask[t] & ~cE) == 1) oT |= 1ull << t;
                    }
            }
            auto set_tcode = [&](int t, uint64_t code) {
                if (t < 32) tc_lo |= code << (2 * t);
                else tc_hi |= code << (2 * (t - 32));
            };
            // push every unclassified cofacet of a classified cell with one unclassified facet
            auto push_cof_tri_of_edge = [&](int e) {
                const uint64_t mm = T.edge_tmask[e] & lowT & ~cT;
#pragma unroll
                for (int h = 0; h < 2; h++)
                    for (uint32_t m = h ? (uint32_t)(mm >> 32) : (uint32_t)mm; m; m &= m - 1) {
                        const int b = __ffs(m) - 1 + 32 * h;
                        if (__popc(T.tri_emask[b] & ~cE) == 1) oT |= 1ull << b;
                    }
            };
            auto push_cof_tet_of_tri = [&](int t) {
                for (uint32_t m = T.tri_qmask[t] & lowQ & ~cQ; m; m &= m - 1) {
                    const int b = __ffs(m) - 1;
                    if (__popcll(T.tet_tmask[b] & ~cT) == 1) oQ |= 1u << b;
                }
            };
            for (;;) {
                if (!(zE | zQ | oQ) && !(zT | oT)) break;
                while (oT || oQ) {
                    // pop the minimum-key member of PQone
                    uint32_t best = 0xffffffffu;
                    int bi = -1, bty = 0;
                    // (48 triangle slots: two 32-bit scans are cheaper than one over 64 bits)
#pragma unroll
                    for (int h = 0; h < 2; h++)
                        for (uint32_t m = h ? (uint32_t)(oT >> 32) : (uint32_t)oT; m; m &= m - 1) {
                            const int t = __ffs(m) - 1 + 32 * h;
                            const uint32_t k = mykey[t * kT5Block];
                            if (k < best) { best = k; bi = t; bty = 2; }
                        }
                    for (uint32_t m = oQ; m; m &= m - 1) {
                        const int q = __ffs(m) - 1;
                        const uint32_t k = mykey[(kT5NT + q) * kT5Block];
                        if (k < best) { best = k; bi = q; bty = 3; }
                    }
                    if (bty == 2) {
                        oT &= ~(1ull << bi);
                        if ((cT >> bi) & 1ull) continue;
                        const uint32_t fr = T.tri_emask[bi] & ~cE;
                        if (fr == 0) { zT |= 1ull << bi; continue; }
                        const int e = __ffs(fr) - 1;  // its unique unclassified facet
                        cE |= 1u << e;
                        cT |= 1ull << bi;
                        zE &= ~(1u << e);
                        set_tcode(bi, e == T.tri_a[bi] ? 1ull : 2ull);
                        push_cof_tet_of_tri(bi);  // cofacets of the pair's head ...
                        push_cof_tri_of_edge(e);  // ... and of its tail
                    } else {
                        oQ &= ~(1u << bi);
                        if ((cQ >> bi) & 1u) continue;
                        const uint64_t fr = T.tet_tmask[bi] & ~cT;
                        if (fr == 0) { zQ |= 1u << bi; continue; }
                        const int t = __ffsll((long long)fr) - 1;
                        cT |= 1ull << t;
                        cQ |= 1u << bi;
                        zT &= ~(1ull << t);
                        set_tcode(t, 3ull);
                        const int j = (int)(__popcll(T.tet_tmask[bi] & ((1ull << t) - 1ull)));  // 0: ab, 1: ac, 2: bc
                        qc |= (uint64_t)(j + 1) << (2 * bi);
                        push_cof_tet_of_tri(t);
                    }
                }
                // pop the minimum of PQzero: critical
                uint32_t best = 0xffffffffu;
                int bi = -1, bty = 0;
                for (uint32_t m = zE; m; m &= m - 1) {
                    const int s = __ffs(m) - 1;
                    const uint32_t k = keyE(s);
                    if (k < best) { best = k; bi = s; bty = 1; }
                }
#pragma unroll
                for (int h = 0; h < 2; h++)
                    for (uint32_t m = h ? (uint32_t)(zT >> 32) : (uint32_t)zT; m; m &= m - 1) {
                        const int t = __ffs(m) - 1 + 32 * h;
                        const uint32_t k = mykey[t * kT5Block];
                        if (k < best) { best = k; bi = t; bty = 2; }
                    }
                for (uint32_t m = zQ; m; m &= m - 1) {
                    const int q = __ffs(m) - 1;
                    const uint32_t k = mykey[(kT5NT + q) * kT5Block];
                    if (k < best) { best = k; bi = q; bty = 3; }
                }
                if (bi < 0) continue;
                if (bty == 1) {
                    zE &= ~(1u << bi);
                    if ((cE >> bi) & 1u) continue;
                    cE |= 1u << bi;
                    critE |= 1u << bi;
                    push_cof_tri_of_edge(bi);
                } else if (bty == 2) {
                    zT &= ~(1ull << bi);
                    if ((cT >> bi) & 1ull) continue;
                    cT |= 1ull << bi;
                    critT |= 1ull << bi;
                    push_cof_tet_of_tri(bi);
                } else {
                    zQ &= ~(1u << bi);
                    if ((cQ >> bi) & 1u) continue;
                    cQ |= 1u << bi;
                    critQ |= 1u << bi;
                }
            }
        }
        // gradient bytes: the vertex, then every lower triangle / tetrahedron by id
        A.grad[v] = (uint8_t)vcode;
        for (uint64_t m = lowT; m; m &= m - 1) {
            const int t = __ffsll((long long)m) - 1;
            const uint32_t code = (uint32_t)((t < 32 ? tc_lo >> (2 * t) : tc_hi >> (2 * (t - 32))) & 3ull);
            const uint8_t byte = code == 0 ? 0xff : code == 3 ? 0xfe : T.t_pos[t][code == 1 ? 2 : 1];
            const int64_t anc = v + T.t_anc[t][0] + (int64_t)A.Lx * T.t_anc[t][1] + LxLy * T.t_anc[t][2];
            A.grad[A.N + 10 * anc + T.t_k[t]] = byte;
        }
        for (uint32_t m = lowQ; m; m &= m - 1) {
            const int q = __ffs(m) - 1;
            const uint32_t code = (uint32_t)((qc >> (2 * q)) & 3ull);
            // facet j of the star tet: (x,a,b) omits c, (x,a,c) omits b, (x,b,c) omits a
            const uint8_t byte = code == 0 ? 0xff : T.q_pos[q][code == 1 ? 3 : code == 2 ? 2 : 1];
            const int64_t anc = v + T.q_anc[q][0] + (int64_t)A.Lx * T.q_anc[q][1] + LxLy * T.q_anc[q][2];
            A.grad[11 * A.N + 5 * anc + T.q_k[q]] = byte;
        }
    }
    // critical records: (anchored id, placeholder key x << 12 | G), rewritten to
    // rank(x) << 12 | G by dms_critical (the key format of the Freudenthal path)
    const T5Star& T = S[P];
    auto rk = [&](int s) -> int { return (int)(((s < 12 ? R0 >> (5 * s) : R1 >> (5 * (s - 12)))) & 31ull); };
    const uint64_t rkey = (uint64_t)v << 12;
    {
        const int64_t q0 = t5_warp_append(&A.totals[0], crit_v);
        if (crit_v && q0 < A.cap[0]) { A.crit_id[0][q0] = v; A.crit_key[0][q0] = rkey; }
    }
    {
        int64_t q1 = t5_warp_append(&A.totals[1], (uint32_t)__popc(critE));
        for (uint32_t m = critE; m; m &= m - 1, q1++) {
            const int s = __ffs(m) - 1;
            if (q1 < A.cap[1]) {
                const int64_t anc = v + T.e_anc[s][0] + (int64_t)A.Lx * T.e_anc[s][1] + LxLy * T.e_anc[s][2];
                A.crit_id[1][q1] = 6 * anc + T.e_k[s];
                A.crit_key[1][q1] = rkey | t5_key(rk(s), -1, -1);
            }
        }
    }
    {
        int64_t q2 = t5_warp_append(&A.totals[2], (uint32_t)__popcll(critT));
        for (uint64_t m = critT; m; m &= m - 1, q2++) {
            const int t = __ffsll((long long)m) - 1;
            if (q2 < A.cap[2]) {
                const int a = rk(T.tri_a[t]), b = rk(T.tri_b[t]);
                const int64_t anc = v + T.t_anc[t][0] + (int64_t)A.Lx * T.t_anc[t][1] + LxLy * T.t_anc[t][2];
                A.crit_id[2][q2] = 10 * anc + T.t_k[t];
                A.crit_key[2][q2] = rkey | t5_key(max(a, b), min(a, b), -1);
            }
        }
    }
    {
        int64_t q3 = t5_warp_append(&A.totals[3], (uint32_t)__popc(critQ));
        for (uint32_t m = critQ; m; m &= m - 1, q3++) {
            const int q = __ffs(m) - 1;
            if (q3 < A.cap[3]) {
                const int a = rk(T.tet_a[q]), b = rk(T.tet_b[q]), c = rk(T.tet_c[q]);
                const int hi = max(a, max(b, c)), lo = min(a, min(b, c));
                const int64_t anc = v + T.q_anc[q][0] + (int64_t)A.Lx * T.q_anc[q][1] + LxLy * T.q_anc[q][2];
                A.crit_id[3][q3] = 5 * anc + T.q_k[q];
                A.crit_key[3][q3] = rkey | t5_key(hi, a + b + c - hi - lo, lo);
            }
        }
    }
}

// ------------------------------------------------------------------ D0 / D2 tracing

// D0 (Sec. 5.1, PAPER.md 2494-2621): from a vertex follow the vertex -> edge vectors down
// to a minimum (vertex code = star slot of the paired edge; 0xFF = minimum)
__device__ __forceinline__ int64_t t5_descend(const T5Geo& g, const T5Tab* __restrict__ tab, const uint8_t* __restrict__ grad,
                                              int64_t v, int x, int y, int z) {
    for (;;) {
        const int code = (int)__ldg(grad + v);
        if (code == 0xff) return v;
        const int8_t* o = tab->star[(x + y + z) & 1].off[code];
        x += o[0];
        y += o[1];
        z += o[2];
        v += o[0] + (int64_t)g.Lx * o[1] + (int64_t)g.Lx * g.Ly * o[2];
    }
}

__global__ void k_d0_arcs_t5(T5Geo g, const T5Tab* __restrict__ tab, const uint8_t* __restrict__ grad,
                             const int64_t* __restrict__ c1, int64_t m, const int32_t* __restrict__ node_of0,
                             int32_t* __restrict__ arc_a, int32_t* __restrict__ arc_b) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t id = c1[i];
    const int64_t a = id / 6;
    const int k = (int)(id % 6);
    const int ax = (int)(a % g.Lx), ay = (int)((a / g.Lx) % g.Ly), az = (int)(a / ((int64_t)g.Lx * g.Ly));
    const uint8_t* mk = tab->ids[(ax + ay + az) & 1][1][k];
    int32_t out[2];
    for (int j = 0; j < 2; j++) {
        const int mm = mk[j];
        const int x = ax + (mm & 1), y = ay + ((mm >> 1) & 1), z = az + ((mm >> 2) & 1);
        const int64_t v = x + (int64_t)g.Lx * (y + (int64_t)g.Ly * z);
        out[j] = node_of0[t5_descend(g, tab, grad, v, x, y, z)];
    }
    arc_a[i] = out[0];
    arc_b[i] = out[1];
}

// D2 (Sec. 5.2, PAPER.md 2728-2825): from each cofacet tetrahedron of a critical triangle
// follow the dual gradient (a tetrahedron paired with its facet j continues into the other
// tetrahedron of that facet) to a critical tetrahedron, or to the virtual maximum when the
// path leaves through the boundary.  Two jobs per triangle (ids in emission order).
__global__ void k_dtop_arcs_t5(T5Geo g, const T5Tab* __restrict__ tab, const uint8_t* __restrict__ grad,
                               const int64_t* __restrict__ c2, int64_t m, const int32_t* __restrict__ node_of,
                               int32_t vnode, int32_t* __restrict__ arc_a, int32_t* __restrict__ arc_b) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= 2 * m) return;
    const int64_t i = j >> 1;
    const int side = (int)(j & 1);
    const int64_t id = c2[i];
    const int64_t a = id / 10;
    const int k = (int)(id % 10);
    int cx = (int)(a % g.Lx), cy = (int)((a / g.Lx) % g.Ly), cz = (int)(a / ((int64_t)g.Lx * g.Ly));
    int p = (cx + cy + cz) & 1;
    const uint8_t e = tab->tri_cof[p][k][side];
    int32_t res = vnode;
    if (e != 0xff) {
        int dx, dy, dz;
        t5_dir(e >> 4, dx, dy, dz);
        cx += dx;
        cy += dy;
        cz += dz;
        p ^= (dx | dy | dz) ? 1 : 0;
        int q = e & 15;
        const int64_t LxLy = (int64_t)g.Lx * g.Ly;
        const uint8_t* qcode = grad + 11 * g.N;
        while (t5_cube_ok(g, cx, cy, cz)) {
            const int64_t tid = 5 * (cx + (int64_t)g.Lx * cy + LxLy * cz) + q;
            const int code = (int)__ldg(qcode + tid);
            if (code == 0xff) { res = node_of[tid]; break; }
            const uint8_t nb = tab->tet_nbr[p][q][code];
            t5_dir(nb >> 4, dx, dy, dz);
            cx += dx;
            cy += dy;
            cz += dz;
            p ^= (dx | dy | dz) ? 1 : 0;
            q = nb & 15;
        }
    }
    (side ? arc_b : arc_a)[i] = res;
}

// highest vertex (in K) of an anchored simplex of the five-tetrahedra complex
__device__ __forceinline__ int64_t t5_max_vertex(const float* f, int32_t Lx, int32_t Ly, const T5Tab* tab, int dim,
                                                 int64_t id) {
    if (dim == 0) return id;
    const int64_t per = dim == 1 ? 6 : dim == 2 ? 10 : 5;
    const int64_t a = id / per;
    const int k = (int)(id % per);
    const int ax = (int)(a % Lx), ay = (int)((a / Lx) % Ly), az = (int)(a / ((int64_t)Lx * Ly));
    const uint8_t* mk = tab->ids[(ax + ay + az) & 1][dim][k];
    int64_t best = -1;
    uint32_t ob = 0;
    for (int j = 0; j <= dim; j++) {
        const int mm = mk[j];
        const int64_t p = a + (mm & 1) + (int64_t)Lx * ((mm >> 1) & 1) + (int64_t)Lx * Ly * ((mm >> 2) & 1);
        const uint32_t op = ord_of(__ldg(f + p));
        if (best < 0 || k_less(ob, best, op, p)) { best = p; ob = op; }
    }
    return best;
}

}  // namespace dms
