// star_build.cuh -- host construction of the star tables (see star.cuh).
#pragma once
#include <algorithm>
#include <array>
#include <functional>
#include <cstring>
#include <vector>

#include "star.cuh"

namespace dms {

namespace detail {

using P3 = std::array<int, 3>;

inline int popcount3(int m) { return (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1); }

// {points} (all distinct, containing 0 or not) spans a Freudenthal simplex iff, sorted
// by coordinate sum, consecutive points increase component-wise and the span
// (last - first) is a 0/1 vector.
inline bool is_kuhn_simplex(std::vector<P3> pts) {
    std::sort(pts.begin(), pts.end(), [](const P3& a, const P3& b) {
        return a[0] + a[1] + a[2] < b[0] + b[1] + b[2];
    });
    for (size_t i = 1; i < pts.size(); i++) {
        int s0 = pts[i - 1][0] + pts[i - 1][1] + pts[i - 1][2], s1 = pts[i][0] + pts[i][1] + pts[i][2];
        if (s1 == s0) return false;
        for (int ax = 0; ax < 3; ax++)
            if (pts[i][ax] < pts[i - 1][ax]) return false;
    }
    for (int ax = 0; ax < 3; ax++) {
        int d = pts.back()[ax] - pts.front()[ax];
        if (d < 0 || d > 1) return false;
    }
    return true;
}

// chains S_1 < ... < S_k of non-empty axis subsets of {0..ndim-1}, sorted by
// (S_k, ..., S_1) ascending -- the chain index convention of anchored ids
inline std::vector<std::vector<int>> chains(int ndim, int k) {
    std::vector<std::vector<int>> out;
    const int full = (1 << ndim) - 1;
    std::vector<int> cur;
    std::function<void(int)> rec = [&](int prev) {
        if ((int)cur.size() == k) { out.push_back(cur); return; }
        for (int m = 1; m <= full; m++) {
            if ((m & prev) != prev || m == prev) continue;
            cur.push_back(m);
            rec(m);
            cur.pop_back();
        }
    };
    rec(0);
    std::sort(out.begin(), out.end(), [](const std::vector<int>& a, const std::vector<int>& b) {
        for (int j = (int)a.size() - 1; j >= 0; j--)
            if (a[j] != b[j]) return a[j] < b[j];
        return false;
    });
    return out;
}

// anchor offset (relative to the first point, which is the star centre 0) and chain
// index of the simplex spanned by pts
inline void anchor_and_index(int ndim, const std::vector<P3>& pts, int8_t anc[3], uint8_t* kidx) {
    P3 a = pts[0];
    for (auto& p : pts)
        for (int ax = 0; ax < 3; ax++) a[ax] = std::min(a[ax], p[ax]);
    std::vector<int> masks;
    for (auto& p : pts) {
        int m = 0;
        for (int ax = 0; ax < 3; ax++)
            if (p[ax] - a[ax] == 1) m |= 1 << ax;
        masks.push_back(m);
    }
    std::sort(masks.begin(), masks.end(), [](int x, int y) { return popcount3(x) < popcount3(y); });
    std::vector<int> ch(masks.begin() + 1, masks.end());
    auto all = chains(ndim, (int)ch.size());
    int idx = -1;
    for (size_t i = 0; i < all.size(); i++)
        if (all[i] == ch) idx = (int)i;
    for (int ax = 0; ax < 3; ax++) anc[ax] = (int8_t)a[ax];
    *kidx = (uint8_t)idx;
}

}  // namespace detail

inline bool build_star_tables(int ndim, const int64_t L[3], StarTab* T) {
    using namespace detail;
    std::memset(T, 0, sizeof(StarTab));
    std::memset(T->tri_tet, 255, sizeof(T->tri_tet));
    std::memset(T->edge_tri, 255, sizeof(T->edge_tri));
    std::memset(T->e_slot, 255, sizeof(T->e_slot));
    std::memset(T->t_slot, 255, sizeof(T->t_slot));
    std::memset(T->q_slot, 255, sizeof(T->q_slot));
    T->ndim = ndim;
    // neighbours: non-zero vectors of {-1,0,1}^ndim whose non-zero entries share a sign
    std::vector<P3> nb;
    for (int dz = (ndim > 2 ? -1 : 0); dz <= (ndim > 2 ? 1 : 0); dz++)
        for (int dy = (ndim > 1 ? -1 : 0); dy <= (ndim > 1 ? 1 : 0); dy++)
            for (int dx = -1; dx <= 1; dx++) {
                P3 p{dx, dy, dz};
                bool pos = false, neg = false;
                for (int ax = 0; ax < 3; ax++) { pos |= p[ax] > 0; neg |= p[ax] < 0; }
                if ((pos || neg) && !(pos && neg)) nb.push_back(p);
            }
    // slots by linear index offset == (dz, dy, dx) lexicographic for extents >= 2
    std::sort(nb.begin(), nb.end(), [](const P3& a, const P3& b) {
        if (a[2] != b[2]) return a[2] < b[2];
        if (a[1] != b[1]) return a[1] < b[1];
        return a[0] < b[0];
    });
    T->ne = (int)nb.size();
    for (int s = 0; s < T->ne; s++) {
        for (int ax = 0; ax < 3; ax++) T->off[s][ax] = (int8_t)nb[s][ax];
        T->lin[s] = (int32_t)(nb[s][0] + L[0] * nb[s][1] + L[0] * L[1] * nb[s][2]);
    }
    const P3 zero{0, 0, 0};
    // triangles of the star = pairs of neighbours forming a simplex with the centre
    int nt = 0;
    for (int a = 0; a < T->ne; a++)
        for (int b = a + 1; b < T->ne; b++)
            if (ndim >= 2 && is_kuhn_simplex({zero, nb[a], nb[b]})) {
                T->tri_a[nt] = (uint8_t)a;
                T->tri_b[nt] = (uint8_t)b;
                nt++;
            }
    T->nt = nt;
    std::memset(T->tri_of, 255, sizeof(T->tri_of));
    for (int t = 0; t < nt; t++) {
        T->tri_of[T->tri_a[t]][T->tri_b[t]] = (uint8_t)t;
        T->tri_of[T->tri_b[t]][T->tri_a[t]] = (uint8_t)t;
        T->adj[T->tri_a[t]] |= (uint16_t)(1u << T->tri_b[t]);
        T->adj[T->tri_b[t]] |= (uint16_t)(1u << T->tri_a[t]);
    }
    for (int hi = 1; hi < kMaxNE; hi++)
        for (int lo = 0; lo < hi; lo++) T->hl[hi * (hi - 1) / 2 + lo] = (uint8_t)(hi << 4 | lo);
    int nq = 0;
    for (int a = 0; a < T->ne; a++)
        for (int b = a + 1; b < T->ne; b++)
            for (int c = b + 1; c < T->ne; c++)
                if (ndim >= 3 && is_kuhn_simplex({zero, nb[a], nb[b], nb[c]})) {
                    T->tet_a[nq] = (uint8_t)a;
                    T->tet_b[nq] = (uint8_t)b;
                    T->tet_c[nq] = (uint8_t)c;
                    nq++;
                }
    T->nq = nq;
    if (ndim == 3 && (T->ne != 14 || nt != 36 || nq != 24)) return false;
    if (ndim == 2 && (T->ne != 6 || nt != 6)) return false;
    if (ndim == 1 && T->ne != 2) return false;
    auto tri_of = [&](int a, int b) {
        if (a > b) std::swap(a, b);
        for (int t = 0; t < nt; t++)
            if (T->tri_a[t] == a && T->tri_b[t] == b) return t;
        return -1;
    };
    for (int q = 0; q < nq; q++) {
        int tr[3] = {tri_of(T->tet_a[q], T->tet_b[q]), tri_of(T->tet_a[q], T->tet_c[q]), tri_of(T->tet_b[q], T->tet_c[q])};
        for (int j = 0; j < 3; j++) {
            if (tr[j] < 0) return false;
            T->tet_tri[q][j] = (uint8_t)tr[j];
            T->tet_tmask[q] |= 1ull << tr[j];
            int t = tr[j];
            if (T->tri_tet[t][0] == 255) T->tri_tet[t][0] = (uint8_t)q;
            else if (T->tri_tet[t][1] == 255) T->tri_tet[t][1] = (uint8_t)q;
            else return false;
            T->tri_tet_mask[t] |= 1u << q;
        }
        T->tet_amask[T->tet_a[q]] |= 1u << q;
        T->tet_bmask[T->tet_b[q]] |= 1u << q;
        T->tet_cmask[T->tet_c[q]] |= 1u << q;
    }
    for (int t = 0; t < nt; t++) {
        for (int e : {(int)T->tri_a[t], (int)T->tri_b[t]}) {
            int j = 0;
            while (j < 6 && T->edge_tri[e][j] != 255) j++;
            if (j == 6) return false;
            T->edge_tri[e][j] = (uint8_t)t;
            T->edge_tri_mask[e] |= 1ull << t;
        }
        T->tri_amask[T->tri_a[t]] |= 1ull << t;
        T->tri_bmask[T->tri_b[t]] |= 1ull << t;
    }
    // anchored ids of star cells and the inverse (chain index, centre position) -> slot
    for (int k = 1; k <= ndim; k++) {
        auto ch = chains(ndim, k);
        T->nchain[k] = (int)ch.size();
        for (size_t i = 0; i < ch.size(); i++)
            for (int j = 0; j < k; j++) T->chain[k][i][j] = (uint8_t)ch[i][j];
    }
    T->nchain[0] = 1;
    auto bits = [](int m) { return P3{m & 1, (m >> 1) & 1, (m >> 2) & 1}; };
    auto sub = [](const P3& a, const P3& b) { return P3{a[0] - b[0], a[1] - b[1], a[2] - b[2]}; };
    for (int s = 0; s < T->ne; s++) anchor_and_index(ndim, {zero, nb[s]}, T->e_anc[s], &T->e_k[s]);
    for (int t = 0; t < nt; t++) anchor_and_index(ndim, {zero, nb[T->tri_a[t]], nb[T->tri_b[t]]}, T->t_anc[t], &T->t_k[t]);
    for (int q = 0; q < nq; q++)
        anchor_and_index(ndim, {zero, nb[T->tet_a[q]], nb[T->tet_b[q]], nb[T->tet_c[q]]}, T->q_anc[q], &T->q_k[q]);
    auto find_slot = [&](const std::vector<P3>& rel) -> int {  // rel: offsets of the other vertices
        auto same = [&](std::vector<int> idx) {
            std::vector<P3> a;
            for (int s : idx) a.push_back(nb[s]);
            auto key = [](std::vector<P3> v) { std::sort(v.begin(), v.end()); return v; };
            return key(a) == key(rel);
        };
        if (rel.size() == 1) { for (int s = 0; s < T->ne; s++) if (same({s})) return s; }
        if (rel.size() == 2) { for (int t = 0; t < nt; t++) if (same({T->tri_a[t], T->tri_b[t]})) return t; }
        if (rel.size() == 3) { for (int q = 0; q < nq; q++) if (same({T->tet_a[q], T->tet_b[q], T->tet_c[q]})) return q; }
        return -1;
    };
    // the same cell seen from one of its link vertices
    std::memset(T->q_reslot, 255, sizeof(T->q_reslot));
    std::memset(T->t_reslot, 255, sizeof(T->t_reslot));
    for (int q = 0; q < nq; q++) {
        const int ls[3] = {T->tet_a[q], T->tet_b[q], T->tet_c[q]};
        for (int j = 0; j < 3; j++) {
            std::vector<P3> rel;
            rel.push_back(sub(zero, nb[ls[j]]));
            for (int i = 0; i < 3; i++) if (i != j) rel.push_back(sub(nb[ls[i]], nb[ls[j]]));
            const int r = find_slot(rel);
            if (r < 0) return false;
            T->q_reslot[q][j] = (uint8_t)r;
        }
    }
    for (int t = 0; t < nt; t++) {
        const int ls[2] = {T->tri_a[t], T->tri_b[t]};
        for (int j = 0; j < 2; j++) {
            std::vector<P3> rel;
            rel.push_back(sub(zero, nb[ls[j]]));
            rel.push_back(sub(nb[ls[1 - j]], nb[ls[j]]));
            const int r = find_slot(rel);
            if (r < 0) return false;
            T->t_reslot[t][j] = (uint8_t)r;
        }
    }
    for (int k = 1; k <= ndim; k++) {
        for (int i = 0; i < T->nchain[k]; i++) {
            std::vector<P3> pts{zero};
            for (int j = 0; j < k; j++) pts.push_back(bits(T->chain[k][i][j]));
            for (int jc = 0; jc <= k; jc++) {
                std::vector<P3> rel;
                for (int j = 0; j <= k; j++)
                    if (j != jc) rel.push_back(sub(pts[j], pts[jc]));
                int s = find_slot(rel);
                if (s < 0) return false;
                if (k == 1) T->e_slot[i][jc] = (uint8_t)s;
                if (k == 2) T->t_slot[i][jc] = (uint8_t)s;
                if (k == 3) T->q_slot[i][jc] = (uint8_t)s;
            }
        }
    }
    return true;
}


// the dual-chase transition table (see star.cuh ChaseTab)
inline void build_grad_lut(const StarTab& T, GradLut* G) {
    std::memset(G, 0, sizeof(GradLut));
    for (int h = 0; h < 2; h++)
        for (int m = 0; m < 128; m++)
            for (int b = 0; b < 7; b++)
                if ((m >> b) & 1) {
                    const int s = 7 * h + b;
                    if (s >= T.ne) continue;
                    G->ort[h][m] |= T.tri_amask[s] | T.tri_bmask[s];
                    G->orq[h][m] |= T.tet_amask[s] | T.tet_bmask[s] | T.tet_cmask[s];
                }
    for (int m = 0; m < 128; m++)
        for (int b = 0; b < 7; b++)
            if ((m >> b) & 1) G->ex[m] |= 1u << (4 * b);
    for (int q = 0; q < T.nq; q++) {
        G->tet_nb[q] = 0;
        for (int j = 0; j < 3; j++) {
            const int t = T.tet_tri[q][j];
            for (int m = 0; m < 16; m++)
                if ((m >> (t & 3)) & 1) (j == 0 ? G->gat[t >> 2][m].x : j == 1 ? G->gat[t >> 2][m].y : G->gat[t >> 2][m].z) |= 1u << q;
            const int o = T.tri_tet[t][0] == q ? T.tri_tet[t][1] : T.tri_tet[t][0];
            G->tet_nb[q] |= (uint32_t)(o == 255 ? 31 : o) << (8 * j);
        }
    }
}

inline void build_chase_tables(const StarTab& T, ChaseTab* C) {
    // one-lookup transitions of the ascending dual chase (diag.cuh chase_step): top cell
    // T paired with its facet #c -> the other cofacet T2 of that facet in this star
    // (255: none), the slot s2 of T2's vertex off the facet, and T2 seen from s2
    std::memset(C->q_next, 255, sizeof(C->q_next));
    std::memset(C->t_next, 255, sizeof(C->t_next));
    if (T.ndim == 3) {
        for (int q = 0; q < T.nq; q++)
            for (int c = 0; c < 3; c++) {
                const int tt = T.tet_tri[q][c];
                const int T2 = T.tri_tet[tt][0] == q ? T.tri_tet[tt][1] : T.tri_tet[tt][0];
                if (T2 == 255) { C->q_next[q][c] = 0xffffffu; continue; }
                const int s2 = T.tet_a[T2] ^ T.tet_b[T2] ^ T.tet_c[T2] ^ T.tri_a[tt] ^ T.tri_b[tt];
                const int j = T.tet_a[T2] == s2 ? 0 : (T.tet_b[T2] == s2 ? 1 : 2);
                C->q_next[q][c] = (uint32_t)T2 | ((uint32_t)s2 << 8) | ((uint32_t)T.q_reslot[T2][j] << 16);
            }
    }
    if (T.ndim == 2) {
        for (int t = 0; t < T.nt; t++)
            for (int c = 0; c < 2; c++) {
                const int e = c == 0 ? T.tri_a[t] : T.tri_b[t];
                const int T2 = T.edge_tri[e][0] == t ? T.edge_tri[e][1] : T.edge_tri[e][0];
                if (T2 == 255) { C->t_next[t][c] = 0xffffffu; continue; }
                const int s2 = T.tri_a[T2] ^ T.tri_b[T2] ^ e;
                const int j = T.tri_a[T2] == s2 ? 0 : 1;
                C->t_next[t][c] = (uint32_t)T2 | ((uint32_t)s2 << 8) | ((uint32_t)T.t_reslot[T2][j] << 16);
            }
    }
}

}  // namespace dms
