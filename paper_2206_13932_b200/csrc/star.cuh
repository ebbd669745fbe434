// star.cuh -- the star of a vertex in the Freudenthal triangulation, as small tables.
//
// PAPER.md 1360-1366 (Sec. 2.1): grids are triangulated by the Freudenthal (Kuhn)
// scheme, giving the 6-vertex (2D) / 14-vertex (3D) neighbourhood.  A set of lattice
// points {0, o_1, ..., o_k} spans a simplex of that triangulation iff, sorted by
// coordinate sum, the points increase component-wise and the last minus the first is
// a 0/1 vector.  The tables below are derived from that rule on the host at context
// creation (no enumeration is shared with the oracle).
//
// Slots: the neighbours n_s = x + off[s] are numbered by increasing linear index
// offset, so for equal values the index tie-break of K is a slot comparison:
//   K(n_s) < K(n_t) <=> f_s < f_t or (f_s == f_t and s < t), and x sits between slot
//   NE/2-1 and NE/2.
// Star cells of x: edge (x, n_s) = slot s; triangle (x, n_a, n_b) = "tri slot";
// tetrahedron (x, n_a, n_b, n_c) = "tet slot".
#pragma once
#include <cstdint>

namespace dms {

constexpr int kMaxNE = 14, kMaxNT = 36, kMaxNQ = 24;

struct alignas(16) StarTab {
    int ndim, ne, nt, nq;
    int8_t off[kMaxNE][3];
    int32_t lin[kMaxNE];              // linear index offsets for the grid
    uint8_t tri_a[kMaxNT], tri_b[kMaxNT];                 // neighbour slots, a < b
    uint8_t tet_a[kMaxNQ], tet_b[kMaxNQ], tet_c[kMaxNQ];  // a < b < c
    uint8_t tet_tri[kMaxNQ][3];       // tri slots (a,b), (a,c), (b,c)
    uint8_t tri_tet[kMaxNT][2];       // tet slots containing the tri (255: none)
    uint8_t edge_tri[kMaxNE][6];      // tri slots containing edge s (255: none)
    uint64_t edge_tri_mask[kMaxNE];   // same as a mask over tri slots
    uint32_t tri_tet_mask[kMaxNT];    // tet slots containing the tri
    uint64_t tri_amask[kMaxNE], tri_bmask[kMaxNE];  // tri slots whose a (b) end is slot s
    uint32_t tet_amask[kMaxNE], tet_bmask[kMaxNE], tet_cmask[kMaxNE];
    uint8_t tri_of[kMaxNE][kMaxNE];   // (slot a, slot b) -> tri slot (255: not a triangle)
    uint8_t hl[96];                   // triangle key index C(hi,2)+lo -> hi << 4 | lo
    uint64_t tet_tmask[kMaxNQ];       // the 3 triangle slots of a tet slot, as a mask
    uint16_t adj[kMaxNE];             // link adjacency: slots u with (x, n_s, n_u) a triangle
    uint8_t q_reslot[kMaxNQ][3];      // tet slot T seen from its link vertex j (a,b,c) -> slot there
    uint8_t t_reslot[kMaxNT][2];      // tri slot t seen from its link vertex j (a,b) -> slot there
    // anchored ids of star cells: anchor offset from x and chain index
    int8_t e_anc[kMaxNE][3];  uint8_t e_k[kMaxNE];
    int8_t t_anc[kMaxNT][3];  uint8_t t_k[kMaxNT];
    int8_t q_anc[kMaxNQ][3];  uint8_t q_k[kMaxNQ];
    // chain index k and position j of the star centre inside the chain -> slot
    uint8_t e_slot[7][2];     // edges:     7 chains x 2 positions
    uint8_t t_slot[12][3];    // triangles
    uint8_t q_slot[6][4];     // tetrahedra
    // chains per dimension: masks S_1..S_k (x=1,y=2,z=4) of chain index k
    uint8_t chain[4][12][3];
    int nchain[4];
};

// One-lookup transitions of the ascending dual chase (diag.cuh chase_step), kept out of
// StarTab so the gradient kernels' shared-memory copy stays small: top cell T paired
// with its facet #c -> T2 | s2 << 8 | (T2 seen from s2) << 16 (T2 = 255: no other
// cofacet of that facet in this star).
struct alignas(16) ChaseTab {
    uint32_t q_next[kMaxNQ][3];  // 3D: tetrahedra
    uint32_t t_next[kMaxNT][2];  // 2D: triangles
};

// 3D gradient kernel: masks that are unions over a set of link vertices, looked up by the
// two 7-bit halves of the set (slots 0-6, 7-13) and OR-ed: ort / orq = the star triangles
// / tetrahedra holding any of the vertices; ex = bit i -> bit 4 i (a nibble per slot).
// gat: the forest triangles T (a set of star triangles) -> per star tetrahedron, which of
// its three triangles tet_tri[q][j] are in T: nibble i of T with value m contributes
// gat[i][m][j] (a mask over tetrahedra).  tet_nb: byte j = the other tetrahedron holding
// the triangle tet_tri[q][j] (31: none).
struct alignas(16) Gat4 { uint32_t x, y, z, w; };
struct alignas(16) GradLut {
    uint64_t ort[2][128];
    uint32_t orq[2][128];
    uint32_t ex[128];
    Gat4 gat[9][16];
    uint32_t tet_nb[kMaxNQ];
};
inline void build_grad_lut(const StarTab& T, GradLut* G);

// Build the tables for a grid (host).  Returns false if something is inconsistent.
bool build_star_tables(int ndim, const int64_t L[3], StarTab* T);
inline void build_chase_tables(const StarTab& T, ChaseTab* C);

}  // namespace dms
