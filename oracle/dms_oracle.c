/*
 * dms_oracle.c -- plain, slow, obviously-correct CPU oracle for the DMS front end.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2206_13932_b200/).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (arXiv 2206.13932), S:n = SPEC.md line n.
 * Readings of silent/ambiguous passages are listed in DESIGN.md ("Readings", Z1..Z17).
 *
 * What it computes (every step in the paper's order and notation):
 *   O1 vertex order      -- injective order K(v) = (f(v), v)
 *   O2 complex           -- Freudenthal/Kuhn triangulation, explicit
 *   O3 gradient          -- Robins et al. ProcessLowerStars per vertex P:1965-1971
 *   O4 C_k               -- Alg. 2 "zero-persistence skip", lex sort
 *   O5 D0                -- Sec. 5.1 unstable sets + Union-Find
 *   O6 D_{d-1}           -- Sec. 5.2 dual gradient, stable sets, UF in decreasing
 *                           order, virtual maximum on the boundary
 *                           ("ignore" mode: boundary arcs dropped)
 *   O8 infinite classes  -- Sec. 6
 *   O2' complex (3D)     -- five tetrahedra per cube, the subdivision of the paper's
 *                           benchmarks                                 P:662-664 (Sec. 8.1)
 *
 * Parity pins: tests/test_oracle_pins.py (hand-built fields, SPEC examples, Euler
 * characteristic, gradient validity, Robins' guarantee, brute-force Kruskal and
 * boundary-matrix reduction written independently in tests/brute.py).
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>
#include <time.h>

/* ------------------------------------------------------------------ grid + order */

typedef struct {
    int ndim;
    int64_t L[3];      /* extents, unused axes = 1 */
    int64_t N;
    const float *f;
    int64_t ncell[4];  /* anchored cells per vertex for each simplex dimension */
    int cplx;          /* 0: Freudenthal (Kuhn) triangulation; 1: five tetrahedra per cube (3D) */
} grid;

/* K(u) < K(v): compare values (IEEE <, so -0 == +0), break ties by vertex index.
 * P:1368-1372 ("symbolic perturbation inspired from Simulation of Simplicity"),
 * readings Z2/Z3. */
static inline int klt(const grid *g, int64_t u, int64_t v)
{
    float a = g->f[u], b = g->f[v];
    if (a < b) return 1;
    if (a > b) return 0;
    return u < v;
}

static inline void coords(const grid *g, int64_t v, int64_t c[3])
{
    c[0] = v % g->L[0];
    c[1] = (v / g->L[0]) % g->L[1];
    c[2] = v / (g->L[0] * g->L[1]);
}

static inline int64_t vid(const grid *g, const int64_t c[3])
{
    return c[0] + g->L[0] * (c[1] + g->L[1] * c[2]);
}

/* ------------------------------------------------------------------ simplices */

/* A simplex as its vertex list sorted by decreasing K (v[0] = highest vertex),
 * the representation the lexicographic comparison of P:1380-1414 works on. */
typedef struct {
    int dim;
    int64_t v[4];
} simp;

static void simp_sort(const grid *g, simp *s)
{
    for (int i = 1; i <= s->dim; i++)
        for (int j = i; j > 0 && klt(g, s->v[j - 1], s->v[j]); j--) {
            int64_t t = s->v[j]; s->v[j] = s->v[j - 1]; s->v[j - 1] = t;
        }
}

/* Lexicographic comparison: compare the decreasing vertex sequences
 * element by element; if one is a prefix of the other (a face), it is smaller. */
static int lexcmp(const grid *g, const simp *a, const simp *b)
{
    int m = a->dim < b->dim ? a->dim : b->dim;
    for (int i = 0; i <= m; i++) {
        if (a->v[i] != b->v[i]) return klt(g, a->v[i], b->v[i]) ? -1 : 1;
    }
    return a->dim - b->dim;
}

static int simp_eq(const simp *a, const simp *b)
{
    if (a->dim != b->dim) return 0;
    for (int i = 0; i <= a->dim; i++) if (a->v[i] != b->v[i]) return 0;
    return 1;
}

/* is a a facet of b (dimension one less, vertex subset)? */
static int is_facet(const simp *a, const simp *b)
{
    if (a->dim + 1 != b->dim) return 0;
    for (int i = 0; i <= a->dim; i++) {
        int found = 0;
        for (int j = 0; j <= b->dim; j++) if (a->v[i] == b->v[j]) { found = 1; break; }
        if (!found) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------ anchored ids
 * Reading Z13: a k-simplex of the Kuhn triangulation is a chain
 * 0 = S_0 < S_1 < ... < S_k of axis subsets (bit masks x=1, y=2, z=4) translated by
 * its anchor a (component-wise minimum vertex).  Its id is ncell[k] * vid(a) + idx,
 * idx = position of (S_k, ..., S_1) among all such chains sorted ascending.
 * The table of chains is enumerated here by brute force. */

static int chain_count[4][4];     /* [ndim][k]                                     */
static int chain_ndim_built = 0;  /* bit mask of ndims built                        */
static int chain_tab[4][4][16][3];/* [ndim][k][idx][j]                              */

static int popc(int m) { int c = 0; while (m) { c += m & 1; m >>= 1; } return c; }

static int chain_cmp_desc(const int *a, const int *b, int k)
{
    for (int j = k - 1; j >= 0; j--) if (a[j] != b[j]) return a[j] < b[j] ? -1 : 1;
    return 0;
}

static void build_chains(int ndim)
{
    if (chain_ndim_built & (1 << ndim)) return;
    int full = (1 << ndim) - 1;
    for (int k = 1; k <= ndim; k++) {
        int n = 0;
        int cand[64][3];
        /* all strictly increasing chains of k non-empty subsets of the axis set */
        for (int s1 = 1; s1 <= full; s1++) {
            if (k == 1) { cand[n][0] = s1; n++; continue; }
            for (int s2 = 1; s2 <= full; s2++) {
                if ((s1 & s2) != s1 || s1 == s2) continue;
                if (k == 2) { cand[n][0] = s1; cand[n][1] = s2; n++; continue; }
                for (int s3 = 1; s3 <= full; s3++) {
                    if ((s2 & s3) != s2 || s2 == s3) continue;
                    cand[n][0] = s1; cand[n][1] = s2; cand[n][2] = s3; n++;
                }
            }
        }
        /* sort by (S_k, ..., S_1) ascending (insertion sort, n <= 12) */
        for (int i = 1; i < n; i++)
            for (int j = i; j > 0 && chain_cmp_desc(cand[j], cand[j - 1], k) < 0; j--) {
                int t[3]; memcpy(t, cand[j], sizeof t); memcpy(cand[j], cand[j - 1], sizeof t);
                memcpy(cand[j - 1], t, sizeof t);
            }
        for (int i = 0; i < n; i++) memcpy(chain_tab[ndim][k][i], cand[i], sizeof cand[i]);
        chain_count[ndim][k] = n;
    }
    chain_ndim_built |= 1 << ndim;
}

/* ------------------------------------------------------------------ five-tetrahedra complex
 * P:662-664 (Sec. 8.1): the paper's 3D benchmark volumes are "triangulated into a
 * simplicial complex by breaking up each cell into ... five tetrahedra".  Reading Z21
 * (DESIGN.md): the cube with minimum corner a, parity p = (ax + ay + az) mod 2, is cut
 * into the central tetrahedron on its four corners c (local offsets, bit masks x=1,
 * y=2, z=4) with popcount(c) + p even, and the four corner tetrahedra {o, o^1, o^2, o^4}
 * at its other four corners o.  The central corners are the vertices of even coordinate
 * sum in every cube, so each square face is cut along the diagonal joining its two
 * even-sum corners from both sides: the cubes fit together (a conforming complex).
 *
 * Ids (reading Z21): a k-simplex is anchored at its component-wise minimum a (not
 * necessarily one of its vertices); its id is t5_count[k] * vid(a) + idx, idx = the
 * position of its vertex offsets from a (ascending masks) among all k-simplices of the
 * cube at a with component-wise minimum a, for a's parity, sorted ascending as tuples. */

static int t5_built = 0;
static int t5_count[4];              /* cells per anchor: 1, 6, 10, 5 */
static int t5_tab[2][4][16][4];      /* [parity][k][idx][j]: ascending vertex masks */

/* the five tetrahedra of a cube of parity p, as local corner masks */
static void t5_cube_tets(int p, int tets[5][4])
{
    int nc = 0, nt = 1;
    for (int c = 0; c < 8; c++)
        if (((popc(c) + p) & 1) == 0) tets[0][nc++] = c;                 /* central */
        else { tets[nt][0] = c; tets[nt][1] = c ^ 1; tets[nt][2] = c ^ 2; tets[nt][3] = c ^ 4; nt++; }
}

static int cmp_int(const void *a, const void *b) { return *(const int *)a - *(const int *)b; }

static void build_t5(void)
{
    if (t5_built) return;
    for (int p = 0; p < 2; p++) {
        int tets[5][4];
        t5_cube_tets(p, tets);
        for (int k = 1; k <= 3; k++) {
            int n = 0, cand[16][4];
            for (int t = 0; t < 5; t++)
                for (int sub = 1; sub < 16; sub++) {
                    if (popc(sub) != k + 1) continue;
                    int m[4], q = 0, andm = 7;
                    for (int j = 0; j < 4; j++) if ((sub >> j) & 1) { m[q++] = tets[t][j]; andm &= tets[t][j]; }
                    if (andm != 0) continue;            /* anchored elsewhere */
                    qsort(m, k + 1, sizeof(int), cmp_int);
                    int dup = 0;
                    for (int i = 0; i < n && !dup; i++) dup = !memcmp(cand[i], m, (k + 1) * sizeof(int));
                    if (!dup) { memcpy(cand[n], m, (k + 1) * sizeof(int)); n++; }
                }
            /* ascending tuples (insertion sort, n <= 10) */
            for (int i = 1; i < n; i++)
                for (int j = i; j > 0; j--) {
                    int c = 0;
                    for (int u = 0; u <= k && !c; u++) c = cand[j][u] - cand[j - 1][u];
                    if (c >= 0) break;
                    int t[4]; memcpy(t, cand[j], sizeof t); memcpy(cand[j], cand[j - 1], sizeof t);
                    memcpy(cand[j - 1], t, sizeof t);
                }
            if (p == 1 && n != t5_count[k]) abort();  /* both parities have the same counts */
            t5_count[k] = n;
            for (int i = 0; i < n; i++) memcpy(t5_tab[p][k][i], cand[i], sizeof cand[i]);
        }
    }
    t5_count[0] = 1;
    t5_built = 1;
}

static inline int parity3(const int64_t a[3]) { return (int)((a[0] + a[1] + a[2]) & 1); }

static void grid_init(grid *g, int ndim, const int64_t *L, const float *f, int cplx)
{
    g->ndim = ndim;
    g->cplx = cplx;
    for (int i = 0; i < 3; i++) g->L[i] = (i < ndim) ? L[i] : 1;
    g->N = g->L[0] * g->L[1] * g->L[2];
    g->f = f;
    build_chains(ndim);
    g->ncell[0] = 1;
    if (cplx) {
        build_t5();
        for (int k = 1; k <= 3; k++) g->ncell[k] = t5_count[k];
        return;
    }
    for (int k = 1; k <= 3; k++) g->ncell[k] = (k <= ndim) ? chain_count[ndim][k] : 0;
}

static int64_t simp_id(const grid *g, const simp *s)
{
    if (s->dim == 0) return s->v[0];
    int64_t c[4][3], a[3];
    for (int i = 0; i <= s->dim; i++) coords(g, s->v[i], c[i]);
    for (int ax = 0; ax < 3; ax++) {
        a[ax] = c[0][ax];
        for (int i = 1; i <= s->dim; i++) if (c[i][ax] < a[ax]) a[ax] = c[i][ax];
    }
    int masks[4], nm = 0;
    for (int i = 0; i <= s->dim; i++) {
        int m = 0;
        for (int ax = 0; ax < 3; ax++) if (c[i][ax] - a[ax] == 1) m |= 1 << ax;
        masks[nm++] = m;
    }
    if (g->cplx) {  /* five tetrahedra: ascending masks looked up in the anchor parity's table */
        qsort(masks, nm, sizeof(int), cmp_int);
        int p = parity3(a), k = s->dim;
        for (int i = 0; i < t5_count[k]; i++)
            if (!memcmp(t5_tab[p][k][i], masks, nm * sizeof(int))) return g->ncell[k] * vid(g, a) + i;
        abort();  /* not a simplex of the complex: cannot happen */
    }
    /* sort masks by population count: S_0 = 0 < S_1 < ... < S_k */
    for (int i = 1; i < nm; i++)
        for (int j = i; j > 0 && popc(masks[j]) < popc(masks[j - 1]); j--) {
            int t = masks[j]; masks[j] = masks[j - 1]; masks[j - 1] = t;
        }
    int k = s->dim;
    int idx = -1;
    for (int i = 0; i < chain_count[g->ndim][k]; i++) {
        int ok = 1;
        for (int j = 0; j < k; j++) if (chain_tab[g->ndim][k][i][j] != masks[j + 1]) { ok = 0; break; }
        if (ok) { idx = i; break; }
    }
    if (idx < 0) abort();  /* not a Kuhn simplex: cannot happen */
    return g->ncell[k] * vid(g, a) + idx;
}

/* inverse of simp_id (vertices sorted by decreasing K) */
static void simp_from_id(const grid *g, int dim, int64_t id, simp *s)
{
    s->dim = dim;
    if (dim == 0) { s->v[0] = id; return; }
    int64_t av = id / g->ncell[dim];
    int idx = (int)(id % g->ncell[dim]);
    int64_t a[3];
    coords(g, av, a);
    if (g->cplx) {
        const int *m = t5_tab[parity3(a)][dim][idx];
        for (int j = 0; j <= dim; j++) {
            int64_t c[3];
            for (int ax = 0; ax < 3; ax++) c[ax] = a[ax] + ((m[j] >> ax) & 1);
            s->v[j] = vid(g, c);
        }
        simp_sort(g, s);
        return;
    }
    s->v[0] = av;
    for (int j = 0; j < dim; j++) {
        int m = chain_tab[g->ndim][dim][idx][j];
        int64_t c[3];
        for (int ax = 0; ax < 3; ax++) c[ax] = a[ax] + ((m >> ax) & 1);
        s->v[j + 1] = vid(g, c);
    }
    simp_sort(g, s);
}

/* Does this anchored id denote a simplex inside the grid? */
static int id_valid(const grid *g, int dim, int64_t id)
{
    if (dim == 0) return id >= 0 && id < g->N;
    int64_t av = id / g->ncell[dim];
    int idx = (int)(id % g->ncell[dim]);
    int64_t a[3];
    coords(g, av, a);
    int full = 0;
    if (g->cplx) for (int j = 0; j <= dim; j++) full |= t5_tab[parity3(a)][dim][idx][j];
    else for (int j = 0; j < dim; j++) full |= chain_tab[g->ndim][dim][idx][j];
    for (int ax = 0; ax < 3; ax++) if (((full >> ax) & 1) && a[ax] + 1 >= g->L[ax]) return 0;
    return 1;
}

/* ------------------------------------------------------------------ stars */

static const int perm1[1][3] = {{0}};
static const int perm2[2][3] = {{0, 1}, {1, 0}};
static const int perm3[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

/* The top simplices of the d-cube with minimum corner a, as vertex ids:
 * Freudenthal -- d! simplices q_0 < ... < q_d with q_{j+1} = q_j + e_{pi(j)}, one per
 * permutation pi; five tetrahedra (cplx = 1) -- t5_cube_tets.  Returns the count. */
static int cube_simplices(const grid *g, const int64_t a[3], int64_t q[6][4])
{
    int d = g->ndim;
    if (g->cplx) {
        int tets[5][4];
        t5_cube_tets(parity3(a), tets);
        for (int t = 0; t < 5; t++)
            for (int j = 0; j < 4; j++) {
                int64_t qc[3];
                for (int ax = 0; ax < 3; ax++) qc[ax] = a[ax] + ((tets[t][j] >> ax) & 1);
                q[t][j] = vid(g, qc);
            }
        return 5;
    }
    int nperm = d == 1 ? 1 : d == 2 ? 2 : 6;
    const int (*perm)[3] = d == 1 ? perm1 : d == 2 ? perm2 : perm3;
    for (int p = 0; p < nperm; p++) {
        int64_t qc[3] = {a[0], a[1], a[2]};
        q[p][0] = vid(g, qc);
        for (int j = 0; j < d; j++) { qc[perm[p][j]] += 1; q[p][j + 1] = vid(g, qc); }
    }
    return nperm;
}

/* All simplices of the complex containing x: every d-cube incident to x is split into
 * its top simplices (cube_simplices); the star of x is every face of those simplices
 * that contains x.  If lower_only, keep the lower star St^-(x): faces
 * whose other vertices all precede x in K order.  Returns the number of simplices
 * (excluding the vertex x itself). */
static int star(const grid *g, int64_t x, int lower_only, simp *out)
{
    int d = g->ndim;
    int64_t c[3];
    coords(g, x, c);
    int n = 0;
    for (int b = 0; b < (1 << d); b++) {
        int64_t a[3] = {c[0], c[1], c[2]};
        int ok = 1;
        for (int ax = 0; ax < d; ax++) {
            a[ax] -= (b >> ax) & 1;
            if (a[ax] < 0 || a[ax] > g->L[ax] - 2) ok = 0;
        }
        if (!ok) continue;
        int64_t qs[6][4];
        int nq = cube_simplices(g, a, qs);
        for (int p = 0; p < nq; p++) {
            const int64_t *q = qs[p];
            int j0 = -1;
            for (int j = 0; j <= d; j++) if (q[j] == x) j0 = j;
            if (j0 < 0) continue;
            int64_t others[3];
            int no = 0;
            for (int j = 0; j <= d; j++) if (j != j0) others[no++] = q[j];
            for (int m = 1; m < (1 << no); m++) {
                simp s;
                s.dim = 0;
                s.v[0] = x;
                int keep = 1;
                for (int j = 0; j < no; j++) if ((m >> j) & 1) {
                    if (lower_only && !klt(g, others[j], x)) keep = 0;
                    s.v[++s.dim] = others[j];
                }
                if (!keep) continue;
                simp_sort(g, &s);
                int dup = 0;
                for (int i = 0; i < n; i++) if (simp_eq(&out[i], &s)) { dup = 1; break; }
                if (!dup) out[n++] = s;
            }
        }
    }
    return n;
}

/* ------------------------------------------------------------------ growable buffers */

typedef struct { void *p; int64_t n, cap; size_t el; } vec;

static void vpush(vec *v, const void *x)
{
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 1024;
        v->p = realloc(v->p, v->cap * v->el);
        if (!v->p) abort();
    }
    memcpy((char *)v->p + v->n * v->el, x, v->el);
    v->n++;
}

static void vappend(vec *v, const vec *w)
{
    for (int64_t i = 0; i < w->n; i++) vpush(v, (const char *)w->p + i * w->el);
}

/* ------------------------------------------------------------------ ProcessLowerStars */

typedef struct {
    const grid *g;
    int64_t *vpart;    /* [N]: id of the edge paired with vertex v, -1 if critical */
    int64_t *toppart;  /* [ncell[d]*N]: id of the facet paired with a d-simplex, -1 critical */
    int64_t *epart;    /* optional [ncell[1]*N]: id of the triangle an edge is paired with (the
                        * edge is the tail of a vector), else untouched (-1) -- for D1 */
    vec pairs;         /* int64 triples (tail dim, tail id, head id) */
    vec crit;          /* simp */
    int want_pairs;
} lsctx;

/* facet lists inside the lower star: fac[a][0..nfac[a]) = indices j with L[j] a facet of L[a] */
typedef struct { int nfac[128]; unsigned char fac[128][4]; } facets_t;

/* number of facets of L[a] (inside the lower star) that are still unclassified,
 * and the last such facet found */
static int num_unpaired(const facets_t *F, const int *state, int a, int *which)
{
    int cnt = 0;
    for (int i = 0; i < F->nfac[a]; i++) {
        int j = F->fac[a][i];
        if (state[j] == 0) { cnt++; *which = j; }
    }
    return cnt;
}

static int has_facet(const facets_t *F, int a, int j)
{
    for (int i = 0; i < F->nfac[a]; i++) if (F->fac[a][i] == j) return 1;
    return 0;
}

static void emit_pair(lsctx *c, const simp *tail, const simp *head)
{
    int64_t tid = simp_id(c->g, tail), hid = simp_id(c->g, head);
    if (tail->dim == 0 && c->vpart) c->vpart[tail->v[0]] = hid;
    if (head->dim == c->g->ndim && c->toppart) c->toppart[hid] = tid;
    if (tail->dim == 1 && head->dim == 2 && c->epart) c->epart[tid] = hid;
    if (c->want_pairs) {
        int64_t t[3] = {tail->dim, tid, hid};
        vpush(&c->pairs, t);
    }
}

static void emit_crit(lsctx *c, const simp *s)
{
    if (s->dim == 0 && c->vpart) c->vpart[s->v[0]] = -1;
    if (s->dim == c->g->ndim && c->toppart) c->toppart[simp_id(c->g, s)] = -1;
    vpush(&c->crit, s);
}

static int cmp_simp_r(const void *a, const void *b, void *g) { return lexcmp((const grid *)g, a, b); }

/* Robins, Wood & Sheppard (PAMI 2011) ProcessLowerStars, the expansion algorithm the
 * paper uses for the discrete gradient, on the
 * lower star of one vertex x.  Priorities are the lexicographic order of P:1380-1414
 * (reading Z1).  PQzero holds cells with no unclassified facet in the lower star
 * (critical candidates), PQone holds cells with exactly one.  The queues are kept as
 * sets (a flag per cell); popping the minimum = the first flagged cell of the lower
 * star sorted by G.  A cell that got classified while queued is skipped on pop. */
static void process_lower_star(lsctx *c, int64_t x)
{
    const grid *g = c->g;
    simp L[128];
    int state[128];  /* 0 unclassified, 1 paired, 2 critical */
    char pq0[128], pq1[128];
    int n = star(g, x, 1, L);
    simp sx = {0, {x, 0, 0, 0}};
    if (n == 0) {  /* L = {x}: x is a minimum */
        emit_crit(c, &sx);
        return;
    }
    qsort_r(L, n, sizeof(simp), cmp_simp_r, (void *)g);
    facets_t F;
    for (int i = 0; i < n; i++) {
        state[i] = 0; pq0[i] = 0; pq1[i] = 0;
        F.nfac[i] = 0;
        for (int j = 0; j < n; j++) if (is_facet(&L[j], &L[i])) F.fac[i][F.nfac[i]++] = (unsigned char)j;
    }
    /* delta := the edge of L(x) with minimal G; pair (x, delta) */
    int delta = -1;
    for (int i = 0; i < n; i++) if (L[i].dim == 1) { delta = i; break; }
    emit_pair(c, &sx, &L[delta]);
    state[delta] = 1;
    /* all other edges -> PQzero */
    for (int i = 0; i < n; i++) if (L[i].dim == 1 && i != delta) pq0[i] = 1;
    /* cofacets of delta with one unclassified facet -> PQone */
    for (int i = 0; i < n; i++) {
        int w;
        if (has_facet(&F, i, delta) && num_unpaired(&F, state, i, &w) == 1) pq1[i] = 1;
    }
    for (;;) {
        int any0 = 0, any1 = 0;
        for (int i = 0; i < n; i++) { any0 |= pq0[i]; any1 |= pq1[i]; }
        if (!any0 && !any1) break;
        /* while PQone not empty */
        for (;;) {
            int a = -1;
            for (int i = 0; i < n; i++) if (pq1[i]) { a = i; break; }
            if (a < 0) break;
            pq1[a] = 0;
            if (state[a] != 0) continue;
            int t = -1;
            int nu = num_unpaired(&F, state, a, &t);
            if (nu == 0) {
                pq0[a] = 1;
            } else {
                /* pair(alpha) = its unique unclassified facet t */
                emit_pair(c, &L[t], &L[a]);
                state[t] = 1;
                state[a] = 1;
                pq0[t] = 0;
                for (int b = 0; b < n; b++) {
                    int w;
                    if (state[b] == 0 && (has_facet(&F, b, a) || has_facet(&F, b, t)) &&
                        num_unpaired(&F, state, b, &w) == 1)
                        pq1[b] = 1;
                }
            }
        }
        /* if PQzero not empty: pop gamma, it is critical */
        int gm = -1;
        for (int i = 0; i < n; i++) if (pq0[i]) { gm = i; break; }
        if (gm < 0) continue;
        pq0[gm] = 0;
        if (state[gm] != 0) continue;
        state[gm] = 2;
        emit_crit(c, &L[gm]);
        for (int b = 0; b < n; b++) {
            int w;
            if (state[b] == 0 && has_facet(&F, b, gm) && num_unpaired(&F, state, b, &w) == 1)
                pq1[b] = 1;
        }
    }
}

/* ------------------------------------------------------------------ results */

#define ORC_MAXD 4

typedef struct {
    int64_t birth_id, death_id;
    int32_t birth_vertex, death_vertex;
    float birth_value, death_value;
} orc_pair;

typedef struct orc_result {
    grid g;
    int64_t ncrit[ORC_MAXD];
    int64_t *crit[ORC_MAXD];     /* ids, lexicographically sorted (full run) */
    int64_t npairs;
    int64_t *pairs;              /* gradient pairs, triples */
    int64_t nd0, ndtop, ndtop_ign;
    orc_pair *d0, *dtop, *dtop_ign;  /* dtop_ign: D_{d-1} in the "ignore" boundary mode */
    int64_t nun0, nuntop;
    int64_t *un0, *untop;        /* unpaired saddles after D0 / D_{d-1} */
    int64_t *arcs0, *arcstop;    /* per arc: the two extremum ends (ids; -1 = VIRTUAL) */
    int64_t nd1;
    orc_pair *d1;                /* 3D, want_d1: D1 pairs in increasing death (2-saddle) order */
    int64_t *gen_off, *gen;      /* the generator (earliest cycle, edge ids) of D1 pair i:
                                    gen[gen_off[i] .. gen_off[i+1]) */
    int64_t nun1;
    int64_t *un1;                /* 1-saddles left unpaired after D1 (infinite D1 classes) */
    double ms[8];                /* stage times: order, gradient, sort C_k, D0, Dtop, D1 */
} orc_result;

typedef struct {
    lsctx c;
    int64_t v0, v1;
    const int64_t *verts;
} job;

static void *run_job(void *p)
{
    job *j = (job *)p;
    for (int64_t i = j->v0; i < j->v1; i++)
        process_lower_star(&j->c, j->verts ? j->verts[i] : i);
    return NULL;
}

static double now_ms(void)
{
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
}

/* run ProcessLowerStars over the given vertices (all if verts == NULL) */
static void gradient(const grid *g, const int64_t *verts, int64_t nv, int nthreads, int want_pairs,
                     int64_t *vpart, int64_t *toppart, int64_t *epart, vec *pairs, vec *crit)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    job *jobs = calloc(nthreads, sizeof(job));
    pthread_t *th = calloc(nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; t++) {
        jobs[t].c.g = g;
        jobs[t].c.vpart = vpart;
        jobs[t].c.toppart = toppart;
        jobs[t].c.epart = epart;
        jobs[t].c.want_pairs = want_pairs;
        jobs[t].c.pairs.el = 3 * sizeof(int64_t);
        jobs[t].c.crit.el = sizeof(simp);
        jobs[t].v0 = nv * t / nthreads;
        jobs[t].v1 = nv * (t + 1) / nthreads;
        jobs[t].verts = verts;
    }
    if (nthreads == 1) run_job(&jobs[0]);
    else {
        for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, run_job, &jobs[t]);
        for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    }
    for (int t = 0; t < nthreads; t++) {
        vappend(pairs, &jobs[t].c.pairs);
        vappend(crit, &jobs[t].c.crit);
        free(jobs[t].c.pairs.p);
        free(jobs[t].c.crit.p);
    }
    free(jobs);
    free(th);
}

static int check_args(int ndim, const int64_t *L)
{
    if (ndim < 1 || ndim > 3) return 2;
    int64_t n = 1;
    for (int i = 0; i < ndim; i++) {
        if (L[i] < 2) return 2;
        n *= L[i];
        if (n >= ((int64_t)1 << 31)) return 4;
    }
    return 0;
}

/* ------------------------------------------------------------------ O1 ranks */

static int cmp_vertex_r(const void *a, const void *b, void *g)
{
    int64_t u = *(const int64_t *)a, v = *(const int64_t *)b;
    if (u == v) return 0;
    return klt((const grid *)g, u, v) ? -1 : 1;
}

/* rank(v) = #{u : K(u) < K(v)}, by sorting the vertices with the K
 * comparison.  Returns 3 if some value is NaN. */
int orc_ranks(int64_t n, const float *f, int32_t *rank)
{
    for (int64_t i = 0; i < n; i++) if (isnan(f[i])) return 3;
    grid g;
    memset(&g, 0, sizeof g);
    g.f = f;
    g.N = n;
    int64_t *idx = malloc(n * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) idx[i] = i;
    qsort_r(idx, n, sizeof(int64_t), cmp_vertex_r, &g);
    for (int64_t i = 0; i < n; i++) rank[idx[i]] = (int32_t)i;
    free(idx);
    return 0;
}

/* ------------------------------------------------------------------ union-find */

static int64_t uf_find(int64_t *parent, int64_t a)
{
    while (parent[a] != a) a = parent[a];
    return a;
}

static float fmax_all(const grid *g)
{
    int64_t m = 0;
    for (int64_t v = 1; v < g->N; v++) if (klt(g, m, v)) m = v;
    return g->f[m];
}

/* ------------------------------------------------------------------ full run */

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : x > y;
}

static int cmp_triple(const void *a, const void *b)
{
    const int64_t *x = a, *y = b;
    for (int i = 0; i < 3; i++) if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}

/* the d-simplices having the (d-1)-simplex s as a facet (1 on the grid boundary,
 * else 2), sorted by id: scan the top simplices of every d-cube around s's first vertex
 * (each top simplex comes from exactly one cube). */
static int cofacets(const grid *g, const simp *s, int64_t out[2])
{
    int d = g->ndim;
    int64_t c[3];
    int64_t x = s->v[0];
    coords(g, x, c);
    int nf = 0;
    for (int b = 0; b < (1 << d); b++) {
        int64_t a[3] = {c[0], c[1], c[2]};
        int ok = 1;
        for (int ax = 0; ax < d; ax++) {
            a[ax] -= (b >> ax) & 1;
            if (a[ax] < 0 || a[ax] > g->L[ax] - 2) ok = 0;
        }
        if (!ok) continue;
        int64_t qs[6][4];
        int nq = cube_simplices(g, a, qs);
        for (int p = 0; p < nq; p++) {
            simp t;
            t.dim = d;
            for (int j = 0; j <= d; j++) t.v[j] = qs[p][j];
            int contains = 1;
            for (int i = 0; i <= s->dim && contains; i++) {
                int found = 0;
                for (int j = 0; j <= d; j++) if (t.v[j] == s->v[i]) found = 1;
                contains = found;
            }
            if (!contains) continue;
            if (nf == 2) abort();
            simp_sort(g, &t);
            out[nf++] = simp_id(g, &t);
        }
    }
    if (nf == 2 && out[0] > out[1]) { int64_t t = out[0]; out[0] = out[1]; out[1] = t; }
    return nf;
}

static orc_pair mkpair(const grid *g, int bdim, int64_t bid, int ddim, int64_t did, float fstar)
{
    orc_pair p;
    simp b, d;
    simp_from_id(g, bdim, bid, &b);
    p.birth_id = bid;
    p.birth_vertex = (int32_t)b.v[0];
    p.birth_value = g->f[b.v[0]];
    if (did < 0) {
        p.death_id = -1;
        p.death_vertex = -1;
        p.death_value = fstar;
    } else {
        simp_from_id(g, ddim, did, &d);
        p.death_id = did;
        p.death_vertex = (int32_t)d.v[0];
        p.death_value = g->f[d.v[0]];
    }
    return p;
}

/* Full front end. nthreads only fans the per-vertex gradient loop out;
 * everything else is sequential as in the paper's D0/D_{d-1} union-find. */
/* flags: bit 0 want_pairs (the gradient vectors), bit 1 want_d1 (3D: D1 by Alg. 3 and
 * the generators of Sec. 9) */
/* cplx: 0 Freudenthal, 1 five tetrahedra per cube (3D only; else status 1) */
int orc_run3(int ndim, const int64_t *L, const float *f, int nthreads, int flags, int cplx, orc_result **out)
{
    const int want_pairs = flags & 1;
    const int want_d1 = (flags & 2) && ndim == 3;
    int st = check_args(ndim, L);
    if (st) return st;
    if (cplx < 0 || cplx > 1 || (cplx == 1 && ndim != 3)) return 1;
    orc_result *r = calloc(1, sizeof(orc_result));
    grid *g = &r->g;
    grid_init(g, ndim, L, f, cplx);
    int d = ndim;
    double t0 = now_ms();
    for (int64_t i = 0; i < g->N; i++) if (isnan(f[i])) { free(r); return 3; }
    float fstar = fmax_all(g);
    r->ms[0] = now_ms() - t0;

    /* O3: gradient over every lower star */
    t0 = now_ms();
    int64_t ntop = g->ncell[d] * g->N;
    int64_t *vpart = malloc(g->N * sizeof(int64_t));
    int64_t *toppart = malloc(ntop * sizeof(int64_t));
    for (int64_t i = 0; i < ntop; i++) toppart[i] = -2;
    vec pairs = {0}, crit = {0};
    pairs.el = 3 * sizeof(int64_t);
    crit.el = sizeof(simp);
    int64_t *epart = NULL;
    if (want_d1) {
        int64_t ne = g->ncell[1] * g->N;
        epart = malloc(ne * sizeof(int64_t));
        for (int64_t i = 0; i < ne; i++) epart[i] = -1;
    }
    gradient(g, NULL, g->N, nthreads, want_pairs, vpart, toppart, epart, &pairs, &crit);
    r->ms[1] = now_ms() - t0;

    /* O4: Alg. 2 -- critical simplices into C_k, each sorted lexicographically */
    t0 = now_ms();
    simp *cs[ORC_MAXD];
    for (int k = 0; k <= d; k++) { cs[k] = malloc((crit.n + 1) * sizeof(simp)); r->ncrit[k] = 0; }
    for (int64_t i = 0; i < crit.n; i++) {
        simp *s = (simp *)crit.p + i;
        cs[s->dim][r->ncrit[s->dim]++] = *s;
    }
    for (int k = 0; k <= d; k++) {
        qsort_r(cs[k], r->ncrit[k], sizeof(simp), cmp_simp_r, g);
        r->crit[k] = malloc((r->ncrit[k] + 1) * sizeof(int64_t));
        for (int64_t i = 0; i < r->ncrit[k]; i++) r->crit[k][i] = simp_id(g, &cs[k][i]);
    }
    free(crit.p);
    if (want_pairs) {
        r->npairs = pairs.n;
        r->pairs = pairs.p;
        qsort(r->pairs, r->npairs, 3 * sizeof(int64_t), cmp_triple);
    } else free(pairs.p);
    r->ms[2] = now_ms() - t0;

    /* O5: D0, Sec. 5.1.  (a) unstable sets of the critical edges: from each vertex
     * of the edge follow the vertex -> edge vectors down to a minimum;  (b) the graph
     * G_D0 (nodes minima, arcs critical edges);  (c,d) Union-Find over the arcs in
     * increasing lexicographic order, the younger (higher) minimum dies (Elder rule,
     * P:1641-1664), the older one stays the representative. */
    t0 = now_ms();
    {
        int64_t m = r->ncrit[1];
        int64_t *parent = malloc(g->N * sizeof(int64_t));
        for (int64_t i = 0; i < r->ncrit[0]; i++) parent[r->crit[0][i]] = r->crit[0][i];
        r->d0 = malloc((m + 2) * sizeof(orc_pair));
        r->un0 = malloc((m + 1) * sizeof(int64_t));
        r->arcs0 = malloc((2 * m + 1) * sizeof(int64_t));
        r->nd0 = r->nun0 = 0;
        for (int64_t i = 0; i < m; i++) {
            simp e = cs[1][i];
            int64_t end[2];
            for (int s = 0; s < 2; s++) {
                int64_t v = e.v[s];
                while (vpart[v] != -1) {  /* v paired with edge vpart[v]: go to its other vertex */
                    simp pe;
                    simp_from_id(g, 1, vpart[v], &pe);
                    v = (pe.v[0] == v) ? pe.v[1] : pe.v[0];
                }
                end[s] = v;
            }
            r->arcs0[2 * i] = end[0];
            r->arcs0[2 * i + 1] = end[1];
            int64_t a = uf_find(parent, end[0]), b = uf_find(parent, end[1]);
            if (a == b) { r->un0[r->nun0++] = r->crit[1][i]; continue; }  /* 1-cycle */
            int64_t young = klt(g, a, b) ? b : a, old = (young == a) ? b : a;
            r->d0[r->nd0++] = mkpair(g, 0, young, 1, r->crit[1][i], fstar);
            parent[young] = old;
        }
        /* Sec. 6: unpaired minima are infinite classes (f(min), f*) */
        for (int64_t i = 0; i < r->ncrit[0]; i++) {
            int64_t v = r->crit[0][i];
            if (parent[v] == v) r->d0[r->nd0++] = mkpair(g, 0, v, 1, -1, fstar);
        }
        free(parent);
    }
    r->ms[3] = now_ms() - t0;

    /* O6: D_{d-1}, Sec. 5.2.  Dual gradient: stable sets of the critical
     * (d-1)-simplices, followed from each cofacet c: while c is not critical,
     * s' = Pair(c) (the facet c is paired with), c = the other cofacet of s', or the
     * virtual maximum when s' is on the boundary (reading Z6: exact
     * mode).  Union-Find over the arcs in decreasing lexicographic order;
     * a merge pays the younger (lower) maximum; the virtual maximum is the oldest. */
    t0 = now_ms();
    {
        int64_t m = r->ncrit[d - 1];
        int64_t V = ntop;  /* the virtual maximum */
        int64_t *parent = malloc((ntop + 1) * sizeof(int64_t));
        for (int64_t i = 0; i < r->ncrit[d]; i++) parent[r->crit[d][i]] = r->crit[d][i];
        parent[V] = V;
        r->dtop = malloc((m + 2) * sizeof(orc_pair));
        r->untop = malloc((m + 1) * sizeof(int64_t));
        r->arcstop = malloc((2 * m + 1) * sizeof(int64_t));
        r->ndtop = r->nuntop = 0;
        /* "older" for maxima: larger lexicographic key; V older than all */
        for (int64_t i = m - 1; i >= 0; i--) {
            simp s = cs[d - 1][i];
            int64_t end[2];
            for (int side = 0; side < 2; side++) {
                int64_t cf[2];
                int ncf = cofacets(g, &s, cf);
                int64_t c = side < ncf ? cf[side] : -1;  /* -1: the virtual maximum */
                while (c >= 0 && toppart[c] != -1) {
                    simp sp;
                    simp_from_id(g, d - 1, toppart[c], &sp);  /* s' = Pair(c) */
                    int64_t cf2[2];
                    int n2 = cofacets(g, &sp, cf2);
                    int64_t next = -1;
                    for (int j = 0; j < n2; j++) if (cf2[j] != c) next = cf2[j];
                    c = next;
                }
                end[side] = c < 0 ? V : c;
            }
            r->arcstop[2 * i] = end[0] == V ? -1 : end[0];
            r->arcstop[2 * i + 1] = end[1] == V ? -1 : end[1];
            int64_t a = uf_find(parent, end[0]), b = uf_find(parent, end[1]);
            if (a == b) { r->untop[r->nuntop++] = r->crit[d - 1][i]; continue; }
            int64_t young, old;
            if (a == V) { young = b; old = a; }
            else if (b == V) { young = a; old = b; }
            else {
                simp sa, sb;
                simp_from_id(g, d, a, &sa);
                simp_from_id(g, d, b, &sb);
                if (lexcmp(g, &sa, &sb) < 0) { young = a; old = b; } else { young = b; old = a; }
            }
            r->dtop[r->ndtop++] = mkpair(g, d - 1, r->crit[d - 1][i], d, young, fstar);
            parent[young] = old;
        }
        /* Sec. 6 for d = 1: the (d-1) = 0-simplex left unpaired is an infinite D0 class */
        if (d == 1)
            for (int64_t j = 0; j < r->nuntop; j++)
                r->dtop[r->ndtop++] = mkpair(g, 0, r->untop[j], 1, -1, fstar);
        qsort(r->untop, r->nuntop, sizeof(int64_t), cmp_i64);

        /* O6' "ignore" boundary mode (App. A; reading Z7): no
         * virtual maximum -- an arc that reaches the boundary is dropped (its saddle
         * stays unpaired), the same Union-Find in decreasing order runs on the other
         * arcs, and the global maximum is left unpaired (its class is the D0 infinite
         * class (global min, f*), "paired by convention to the global minimum", Sec. 6).
         * No infinite records. */
        for (int64_t i = 0; i < r->ncrit[d]; i++) parent[r->crit[d][i]] = r->crit[d][i];
        r->dtop_ign = malloc((m + 1) * sizeof(orc_pair));
        r->ndtop_ign = 0;
        for (int64_t i = m - 1; i >= 0; i--) {
            const int64_t e0 = r->arcstop[2 * i], e1 = r->arcstop[2 * i + 1];
            if (e0 < 0 || e1 < 0) continue;  /* a half-arc to the outside: dropped */
            int64_t a = uf_find(parent, e0), b = uf_find(parent, e1);
            if (a == b) continue;
            simp sa, sb;
            simp_from_id(g, d, a, &sa);
            simp_from_id(g, d, b, &sb);
            int64_t young, old;
            if (lexcmp(g, &sa, &sb) < 0) { young = a; old = b; } else { young = b; old = a; }
            r->dtop_ign[r->ndtop_ign++] = mkpair(g, d - 1, r->crit[d - 1][i], d, young, fstar);
            parent[young] = old;
        }
        free(parent);
    }
    /* unpaired lists in ascending lexicographic order */
    {
        /* un0 was produced in ascending order already; untop: re-sort by lex key */
        simp *tmp = malloc((r->nuntop + 1) * sizeof(simp));
        for (int64_t i = 0; i < r->nuntop; i++) simp_from_id(g, d - 1, r->untop[i], &tmp[i]);
        qsort_r(tmp, r->nuntop, sizeof(simp), cmp_simp_r, g);
        for (int64_t i = 0; i < r->nuntop; i++) r->untop[i] = simp_id(g, &tmp[i]);
        free(tmp);
    }
    r->ms[4] = now_ms() - t0;

    /* O9 (3D, want_d1): D1 by Alg. 3 "PairCriticalSimplices" with boundary
     * caching, on the 2-saddles that D_{d-1} left unpaired (sandwiching:
     * the critical simplices already paired in D0 and D_{d-1} are discarded,
     * P:1125-1155), in increasing lexicographic order.  Boundary(sigma) starts as the
     * boundary of sigma (its three edges); while it is not empty, tau = its highest edge
     * in the lexicographic order:
     *   tau critical, not yet paired in D1: it created the 1-cycle; pair (tau, sigma);
     *   tau critical, paired with sigma' in D1: Boundary += Boundary(sigma') (cached);
     *   tau regular: Pair(tau) is the triangle t of its discrete vector:
     *     Boundary += boundary of t.
     * Additions are mod 2.  The final Boundary of a pair is its generator,
     * the earliest 1-cycle homologous to the boundary of sigma (Sec. 9). */
    t0 = now_ms();
    if (want_d1) {
        int64_t ne = g->ncell[1] * g->N;
        signed char *estate = calloc(ne, 1);  /* 1: critical, paired in D0; 2: critical, positive */
        int32_t *owner = malloc(ne * sizeof(int32_t));
        for (int64_t i = 0; i < ne; i++) owner[i] = -1;
        for (int64_t i = 0; i < r->ncrit[1]; i++) estate[r->crit[1][i]] = 1;
        for (int64_t i = 0; i < r->nun0; i++) estate[r->un0[i]] = 2;
        int64_t m = r->nuntop;
        r->d1 = malloc((m + 1) * sizeof(orc_pair));
        r->gen_off = malloc((m + 2) * sizeof(int64_t));
        simp **cache = calloc(m + 1, sizeof(simp *));
        int64_t *ncache = calloc(m + 1, sizeof(int64_t));
        vec gen = {0};
        gen.el = sizeof(int64_t);
        int64_t capB = 64, nB = 0;
        simp *B = malloc(capB * sizeof(simp)), *T = malloc(capB * sizeof(simp));
        r->nd1 = 0;
        r->gen_off[0] = 0;
        for (int64_t i = 0; i < m; i++) {
            simp sg;
            simp_from_id(g, 2, r->untop[i], &sg);
            simp fac[3];
            for (int j = 0; j < 3; j++) {  /* facets of sg, vertices still decreasing */
                fac[j].dim = 1;
                int q = 0;
                for (int u = 0; u < 3; u++) if (u != 2 - j) fac[j].v[q++] = sg.v[u];
            }
            qsort_r(fac, 3, sizeof(simp), cmp_simp_r, g);
            nB = 3;
            memcpy(B, fac, 3 * sizeof(simp));
            while (nB > 0) {
                const simp *tau = &B[nB - 1];
                int64_t tid = simp_id(g, tau);
                const simp *add;
                int64_t nadd;
                simp tf[3];
                if (estate[tid] == 2) {
                    if (owner[tid] < 0) break;  /* unpaired: tau created the cycle */
                    add = cache[owner[tid]];
                    nadd = ncache[owner[tid]];
                } else if (estate[tid] == 1) {
                    abort();  /* a D0 death edge is negative: never the highest edge of a cycle */
                } else {
                    int64_t t = epart[tid];
                    if (t < 0) abort();  /* a regular edge on a cycle is the tail of a vector */
                    simp st;
                    simp_from_id(g, 2, t, &st);
                    for (int j = 0; j < 3; j++) {
                        tf[j].dim = 1;
                        int q = 0;
                        for (int u = 0; u < 3; u++) if (u != 2 - j) tf[j].v[q++] = st.v[u];
                    }
                    qsort_r(tf, 3, sizeof(simp), cmp_simp_r, g);
                    add = tf;
                    nadd = 3;
                }
                /* Boundary += add (mod 2): merge of two sorted lists, equal entries cancel */
                if (nB + nadd > capB) {
                    while (nB + nadd > capB) capB *= 2;
                    B = realloc(B, capB * sizeof(simp));
                    T = realloc(T, capB * sizeof(simp));
                }
                int64_t a = 0, b = 0, n = 0;
                while (a < nB || b < nadd) {
                    int c = a >= nB ? 1 : (b >= nadd ? -1 : lexcmp(g, &B[a], &add[b]));
                    if (c < 0) T[n++] = B[a++];
                    else if (c > 0) T[n++] = add[b++];
                    else { a++; b++; }
                }
                simp *sw = B; B = T; T = sw;
                nB = n;
            }
            if (nB == 0) abort();  /* grids are balls: every such 2-saddle kills a 1-cycle */
            int64_t tid = simp_id(g, &B[nB - 1]);
            int64_t k = r->nd1;
            owner[tid] = (int32_t)k;
            cache[k] = malloc(nB * sizeof(simp));
            memcpy(cache[k], B, nB * sizeof(simp));
            ncache[k] = nB;
            r->d1[k] = mkpair(g, 1, tid, 2, r->untop[i], fstar);
            for (int64_t j = 0; j < nB; j++) {
                int64_t eid = simp_id(g, &B[j]);
                vpush(&gen, &eid);
            }
            r->nd1++;
            r->gen_off[r->nd1] = gen.n;
        }
        r->gen = gen.p ? gen.p : malloc(sizeof(int64_t));
        r->un1 = malloc((r->nun0 + 1) * sizeof(int64_t));
        r->nun1 = 0;
        for (int64_t i = 0; i < r->nun0; i++)
            if (owner[r->un0[i]] < 0) r->un1[r->nun1++] = r->un0[i];
        for (int64_t k = 0; k < r->nd1; k++) free(cache[k]);
        free(cache);
        free(ncache);
        free(B);
        free(T);
        free(estate);
        free(owner);
    }
    r->ms[5] = now_ms() - t0;
    free(epart);
    for (int k = 0; k <= d; k++) free(cs[k]);
    free(vpart);
    free(toppart);
    *out = r;
    return 0;
}

int orc_run2(int ndim, const int64_t *L, const float *f, int nthreads, int flags, orc_result **out)
{
    return orc_run3(ndim, L, f, nthreads, flags, 0, out);
}

int orc_run(int ndim, const int64_t *L, const float *f, int nthreads, int want_pairs, orc_result **out)
{
    return orc_run3(ndim, L, f, nthreads, want_pairs ? 1 : 0, 0, out);
}

/* Gradient restricted to the lower stars of the given vertices (for sampled parity
 * at sizes where the full run is too slow).  Pairs sorted; critical ids per dim
 * sorted by id. */
int orc_gradient_sample2(int ndim, const int64_t *L, const float *f, const int64_t *verts, int64_t nv,
                         int nthreads, int cplx, orc_result **out)
{
    int st = check_args(ndim, L);
    if (st) return st;
    if (cplx < 0 || cplx > 1 || (cplx == 1 && ndim != 3)) return 1;
    orc_result *r = calloc(1, sizeof(orc_result));
    grid *g = &r->g;
    grid_init(g, ndim, L, f, cplx);
    vec pairs = {0}, crit = {0};
    pairs.el = 3 * sizeof(int64_t);
    crit.el = sizeof(simp);
    gradient(g, verts, nv, nthreads, 1, NULL, NULL, NULL, &pairs, &crit);
    r->npairs = pairs.n;
    r->pairs = pairs.p;
    qsort(r->pairs, r->npairs, 3 * sizeof(int64_t), cmp_triple);
    for (int k = 0; k <= ndim; k++) {
        r->crit[k] = malloc((crit.n + 1) * sizeof(int64_t));
        r->ncrit[k] = 0;
    }
    for (int64_t i = 0; i < crit.n; i++) {
        simp *s = (simp *)crit.p + i;
        r->crit[s->dim][r->ncrit[s->dim]++] = simp_id(g, s);
    }
    for (int k = 0; k <= ndim; k++) qsort(r->crit[k], r->ncrit[k], sizeof(int64_t), cmp_i64);
    free(crit.p);
    *out = r;
    return 0;
}

int orc_gradient_sample(int ndim, const int64_t *L, const float *f, const int64_t *verts, int64_t nv,
                        int nthreads, orc_result **out)
{
    return orc_gradient_sample2(ndim, L, f, verts, nv, nthreads, 0, out);
}

/* ------------------------------------------------------------------ accessors */

enum { ORC_CRIT = 0, ORC_PAIRS = 1, ORC_D0 = 2, ORC_DTOP = 3, ORC_UN0 = 4, ORC_UNTOP = 5,
       ORC_ARCS0 = 6, ORC_ARCSTOP = 7, ORC_MS = 8, ORC_D1 = 9, ORC_GEN_OFF = 10, ORC_GEN = 11,
       ORC_UN1 = 12, ORC_DTOP_IGN = 13 };

int64_t orc_count(const orc_result *r, int what, int k)
{
    switch (what) {
    case ORC_CRIT: return (k >= 0 && k <= r->g.ndim) ? r->ncrit[k] : 0;
    case ORC_PAIRS: return r->npairs;
    case ORC_D0: return r->nd0;
    case ORC_DTOP: return r->ndtop;
    case ORC_UN0: return r->nun0;
    case ORC_UNTOP: return r->nuntop;
    case ORC_ARCS0: return r->arcs0 ? r->ncrit[1] : 0;
    case ORC_ARCSTOP: return r->arcstop ? r->ncrit[r->g.ndim - 1] : 0;
    case ORC_MS: return 6;
    case ORC_D1: return r->d1 ? r->nd1 : 0;
    case ORC_GEN_OFF: return r->gen_off ? r->nd1 + 1 : 0;
    case ORC_GEN: return r->gen_off ? r->gen_off[r->nd1] : 0;
    case ORC_UN1: return r->un1 ? r->nun1 : 0;
    case ORC_DTOP_IGN: return r->dtop_ign ? r->ndtop_ign : 0;
    }
    return 0;
}

void orc_copy(const orc_result *r, int what, int k, void *dst)
{
    int64_t n = orc_count(r, what, k);
    switch (what) {
    case ORC_CRIT: memcpy(dst, r->crit[k], n * sizeof(int64_t)); break;
    case ORC_PAIRS: memcpy(dst, r->pairs, n * 3 * sizeof(int64_t)); break;
    case ORC_D0: memcpy(dst, r->d0, n * sizeof(orc_pair)); break;
    case ORC_DTOP: memcpy(dst, r->dtop, n * sizeof(orc_pair)); break;
    case ORC_UN0: memcpy(dst, r->un0, n * sizeof(int64_t)); break;
    case ORC_UNTOP: memcpy(dst, r->untop, n * sizeof(int64_t)); break;
    case ORC_ARCS0: memcpy(dst, r->arcs0, 2 * n * sizeof(int64_t)); break;
    case ORC_ARCSTOP: memcpy(dst, r->arcstop, 2 * n * sizeof(int64_t)); break;
    case ORC_MS: memcpy(dst, r->ms, 6 * sizeof(double)); break;
    case ORC_D1: memcpy(dst, r->d1, n * sizeof(orc_pair)); break;
    case ORC_GEN_OFF: memcpy(dst, r->gen_off, n * sizeof(int64_t)); break;
    case ORC_GEN: memcpy(dst, r->gen, n * sizeof(int64_t)); break;
    case ORC_UN1: memcpy(dst, r->un1, n * sizeof(int64_t)); break;
    case ORC_DTOP_IGN: memcpy(dst, r->dtop_ign, n * sizeof(orc_pair)); break;
    }
}

void orc_free(orc_result *r)
{
    if (!r) return;
    for (int k = 0; k < ORC_MAXD; k++) free(r->crit[k]);
    free(r->pairs);
    free(r->d0);
    free(r->dtop);
    free(r->dtop_ign);
    free(r->un0);
    free(r->untop);
    free(r->arcs0);
    free(r->arcstop);
    free(r->d1);
    free(r->gen_off);
    free(r->gen);
    free(r->un1);
    free(r);
}

/* anchored id <-> vertices, exported for the oracle's own tests */
int orc_simplex_vertices2(int ndim, const int64_t *L, int dim, int64_t id, int cplx, int64_t *verts_out)
{
    if (check_args(ndim, L)) return 2;
    if (cplx < 0 || cplx > 1 || (cplx == 1 && ndim != 3)) return 1;
    grid g;
    grid_init(&g, ndim, L, NULL, cplx);
    if (dim < 0 || dim > ndim) return 1;
    if (id < 0 || id >= g.ncell[dim] * g.N || !id_valid(&g, dim, id)) return 1;
    /* vertices (no values needed) */
    int64_t av = dim ? id / g.ncell[dim] : id;
    int idx = dim ? (int)(id % g.ncell[dim]) : 0;
    int64_t a[3];
    coords(&g, av, a);
    if (cplx) {
        const int *m = t5_tab[parity3(a)][dim][idx];
        for (int j = 0; j <= dim; j++) {
            int64_t c[3];
            for (int ax = 0; ax < 3; ax++) c[ax] = a[ax] + ((m[j] >> ax) & 1);
            verts_out[j] = vid(&g, c);
        }
        return 0;
    }
    verts_out[0] = av;
    for (int j = 0; j < dim; j++) {
        int m = chain_tab[ndim][dim][idx][j];
        int64_t c[3];
        for (int ax = 0; ax < 3; ax++) c[ax] = a[ax] + ((m >> ax) & 1);
        verts_out[j + 1] = vid(&g, c);
    }
    return 0;
}

int orc_simplex_vertices(int ndim, const int64_t *L, int dim, int64_t id, int64_t *verts_out)
{
    return orc_simplex_vertices2(ndim, L, dim, id, 0, verts_out);
}

int64_t orc_cells_per_vertex2(int ndim, int dim, int cplx)
{
    if (cplx) {
        build_t5();
        return (ndim == 3 && dim >= 0 && dim <= 3) ? t5_count[dim] : 0;
    }
    build_chains(ndim);
    return dim == 0 ? 1 : chain_count[ndim][dim];
}

int64_t orc_cells_per_vertex(int ndim, int dim)
{
    return orc_cells_per_vertex2(ndim, dim, 0);
}
