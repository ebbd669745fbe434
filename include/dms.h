/*
 * dms.h -- C ABI of the B200-native Discrete Morse Sandwich front end.
 *
 * Computes, for a float32 scalar field on a Freudenthal-triangulated regular grid
 * (1D/2D/3D), the pieces of arXiv 2206.13932 ("Discrete Morse Sandwich"):
 *   dms_order        global vertex order              PAPER.md 1368-1372 (Sec. 2.1), 1069-1071 (Sec. 7.1)
 *   dms_gradient     lower-star discrete gradient     PAPER.md 1965-1971 (Sec. 2.6), 272-294 (Sec. 4.1c)
 *   dms_critical     critical simplices C_k, sorted   PAPER.md 317-362 (Alg. 2)
 *   dms_diagram0     D0 (minimum-saddle pairs)        PAPER.md 2481-2685 (Sec. 5.1)
 *   dms_diagram_top  D_{d-1} (saddle-maximum pairs)   PAPER.md 2690-2825 (Sec. 5.2)
 *   infinite classes (inside the two diagram calls)   PAPER.md 2860-2878 (Sec. 6)
 *   dms_diagram1     D1 (3D) by PairCriticalSimplices PAPER.md 364-417 (Alg. 3), 1125-1150 (Sec. 7.2)
 *   dms_generators   persistent 1-cycle generators    PAPER.md 1188-1215 (Sec. 9)
 * Everything runs in hand-written CUDA kernels for sm_100a on the caller's stream;
 * there is no CPU fallback.  Readings of the paper's silent points (tie-break,
 * simplex ids, boundary handling, output order) are listed in DESIGN.md.
 *
 * Conventions
 *   grid      dims[0] = Lx (fastest), dims[1] = Ly, dims[2] = Lz; vertex id
 *             v = x + Lx*(y + Ly*z); ndim in {1,2,3}, every used extent >= 2, N < 2^31.
 *   order     K(u) < K(v)  iff  f(u) < f(v) (IEEE, so -0 == +0) or (f(u) == f(v) and u < v).
 *   simplex   anchored id = C_k * vid(anchor) + chain index,
 *             C_k = cells per vertex: 3D 1/7/12/6, 2D 1/3/2, 1D 1/1 for k = 0..d.
 *   lex order the lexicographic order of PAPER.md 1380-1414 (decreasing K tuples).
 *
 * Memory ownership
 *   d_f is BORROWED (device, read-only) and must stay valid until dms_destroy.
 *   d_rank / d_grad are CALLER-OWNED device buffers written asynchronously.
 *   Arrays returned through pointer-to-pointer arguments are LIBRARY-OWNED device
 *   buffers, valid until the next call that recomputes them or dms_destroy.
 *   The workspace is allocated at dms_create.
 *
 * Errors
 *   Every entry point returns a dms_status; no C++ exception crosses the ABI.
 *   With DMS_CHECK_INVARIANTS=1 in the environment (debug), dms_run_all* also verify the
 *   identities every result satisfies (ranks a permutation, Euler characteristic 1, every
 *   extremum dying once, the D1 saddle counts of both sandwich sides) and return
 *   DMS_ERR_INVARIANT on a violation.
 *   Argument/shape errors are synchronous.  A NaN in f is detected on the device and
 *   reported by the next synchronising call (dms_critical, dms_diagram0,
 *   dms_diagram_top, dms_sync) as DMS_ERR_NAN.  CUDA errors -> DMS_ERR_CUDA
 *   (sticky: later calls on the same context return DMS_ERR_STATE).
 *
 * Synchronisation and threads
 *   Only calls returning host counts (h_count, h_n) synchronise the stream (and
 *   dms_run_all / dms_run_all_host, which wait for the critical counts and for each
 *   union-find's convergence flag).  The
 *   library also uses two internal streams of its own (the vertex order; D0 beside
 *   D_{d-1}); their work is joined into the caller's stream before a call returns.
 *   A context is not thread-safe: calls on one context must not overlap; distinct
 *   contexts are independent.
 *
 * Size limits
 *   N < 2^31 and (top cells per vertex) * N < 2^31, checked by dms_create
 *   (DMS_ERR_TOO_LARGE) before any device work; the largest 3D cube is about 710^3.
 */
#ifndef DMS_H
#define DMS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dms_ctx dms_ctx; /* opaque */

typedef enum {
    DMS_OK = 0,
    DMS_ERR_ARG = 1,        /* NULL pointer, bad enum                           */
    DMS_ERR_DEGENERATE = 2, /* ndim not in {1,2,3} or a used extent < 2 */
    DMS_ERR_NAN = 3,        /* f contains NaN                           */
    DMS_ERR_TOO_LARGE = 4,  /* N >= 2^31 or simplex ids overflow int32 indexing  */
    DMS_ERR_STATE = 5,      /* sticky earlier error, or an unsupported mode      */
    DMS_ERR_CUDA = 6,       /* a CUDA call failed                               */
    DMS_ERR_OOM = 7,        /* device allocation failed                          */
    DMS_ERR_INVARIANT = 8   /* an internal invariant check failed                */
} dms_status;

/* The simplicial complex on the grid.  DMS_COMPLEX_FREUDENTHAL: the Kuhn/Freudenthal
 * triangulation (PAPER.md 1360-1366; 1D/2D/3D; in 2D the paper's own "two triangles" per
 * cell).  DMS_COMPLEX_5TET (3D only): five tetrahedra per cube, the subdivision of
 * the paper's benchmark volumes (PAPER.md 662-664, Sec. 8.1; reading Z21): the
 * cube with minimum corner a is cut into the central tetrahedron on its corners of even
 * coordinate sum and the four corner tetrahedra at the others.  Anchored ids: the
 * component-wise minimum of the simplex, C_k = 1/6/10/5. */
typedef enum {
    DMS_COMPLEX_FREUDENTHAL = 0,
    DMS_COMPLEX_5TET = 1
} dms_complex;

typedef enum {
    DMS_BOUNDARY_EXACT = 0, /* virtual maximum on the boundary (PAPER.md 2787-2825)          */
    DMS_BOUNDARY_IGNORE = 1 /* no virtual maximum (PAPER.md 2822-2825, App. A 2927-2949)      */
} dms_boundary;

/* One persistence pair (PAPER.md 1641-1697).  death_id = -1 marks an infinite class
 * (Sec. 6), whose death_value is f* = max f. Values are f at the simplices' highest
 * vertices (PAPER.md 1662-1664). 32 bytes. */
typedef struct {
    int64_t birth_id, death_id;         /* anchored simplex ids                 */
    int32_t birth_vertex, death_vertex; /* highest vertex of each (-1 infinite) */
    float birth_value, death_value;
} dms_pair;

/* Create a context for the field d_f (device float32, N values, x fastest) on the
 * CUDA stream `stream` (cudaStream_t, may be 0).  Validates the shape synchronously
 * and allocates the device workspace. */
dms_status dms_create(const int64_t dims[3], int ndim, const float* d_f, void* stream, dms_ctx** out);

/* dms_create on the complex `cplx` (dms_complex; DMS_COMPLEX_5TET needs ndim = 3, else
 * DMS_ERR_ARG).  Every call below works on both complexes, except dms_diagram1,
 * dms_generators and dms_unpaired_saddles(which = 2), which return DMS_ERR_STATE on the
 * five-tetrahedra complex (its D1 is in the oracle only).  Five-tetrahedra gradient
 * layout (16 bytes per vertex, one byte per cell indexed by cell id): [0, N) vertex codes
 * (star slot of the paired edge, 0xFF minimum), [N, 11N) triangle codes, [11N, 16N)
 * tetrahedron codes (j < dim + 1: paired with the facet omitting vertex j of the cell's
 * ascending-mask vertex list, 0xFE: paired with a cofacet, 0xFF: critical). */
dms_status dms_create2(const int64_t dims[3], int ndim, const float* d_f, void* stream, dms_complex cplx,
                       dms_ctx** out);

/* Vertex order (PAPER.md 1368-1372; Sec. 7.1 "global sort"): d_rank[v] = number of
 * vertices u with K(u) < K(v), i.e. a key-value radix sort of (value, index).
 * d_rank: caller-owned device int32[N]; it must stay valid until the next
 * dms_gradient / dms_run_all* call has been synchronised (the critical sort keys read
 * it).  Clears the context's NaN flag first (the flag describes the current field).
 * Asynchronous. */
dms_status dms_order(dms_ctx* ctx, int32_t* d_rank);

/* Bytes of the packed gradient: 3D 16 B/vertex (both complexes), 2D 2 B/vertex, 1D 1 B/vertex. */
size_t dms_gradient_bytes(const dms_ctx* ctx);

/* Lower-star discrete gradient (Robins et al. ProcessLowerStars, PAPER.md 1965-1971)
 * of every vertex, plus the critical simplices of every lower star (Alg. 2).
 * d_grad: caller-owned device buffer of dms_gradient_bytes(ctx) bytes, one packed
 * word per vertex encoding, for every simplex of the vertex's lower star that is the
 * head of a discrete vector, which facet it is paired with (layout: DESIGN.md
 * "Gradient words").  3D Freudenthal, 16 bytes (two uint64) per vertex x, in terms of the
 * star slots of x (neighbours by increasing linear offset): lo bits 4w..4w+3 (w < 14) =
 * 1 + the slot u of the third vertex of the triangle (x, n_w, n_u) that edge (x, n_w) is
 * paired with (0: none), lo bits 56-59 = the edge slot x is paired with (15: x is
 * critical); hi bits 2q..2q+1 (q < 24) = 1 + j if tetrahedron slot q is paired with its
 * facet j (0: not the head of a vector), hi bits 48-61 = the mask of lower neighbours.
 * dms_decode_pairs turns the words into (tail, head) simplex ids.  Independent of dms_order (it compares values and indices
 * directly); dms_critical needs both and runs dms_order if it has not run.
 * Each gradient pass consumes the order computed since the previous pass: calling
 * dms_gradient again without a new dms_order (a changed field) makes the next call
 * that needs ranks recompute the order into a library-owned buffer.  A gradient pass
 * not preceded by dms_order clears the NaN flag.  Asynchronous. */
dms_status dms_gradient(dms_ctx* ctx, void* d_grad);

/* Critical simplices C_0..C_d, each sorted by the lexicographic order (Alg. 2 l. 13,
 * PAPER.md 357-359).  h_count[k] = |C_k| (k > d: 0); d_ids_out[k] = library-owned
 * device int64 array of anchored ids.  Synchronises. */
dms_status dms_critical(dms_ctx* ctx, int64_t h_count[4], const int64_t* d_ids_out[4]);

/* D0 (Sec. 5.1): pairs (minimum, critical edge) in increasing death-edge lex order,
 * then the one infinite class (global minimum, f*).  *d_pairs: library-owned device
 * array of *h_n records.  Synchronises. */
dms_status dms_diagram0(dms_ctx* ctx, const dms_pair** d_pairs, int64_t* h_n);

/* D_{d-1} (Sec. 5.2): pairs (critical (d-1)-simplex, critical d-simplex) in
 * decreasing birth lex order.
 * mode (a dms_boundary value):
 *   DMS_BOUNDARY_EXACT  a virtual maximum, older than every maximum, on the outer
 *       boundary (PAPER.md 2810-2817): every maximum dies; equals the boundary-matrix
 *       reduction.  For d = 1 the infinite class of the global minimum follows (and the
 *       records are D0's, listed by birth: for d = 1 the two are one diagram).
 *   DMS_BOUNDARY_IGNORE no virtual maximum (PAPER.md 2822-2825, App. A 2927-2949;
 *       DESIGN.md reading Z7): an arc whose stable-set tracing leaves through the
 *       boundary is dropped (its saddle stays unpaired), the global maximum stays
 *       unpaired -- its class is D0's infinite (global min, f*) record, "paired by
 *       convention to the global minimum" -- and there are no infinite records.
 *       Computed from the exact mode's arcs (run first if needed); the exact results
 *       and the D1 hand-off (dms_unpaired_saddles) are unchanged.
 * Other values -> DMS_ERR_ARG.  Synchronises. */
dms_status dms_diagram_top(dms_ctx* ctx, dms_boundary mode, const dms_pair** d_pairs, int64_t* h_n);

/* Critical saddles left unpaired (the "sandwich" hand-off, PAPER.md 1125-1155:
 * PairCriticalSimplices only sees the critical simplices that D0 and D_{d-1} did not
 * pair).  which = 0: critical edges unpaired by D0 (the 1-cycle creators, Sec. 5.1(d),
 * PAPER.md 2660-2685); which = 1: critical (d-1)-simplices unpaired by D_{d-1}
 * (Sec. 5.2, PAPER.md 2767-2769; in 3D the 1-cycle destroyers); which = 2 (3D):
 * critical edges still unpaired after D1 (infinite D1 classes, Sec. 6; none on a grid,
 * which is a ball), runs dms_diagram1 if needed.  Ascending lex order; library-owned
 * device int64 anchored ids.  Synchronises. */
dms_status dms_unpaired_saddles(dms_ctx* ctx, int which, const int64_t** d_ids, int64_t* h_n);

/* D1 of a 3D field (Alg. 3 "PairCriticalSimplices", PAPER.md 364-417, with boundary
 * caching PAPER.md 452-501, on the saddles of dms_unpaired_saddles 0 and 1): for each
 * critical triangle sigma left unpaired by D2, in increasing lexicographic order, the
 * pair (tau, sigma), tau = the highest edge of the propagated Boundary(sigma) once it is
 * unpaired.  Computed in parallel rounds with temporary pairs replaced by earlier
 * claimants (PAPER.md 1136-1150); the pairs equal the sequential
 * algorithm's.  *d_pairs: library-owned device array of *h_n records, one per 2-saddle,
 * in increasing death order (no infinite records: see dms_unpaired_saddles 2).
 * ndim != 3 -> DMS_ERR_ARG (2D: D1 is D_{d-1}; 1D: no D1).  Runs the diagrams it needs.
 * An internal inconsistency -> DMS_ERR_INVARIANT.  Synchronises. */
dms_status dms_diagram1(dms_ctx* ctx, const dms_pair** d_pairs, int64_t* h_n);

/* Persistent 1-cycle generators (Sec. 9, PAPER.md 1188-1215): for D1 pair i of
 * dms_diagram1, the earliest 1-cycle homologous to the boundary of its 2-saddle -- the
 * Boundary(sigma) Alg. 3 holds when it stops -- as anchored edge ids in ascending
 * lexicographic order: edges d_edges[d_off[i] .. d_off[i+1]).  d_off: library-owned
 * device int64[*h_n + 1]; d_edges: library-owned device int64[d_off[*h_n]].  Equal to
 * the sequential algorithm's columns (a second round-based pass with the final pairs).
 * 3D only (DMS_ERR_ARG otherwise).  Synchronises. */
dms_status dms_generators(dms_ctx* ctx, const int64_t** d_off, const int64_t** d_edges, int64_t* h_n);

/* Run the whole front end (order, gradient, critical lists, D0, D_{d-1}); the vertex
 * order runs on an internal second stream concurrently with the gradient and is joined
 * before the critical sort.  The host synchronises to read the critical and pair counts.  Results are read with the calls above afterwards.
 * d_rank / d_grad may be NULL (library-owned scratch). */
dms_status dms_run_all(dms_ctx* ctx, int32_t* d_rank, void* d_grad);

/* dms_run_all with the field supplied in HOST memory: h_f (N float32, x-fastest, the
 * layout of dms_create) is uploaded into the device field buffer given to dms_create
 * (which this call overwrites) in slabs of whole planes, and the gradient of each slab
 * starts as soon as the slab and its upper halo plane are on the device, so the
 * host-to-device transfer overlaps the gradient; the vertex order follows the upload
 * on the internal second stream.  h_f should be page-locked (cudaHostAlloc /
 * torch pin_memory) for the copies to be asynchronous; the caller keeps it unchanged
 * until the next synchronising call.  Same results and errors as dms_run_all. */
dms_status dms_run_all_host(dms_ctx* ctx, const float* h_f, int32_t* d_rank, void* d_grad);

/* Wait for the stream and report a pending device-side error (NaN, overflow). */
dms_status dms_sync(dms_ctx* ctx);

/* Host-side decode of packed gradient words of vertices [v0, v1) into discrete
 * vectors (tail dim, tail id, head id), int64 triples.  h_words: host copy of the
 * words of those vertices.  Returns the number of triples written (<= cap), or -1. */
int64_t dms_decode_pairs(const int64_t dims[3], int ndim, const void* h_words, int64_t v0, int64_t v1,
                         int64_t* h_triples, int64_t cap);

/* dms_decode_pairs on either complex.  Five tetrahedra: h_words is the WHOLE gradient
 * buffer (16 N bytes) and the triples are the vectors whose head cell is anchored at a
 * vertex of [v0, v1) (the vertex itself for vertex -> edge vectors). */
int64_t dms_decode_pairs2(const int64_t dims[3], int ndim, dms_complex cplx, const void* h_words, int64_t v0,
                          int64_t v1, int64_t* h_triples, int64_t cap);

/* Copy `bytes` between device/host buffers on the context's stream and wait
 * (cudaMemcpyDefault); used by the binding to move library-owned results. */
dms_status dms_copy(dms_ctx* ctx, void* dst, const void* src, size_t bytes);

/* Per-stage device timing with CUDA events recorded on the context's stream.
 * enable != 0 starts recording (and clears the accumulators); dms_stage_ms waits for
 * the stream and writes the accumulated milliseconds of stages
 * 0 order, 1 gradient (+ compaction), 2 critical sort, 3 D0, 4 D_{d-1},
 * 5 gradient kernel alone, 6 the number of timed gradient launches,
 * 7 D0 v-path tracing, 8 D_{d-1} dual tracing, 9 D0 union-find, 10 D_{d-1} union-find,
 * 11 D1 pairs, 12 D1 generators. */
dms_status dms_set_timing(dms_ctx* ctx, int enable);
dms_status dms_stage_ms(dms_ctx* ctx, double ms_out[13]);

/* Number of kernel launches issued by this context so far (bench accounting). */
int64_t dms_launch_count(const dms_ctx* ctx);

/* Last error message of the context (static storage of the context). */
const char* dms_last_error(const dms_ctx* ctx);

/* Free the context and every library-owned buffer. NULL is a no-op. */
void dms_destroy(dms_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* DMS_H */
