// dms.cu -- C-ABI entry points (include/dms.h) and host orchestration.
//
// One context = one field on the caller's stream (plus two internal streams).  The
// pipeline (Fig. 4 overview, 1236-1332, restricted to the front end):
//   order    radix sort of (ordered f, index) -> rank, on the      (Sec. 2.1, 7.1)
//            second stream beside the gradient
//   gradient k_gradient_pool<3> / k_gradient_lut2 / k_gradient1     (Sec. 2.6, Alg. 2)
//            (+ appended critical records)
//   critical radix sort of each C_k by its lexicographic key       (Alg. 2 l. 13)
//   D0       node map, k_d0_arcs, union-find rounds, emission      (Sec. 5.1, 6)
//   D_{d-1}  node map, memoised work-queue chases, union-find      (Sec. 5.2, 6)
//            rounds, emission; D0 runs on a third stream beside it (Sec. 7.2)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <new>
#include <utility>
#include <vector>

#include "../../include/dms.h"
#include "common.cuh"
#include "order.cuh"
#include "onesweep.cuh"
#include "diag.cuh"
#include "path1d.cuh"
#include "d1.cuh"
#include "grad.cuh"
#include "sort.cuh"
#include "star.cuh"
#include "star_build.cuh"
#include "tet5.cuh"

using namespace dms;

static_assert(sizeof(PairRec) == sizeof(dms_pair), "pair layout");

namespace {

__global__ void k_emit_inf_k(Geo3 g, int dim, const int64_t* id_ptr, const unsigned long long* kmax, PairRec* slot) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const StarTab& S = *g.tab;
    PairRec r;
    r.birth_id = *id_ptr;
    const int64_t bv = max_vertex(g, S, dim, r.birth_id);
    r.birth_vertex = (int32_t)bv;
    r.birth_value = g.f[bv];
    r.death_id = -1;
    r.death_vertex = -1;
    r.death_value = g.f[(int64_t)(*kmax & 0xffffffffull)];  // f* = f at the highest vertex
    *slot = r;
}

// 1D, exact mode: D_{d-1} listed from D0.  For d = 1 the two are the same diagram (the
// dimension-0 pairs of the one lexicographic filtration, PAPER.md 2736-2746; both
// computations reproduce the boundary-matrix reduction at simplex level), so
// the records are D0's, ordered by birth in decreasing order (Z11) instead of by death:
// record of the minimum of age a (its position in C_0) -> slot n0 - 1 - a; the global
// minimum (a = 0, D0's infinite record) comes last, and is the one unpaired minimum.
__global__ void k_dtop_from_d0(const PairRec* __restrict__ d0, int64_t n0, const int32_t* __restrict__ node_of0,
                               const int32_t* __restrict__ age, PairRec* __restrict__ out, const int64_t* c0,
                               int64_t* unp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) unp[0] = c0[0];
    if (i >= n0) return;
    const PairRec r = d0[i];
    out[n0 - 1 - age[node_of0[r.birth_vertex]]] = r;
}

// the infinite class with its slot after the np finite pairs, np read on the device from
// the pair scan (np = scan end + last flag)
__global__ void k_emit_inf_dev(Geo3 g, int dim, const int64_t* id_ptr, const unsigned long long* kmax, PairRec* base,
                               const uint32_t* pos, const uint32_t* flags, int64_t m) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t np = (int64_t)pos[m - 1] + flags[m - 1];
    const StarTab& S = *g.tab;
    PairRec r;
    r.birth_id = *id_ptr;
    const int64_t bv = max_vertex(g, S, dim, r.birth_id);
    r.birth_vertex = (int32_t)bv;
    r.birth_value = g.f[bv];
    r.death_id = -1;
    r.death_vertex = -1;
    r.death_value = g.f[(int64_t)(*kmax & 0xffffffffull)];
    base[np] = r;
}

struct UFBuf {
    int32_t *arc_a = nullptr, *arc_b = nullptr, *out = nullptr, *list = nullptr;
    int4 *rec0 = nullptr, *rec1 = nullptr;  // union-find live arc records
    int4* rsrc = nullptr;                    // all arc records in key order (batched rounds)
    int32_t* live2 = nullptr;
    int32_t* outp = nullptr;   // out in processing order
    uint32_t *key = nullptr, *inv_a = nullptr;  // per arc (emission order)
    int32_t* age = nullptr;                     // per node (emission order)
    int* nlive = nullptr;  // two device counters
    int* h_status = nullptr;  // pinned: the union-find's convergence status
    uint32_t* h_cnt = nullptr;  // pinned: [0..1] last scan position + last flag of the unpaired
                                //   scan, [2..3] the same for the pair scan
    int* trace = nullptr;  // [64] union-find round trace
    int32_t* parent = nullptr;
    unsigned long long* best = nullptr;
    uint32_t *flags = nullptr, *pos = nullptr;
    int64_t cap_arcs = 0, cap_nodes = 0;
    int64_t last_m = 0, last_grid = 0, last_batch = 0;  // diagnostics of the last launch
};

// 1D closed-form union-find scratch (path1d.cuh), one per diagram
struct PathBuf {
    uint32_t* sage = nullptr;
    unsigned long long* sarc = nullptr;
    unsigned long long *lw = nullptr, *rw = nullptr, *dw = nullptr, *bnd = nullptr, *tspan = nullptr;
    uint8_t* unres = nullptr;
    int32_t *pre = nullptr, *suf = nullptr, *npre = nullptr, *nsuf = nullptr;
    uint32_t* tmin = nullptr;
    int* bad = nullptr;
    int* h_bad = nullptr;
    int64_t cap = 0, capb = 0;
    bool used = false;  // the last union-find of this diagram ran here (finish checks it)
};

// D1 (d1.cuh): grow-only buffers
struct D1Buf {
    int32_t* order = nullptr;                 // [N] inverse of rank
    unsigned long long* hkey = nullptr;       // hash of the positive 1-saddles
    int32_t* hval = nullptr;
    int64_t hcap = 0;
    int32_t *owner = nullptr, *stop = nullptr, *done = nullptr, *col_len = nullptr, *big = nullptr;
    int32_t* act[2] = {nullptr, nullptr};
    unsigned long long* claim = nullptr;
    long long* col_off = nullptr;
    uint8_t* status = nullptr;
    unsigned long long* arena = nullptr;
    unsigned long long arena_cap = 0;
    int32_t* ctr = nullptr;                   // [0] nbig, [1] grab, [2] nnext, [3] err; [4..5] arena top (u64),
                                              // [6..13] first failure (4 x i64), [14] deps, [15] changed,
                                              // [16] snapshots
    int32_t* h_ctr = nullptr;                 // pinned copy
    uint32_t *flags = nullptr, *pos = nullptr;
    PairRec* pairs = nullptr;
    int64_t *un1 = nullptr, *gen_off = nullptr, *gen = nullptr;
    int64_t n0 = 0, nsig = 0, nun1 = 0, ngen = 0;
    int64_t cap0 = 0, capsig = 0, capgen = 0, capN = 0;
    int rounds[2] = {0, 0};
    unsigned* stats = nullptr;                // DMS_D1_STATS: [3 * capsig] per-sigma counters
    int4* deps = nullptr;                     // phase-1 column additions (taint pass)
    int64_t capdeps = 0;
    uint32_t* taint = nullptr;
    uint32_t* first_bad = nullptr;            // first non-sequential column addition per sigma
    unsigned long long* best = nullptr;       // restart snapshot per tainted sigma
    int32_t* nadd = nullptr;
    D1Snap* snaps = nullptr;                  // phase-1 stored columns (restart points)
    int64_t capsnaps = 0;
    int64_t ntaint = 0, nrestart = 0;
    bool snaps_ok = true;                     // phase 1 kept every stored column (no collection)
    D1Tab* tab = nullptr;                     // device copy of the propagation tables
};

// a second issue lane (stream + scan scratch + pinned scratch): D0 runs on it beside
// D_{d-1} (PAPER.md 1124: the two diagrams are computed concurrently)
struct Lane {
    cudaStream_t st = nullptr;
    SortScratch ss;
    int* tile_ctr = nullptr;
    unsigned long long* h_pinned = nullptr;
};

}  // namespace

#ifndef DMS_SLABS
#define DMS_SLABS 16
#endif
constexpr int kSlabs = DMS_SLABS;  // dms_run_all_host: at most this many upload slabs

struct dms_ctx {
    int ndim = 0;
    int cplx = DMS_COMPLEX_FREUDENTHAL;  // DMS_COMPLEX_5TET: five tetrahedra per cube (tet5.cuh)
    T5Tab* dt5 = nullptr;                // its tables (device)
    int64_t L[3] = {1, 1, 1};
    int64_t N = 0;
    const float* f = nullptr;
    cudaStream_t st = nullptr;
    cudaStream_t st2 = nullptr;          // the vertex order runs here, beside the gradient
    cudaEvent_t ev_in = nullptr, ev_order = nullptr;
    cudaEvent_t ev_slab[kSlabs] = {};  // dms_run_all_host: upload slabs
    Lane lane3;                   // D0's lane when the diagrams run concurrently
    Lane lane4;                   // D_{d-1}'s trace beside the critical sort
    bool early_traces = false;    // dms_run_all*: trace D0 / D_{d-1} beside the critical sort
    int order_ctas_beside = 1;    // CTAs per SM of the order's persistent grid beside the 3D gradient
    int os_defer_from = 4;        // one-sweep order: passes [os_defer_from, 4) + the rank pass wait for run_order_rest
    bool os_deferred = false;     // ... and are still to be issued
    int os_resume = 4;            // first deferred pass
    cudaEvent_t ev_grad2 = nullptr;
    bool traced[2] = {false, false};
    cudaEvent_t ev_grad = nullptr, ev_trace[2] = {nullptr, nullptr};
    cudaEvent_t ev_crit = nullptr, ev_d0 = nullptr;
    bool half = false;            // concurrent diagrams: the cooperative union-find grids use half the GPU
    cudaEvent_t t_diag[2] = {};   // stage timers spanning issue .. finish
    bool order_pending = false;          // st must wait ev_order before using ranks
    int64_t ncell[4] = {1, 0, 0, 0};
    StarTab htab;
    StarTab* dtab = nullptr;
    ChaseTab* dctab = nullptr;  // dual-chase transitions (device)
    GradLut* dlut3 = nullptr;   // 3D gradient kernel's union masks (device)
    // caller or scratch buffers
    int32_t* rank = nullptr;
    void* grad = nullptr;
    int32_t* rank_scratch = nullptr;
    void* grad_scratch = nullptr;
    // order sort
    uint32_t *okeys[2] = {nullptr, nullptr}, *ovals[2] = {nullptr, nullptr};
    // order in one sweep (onesweep.cuh)
    uint32_t* os_hist = nullptr;              // [4 * 256] digit histograms -> exclusive starts
    uint32_t* os_wcur = nullptr;              // [kOsWinMax] window cursors
    int* os_tctr = nullptr;                   // [4] dynamic tile counters
    unsigned long long* os_status = nullptr;  // [tiles * 256] look-back words
    uint2* os_wbuf = nullptr;                 // [N] (v, p) pairs by window (large N)
    uint32_t os_epoch = 0;
    SortScratch ss;
    // order by sample sort (order.cuh): B buckets, S samples
    int ord_B = 0, ord_S = 0;
    uint64_t* ord_keys = nullptr;                  // [N]
    uint16_t* ord_bid = nullptr;                   // [N]
    uint64_t* ord_skeys[2] = {nullptr, nullptr};   // [S]
    uint32_t* ord_svals[2] = {nullptr, nullptr};   // [S]
    uint64_t* ord_spl = nullptr;                   // [B]
    uint32_t *ord_counts = nullptr, *ord_offs = nullptr;  // [B * sms]
    // critical records
    int64_t cap[4] = {0, 0, 0, 0};
    int64_t* cid[2][4] = {};     // [0]: ids in emission order, [1]: ids in lexicographic order
    uint64_t* ckey[2][4] = {};
    unsigned* bm = nullptr;            // rank bitmap of the critical sorts
    uint32_t *bmcnt = nullptr, *bmpre = nullptr;
    uint32_t *ms_sidx = nullptr, *ms_slot = nullptr, *ms_cnt = nullptr, *ms_base = nullptr;  // [cap] star runs
    unsigned long long* ms_stage = nullptr;
    int64_t ms_cap = 0;
    uint32_t* cidx[2][4] = {};   // sort payload: emission index; perm = cidx[cur]
    int cur[4] = {0, 0, 0, 0};
    int64_t ncrit[4] = {0, 0, 0, 0};
    unsigned long long* status = nullptr;
    int64_t status_words = 0;
    int* tile_ctr = nullptr;
    uint32_t* chase_mark = nullptr;  // D_{d-1} chase stamps, one per top cell
    uint32_t* lut2 = nullptr;        // 2D: ProcessLowerStars result per star pattern
    unsigned long long* cw = nullptr;  // 3D: chase words (tet codes | lower mask << 48)
    uint32_t* cw2 = nullptr;           // 2D: chase words (triangle codes | lower mask << 12)
    uint8_t* vc = nullptr;             // 2D / 3D: vertex codes (D0 descent)
    int sms = 148;                   // multiprocessors of the context's device
    Lut2Off lut2off;
    uint32_t chase_gen = 0;
    unsigned long long* totals = nullptr;
    int* err = nullptr;
    unsigned long long* kmax = nullptr;
    unsigned long long* remaining = nullptr;
    unsigned long long* h_pinned = nullptr;  // small pinned host scratch
    // diagrams
    int32_t *node_of0 = nullptr, *node_oftop = nullptr;
    UFBuf uf[2];
    PairRec* pairs[2] = {nullptr, nullptr};
    int64_t npairs[2] = {0, 0};
    int64_t* unp[2] = {nullptr, nullptr};
    int64_t nunp[2] = {0, 0};
    bool nunp_async[2] = {false, false};  // nunp still in the pinned slot of uf[which]
    int npairs_async[2] = {0, 0};         // > 0: npairs = pinned pair count + (this - 1) infinite records
    int64_t cap_pairs[2] = {0, 0}, cap_unp[2] = {0, 0};  // grow-only result buffers
    // state
    bool order_fresh = false;  // an order computed since the last gradient pass
    bool have_order = false, have_grad = false, have_crit = false, have_d[2] = {false, false};
    bool have_d1 = false, have_gen = false;  // D1 pairs / generators of the current diagrams
    // 1D: the union-finds in closed form on the path graphs (path1d.cuh)
    uint32_t *t1base[2] = {nullptr, nullptr}, *t1cnt[2] = {nullptr, nullptr}, *t1scan[2] = {nullptr, nullptr};
    int64_t t1tiles = 0;
    bool t1_valid = false;           // the last gradient pass filled the per-CTA tables
    int64_t* pmap[2] = {nullptr, nullptr};  // spatial -> emission index of C_0 / C_1
    int64_t cap_pmap = 0;
    bool have_pmap = false;
    PathBuf pb[2];
    bool have_ign = false;                   // D_{d-1} in the "ignore" boundary mode
    bool dtop_short = false;                 // 1D: D_{d-1} was listed from D0 (run_dtop_from_d0), no dual union-find yet
    UFBuf uf_ign;
    PairRec* pairs_ign = nullptr;
    int64_t npairs_ign = 0, cap_ign = 0;
    D1Buf d1;
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[12];
    int64_t launches = 0;
    dms_status sticky = DMS_OK;
    char msg[256] = {0};
};

namespace {

// NVTX names of the stages (host-side ranges for Nsight Systems / ncu --nvtx)
const char* const kStageName[12] = {"dms order", "dms gradient", "dms critical", "dms D0", "dms Dtop", "dms gradient kernel",
                                    "dms D0 trace", "dms Dtop trace", "dms D0 union-find", "dms Dtop union-find",
                                    "dms D1 pairs", "dms D1 generators"};

// records a (start, stop) event pair on the context's stream around a stage (and an NVTX
// range on the host thread)
struct StageTimer {
    dms_ctx* c;
    int stage;
    cudaEvent_t a = nullptr;
    StageTimer(dms_ctx* c_, int s) : c(c_), stage(s) {
        nvtxRangePushA(kStageName[s < 12 ? s : 0]);
        if (c->timing && cudaEventCreate(&a) == cudaSuccess) cudaEventRecord(a, c->st);
    }
    ~StageTimer() {
        nvtxRangePop();
        if (!a) return;
        cudaEvent_t b = nullptr;
        if (cudaEventCreate(&b) == cudaSuccess) {
            cudaEventRecord(b, c->st);
            c->ev[stage].emplace_back(a, b);
        } else {
            cudaEventDestroy(a);
        }
    }
};

cudaEvent_t stage_begin(dms_ctx* c) {
    cudaEvent_t a = nullptr;
    if (c->timing && cudaEventCreate(&a) == cudaSuccess) cudaEventRecord(a, c->st);
    return a;
}
void stage_end(dms_ctx* c, int stage, cudaEvent_t a) {
    if (!a) return;
    cudaEvent_t b = nullptr;
    if (cudaEventCreate(&b) == cudaSuccess) {
        cudaEventRecord(b, c->st);
        c->ev[stage].emplace_back(a, b);
    } else {
        cudaEventDestroy(a);
    }
}

// swaps the context's issue resources with a lane's for a scope
struct LaneSwap {
    dms_ctx* c;
    Lane& L;
    LaneSwap(dms_ctx* c_, Lane& l) : c(c_), L(l) { swap(); }
    ~LaneSwap() { swap(); }
    void swap() {
        std::swap(c->st, L.st);
        std::swap(c->ss, L.ss);
        std::swap(c->tile_ctr, L.tile_ctr);
        std::swap(c->h_pinned, L.h_pinned);
    }
};

void clear_events(dms_ctx* c) {
    for (auto& v : c->ev) {
        for (auto& p : v) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
        v.clear();
    }
}

dms_status fail(dms_ctx* c, dms_status s, const char* what) {
    if (c) {
        std::snprintf(c->msg, sizeof c->msg, "%s", what);
        if (s == DMS_ERR_CUDA) c->sticky = s;
    }
    return s;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            char b_[200];                                                                \
            std::snprintf(b_, sizeof b_, "%s: %s", #call, cudaGetErrorString(e_));       \
            return fail(c, e_ == cudaErrorMemoryAllocation ? DMS_ERR_OOM : DMS_ERR_CUDA, b_); \
        }                                                                                \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, int64_t n) {
    *p = nullptr;
    if (n <= 0) n = 1;
    return cudaMalloc((void**)p, (size_t)n * sizeof(T));
}

inline unsigned grid_for(int64_t n, int block = kBlock) { return (unsigned)std::max<int64_t>(1, ceil_div(n, block)); }

Geo3 geo(const dms_ctx* c) {
    Geo3 g;
    g.ndim = c->ndim;
    g.Lx = (int32_t)c->L[0];
    g.Ly = (int32_t)c->L[1];
    g.Lz = (int32_t)c->L[2];
    g.N = c->N;
    for (int k = 0; k < 4; k++) g.ncell[k] = c->ncell[k];
    g.f = c->f;
    g.grad = c->grad;
    g.tab = c->dtab;
    g.ctab = c->dctab;
    g.cw = c->cw;
    g.cw2 = c->cw2;
    g.vc = c->vc;
    g.t5 = c->cplx == DMS_COMPLEX_5TET ? c->dt5 : nullptr;
    return g;
}

T5Geo t5geo(const dms_ctx* c) {
    T5Geo g;
    g.Lx = (int32_t)c->L[0];
    g.Ly = (int32_t)c->L[1];
    g.Lz = (int32_t)c->L[2];
    g.N = c->N;
    return g;
}

dms_status check_sticky(dms_ctx* c) {
    if (!c) return DMS_ERR_ARG;
    if (c->sticky != DMS_OK) return DMS_ERR_STATE;
    return DMS_OK;
}

dms_status alloc_crit(dms_ctx* c) {
    for (int b = 0; b < 2; b++)
        for (int k = 0; k <= c->ndim; k++) {
            cudaFree(c->cid[b][k]);
            cudaFree(c->ckey[b][k]);
            cudaFree(c->cidx[b][k]);
            CU(dalloc(&c->cid[b][k], c->cap[k]));
            CU(dalloc(&c->ckey[b][k], c->cap[k]));
            CU(dalloc(&c->cidx[b][k], c->cap[k]));
        }
    return DMS_OK;
}

dms_status alloc_uf(dms_ctx* c, UFBuf& u, int64_t arcs, int64_t nodes) {
    arcs = std::max<int64_t>(arcs, 1);
    nodes = std::max<int64_t>(nodes, 1);
    if (arcs > u.cap_arcs) {
        for (int4** p : {&u.rec0, &u.rec1, &u.rsrc}) {
            cudaFree(*p);
            CU(dalloc(p, arcs));
        }
        for (int32_t** p : {&u.arc_a, &u.arc_b, &u.out, &u.list, &u.live2, &u.outp}) {
            cudaFree(*p);
            CU(dalloc(p, arcs));
        }
        for (uint32_t** p : {&u.key, &u.inv_a}) {
            cudaFree(*p);
            CU(dalloc(p, arcs));
        }
        if (!u.nlive) CU(dalloc(&u.nlive, 8));
        if (!u.h_status && cudaMallocHost(&u.h_status, sizeof(int)) != cudaSuccess) return fail(c, DMS_ERR_OOM, "pinned");
        if (!u.h_cnt && cudaMallocHost(&u.h_cnt, 4 * sizeof(uint32_t)) != cudaSuccess) return fail(c, DMS_ERR_OOM, "pinned");
        if (!u.trace) CU(dalloc(&u.trace, 128 + 128));
        for (uint32_t** p : {&u.flags, &u.pos}) { cudaFree(*p); CU(dalloc(p, arcs)); }
        u.cap_arcs = arcs;
    }
    if (nodes > u.cap_nodes) {
        cudaFree(u.parent);
        cudaFree(u.best);
        cudaFree(u.age);
        CU(dalloc(&u.parent, nodes));
        CU(dalloc(&u.best, nodes));
        CU(dalloc(&u.age, nodes));
        u.cap_nodes = nodes;
    }
    return DMS_OK;
}

// The NaN flag describes the field of the current pass: every entry point that reads f
// (dms_order, dms_gradient, dms_run_all, dms_run_all_host) clears it on the caller's
// stream first, so a clean field after a NaN field gives DMS_OK.
dms_status clear_err(dms_ctx* c) {
    CU(cudaMemsetAsync(c->err, 0, sizeof(int), c->st));
    return DMS_OK;
}

dms_status read_err(dms_ctx* c) {
    int e = 0;
    CU(cudaMemcpyAsync(&e, c->err, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    if (e & 1) return fail(c, DMS_ERR_NAN, "NaN in the scalar field");
    return DMS_OK;
}

// ------------------------------------------------------------------ stages

// one-sweep order: the digit passes [p0, p1) on a persistent grid of `grid` CTAs, and after
// pass 3 the rank pass of the windowed form (the buffers and the histograms are in place)
dms_status os_passes(dms_ctx* c, int p0, int p1, unsigned grid, bool lb4) {
    const int64_t n = c->N;
    const int64_t tiles = ceil_div(n, (int64_t)kOsTile);
    static const long long win_env = getenv("DMS_RANK_WIN") ? atoll(getenv("DMS_RANK_WIN")) : -1;
    const bool windowed = win_env < 0 ? n >= (int64_t(1) << 23) : (win_env > 0 && n >= win_env);
    for (int p = p0; p < p1; p++) {
        if (++c->os_epoch >= 0xffffu) {  // epochs wrap: clear the look-back words
            CU(cudaMemsetAsync(c->os_status, 0, (size_t)tiles * 256 * 8, c->st));
            c->os_epoch = 1;
        }
        uint32_t* ki = p % 2 ? c->okeys[1] : c->okeys[0];
        uint32_t* vi = p % 2 ? c->ovals[1] : c->ovals[0];
        uint32_t* ko = p % 2 ? c->okeys[0] : c->okeys[1];
        uint32_t* vo = p % 2 ? c->ovals[0] : c->ovals[1];
        const uint32_t* db = c->os_hist + 256 * p;
        int* tc = c->os_tctr + p;
#define OS_PASS(FIRST, MODE, SHIFT)                                                                                  \
    do {                                                                                                             \
        if (lb4)                                                                                                     \
            k_os_pass<FIRST, MODE, 4><<<grid, kOsT, 0, c->st>>>(ki, vi, c->f, ko, vo, c->rank, c->os_wbuf, c->os_wcur, n, \
                                                               SHIFT, db, c->os_status, c->os_epoch, tc, tiles);    \
        else                                                                                                         \
            k_os_pass<FIRST, MODE, 1><<<grid, kOsT, 0, c->st>>>(ki, vi, c->f, ko, vo, c->rank, c->os_wbuf, c->os_wcur, n, \
                                                               SHIFT, db, c->os_status, c->os_epoch, tc, tiles);    \
    } while (0)
        if (p == 0) OS_PASS(true, 0, 0);
        else if (p < 3) OS_PASS(false, 0, 8 * p);
        else if (windowed) OS_PASS(false, 2, 24);
        else OS_PASS(false, 1, 24);
#undef OS_PASS
        c->launches++;
    }
    if (p1 == 4 && windowed) {
        k_os_rank<<<(unsigned)ceil_div(n, kBlock), kBlock, 0, c->st>>>(c->os_wbuf, n, c->rank);
        c->launches++;
    }
    CU(cudaGetLastError());
    return DMS_OK;
}

// the deferred passes of the one-sweep order (dms_run_all, DMS_ORDER_SPLIT): on the order's
// stream once the gradient kernel is done, on the full grid, beside the diagrams' tracing
dms_status run_order_rest(dms_ctx* c) {
    if (!c->os_deferred) return DMS_OK;
    c->os_deferred = false;
    if (!c->ev_grad2) CU(cudaEventCreateWithFlags(&c->ev_grad2, cudaEventDisableTiming));
    CU(cudaEventRecord(c->ev_grad2, c->st));
    CU(cudaStreamWaitEvent(c->st2, c->ev_grad2, 0));
    cudaStream_t main = c->st;
    c->st = c->st2;
    dms_status s;
    {
        StageTimer tm(c, 0);
        int per = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_os_pass<false, 0, 4>, kOsT, 0);
        const int64_t tiles = ceil_div(c->N, (int64_t)kOsTile);
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)c->sms * std::max(per, 1)));
        s = os_passes(c, c->os_resume, 4, grid, true);
    }
    c->st = main;
    if (s) return s;
    CU(cudaEventRecord(c->ev_order, c->st2));
    return DMS_OK;
}

dms_status run_order_on_stream(dms_ctx* c, int32_t* d_rank, bool beside_gradient = false) {
    StageTimer tm(c, 0);
    c->rank = d_rank ? d_rank : c->rank_scratch;
    CU(cudaMemsetAsync(c->kmax, 0, sizeof(unsigned long long), c->st));
    // Beside the (long, ALU-bound) 3D gradient the order's histogram / scatter passes run
    // on a tile-strided grid of 1-2 CTAs per SM, leaving the rest of every SM to gradient
    // CTAs (c4: 46.6 -> 45.3 ms; in 1D / 2D the order is the longer branch and keeps the
    // full grid).  DMS_ORDER_CTAS overrides (0: full grid).
    static const int octas_env = getenv("DMS_ORDER_CTAS") ? atoi(getenv("DMS_ORDER_CTAS")) : -1;
    // beside the closed-form 3D gradient, the one-sweep order on 1 CTA per SM (c4,
    // 1/2/3/full grid: 22.18 / 23.52 / 25.10 / 25.10 ms, order first, then the gradient:
    // 25.12 ms; c3 1/2/3: 6.52 / 6.59 / 6.70 ms)
    const int octas = octas_env >= 0 ? octas_env : (beside_gradient && c->ndim == 3 ? c->order_ctas_beside : 0);
    // DMS_ORDER_GRID: the persistent order grid in CTAs (finer than whole CTAs per SM; A/B)
    static const int ogrid_env = getenv("DMS_ORDER_GRID") ? atoi(getenv("DMS_ORDER_GRID")) : 0;
    const int64_t order_cap = (ogrid_env > 0 && beside_gradient && c->ndim == 3) ? ogrid_env
                              : octas > 0 ? (int64_t)c->sms * octas : 0;
    if (c->ord_B > 0) {  // sample sort (order.cuh)
        const int B = c->ord_B, S = c->ord_S, G = c->sms;
        static const int ocap_env = getenv("DMS_ORD_CAP") ? atoi(getenv("DMS_ORD_CAP")) : kOrdCap;  // tests: fallback path
        k_ord_sample<<<(unsigned)ceil_div(S, kBlock), kBlock, 0, c->st>>>(c->f, c->N, S, c->ord_skeys[0], c->ord_svals[0]);
        const int w = radix_sort<uint64_t, uint32_t, 8>(c->ord_skeys[0], c->ord_svals[0], c->ord_skeys[1], c->ord_svals[1],
                                                         S, 0, 64, c->ss, c->st, &c->launches);
        k_ord_splitters<<<(unsigned)ceil_div(B, kBlock), kBlock, 0, c->st>>>(c->ord_skeys[w], S, B, c->ord_spl);
        k_ord_count<<<G, kOrdT, (size_t)B * 12, c->st>>>(c->f, c->N, B, c->ord_spl, c->ord_bid, c->ord_counts, c->err,
                                                         c->kmax);
        scan_excl(c->ord_counts, c->ord_offs, (int64_t)B * G, c->ss, c->st, &c->launches);
        k_ord_scatter<<<G, kOrdT, (size_t)B * 4, c->st>>>(c->f, c->N, B, c->ord_bid, c->ord_offs, c->ord_keys);
        k_ord_bucket<<<B, kOrdT, kOrdBucketSmem, c->st>>>(c->ord_keys, c->N, B, G, c->ord_offs, c->rank,
                                                         std::min(ocap_env, kOrdCap));
        c->launches += 6;
        CU(cudaGetLastError());
        c->have_order = true;
        c->order_fresh = true;
        c->have_crit = c->have_d[0] = c->have_d[1] = c->have_d1 = c->have_gen = c->have_ign = c->dtop_short = false;
        return DMS_OK;
    }
    // one-sweep LSD radix sort (onesweep.cuh): one histogram read of f, four look-back
    // passes, the last one writing the ranks (by windows above 2^23 vertices)
    static const int os_env = getenv("DMS_ORDER_OS") ? atoi(getenv("DMS_ORDER_OS")) : 1;
    if (os_env) {
        dms_status s0;
        const int64_t n = c->N;
        const int64_t tiles = ceil_div(n, (int64_t)kOsTile);
        static const long long win_env = getenv("DMS_RANK_WIN") ? atoll(getenv("DMS_RANK_WIN")) : -1;
        const bool windowed = win_env < 0 ? n >= (int64_t(1) << 23) : (win_env > 0 && n >= win_env);
        const int nwin = (int)((n + (int64_t(1) << kWinBits) - 1) >> kWinBits);
        if (!c->os_hist) {
            CU(dalloc(&c->os_hist, 4 * 256));
            CU(dalloc(&c->os_wcur, kOsWinMax));
            CU(dalloc(&c->os_tctr, 4));
            CU(dalloc(&c->os_status, tiles * 256));
            CU(cudaMemsetAsync(c->os_status, 0, (size_t)tiles * 256 * 8, c->st));
            c->os_epoch = 0;
        }
        if (windowed && !c->os_wbuf) CU(dalloc(&c->os_wbuf, n));
        CU(cudaMemsetAsync(c->os_hist, 0, 4 * 256 * sizeof(uint32_t), c->st));
        CU(cudaMemsetAsync(c->os_tctr, 0, 4 * sizeof(int), c->st));
        int per = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_os_pass<false, 0, 4>, kOsT, 0);
        const int64_t res = (int64_t)c->sms * std::max(per, 1);
        const int64_t cap = order_cap > 0 ? std::min<int64_t>(order_cap, res) : res;
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, cap));
        k_os_hist<<<(unsigned)std::min<int64_t>(ceil_div(n, kOsT), (int64_t)c->sms * 8), kOsT, 0, c->st>>>(c->f, n, c->os_hist,
                                                                                                    c->err, c->kmax);
        k_os_scan<<<4, kOsT, 0, c->st>>>(c->os_hist, c->os_wcur, windowed ? nwin : 0);
        c->launches += 2;
        const int p_end = std::min(4, std::max(1, c->os_defer_from));
        if ((s0 = os_passes(c, 0, p_end, grid, order_cap == 0))) return s0;
        c->os_deferred = p_end < 4;
        c->os_resume = p_end;
        CU(cudaGetLastError());
        c->have_order = true;
        c->order_fresh = true;
        c->have_crit = c->have_d[0] = c->have_d[1] = c->have_d1 = c->have_gen = c->have_ign = c->dtop_short = false;
        return DMS_OK;
    }
    // key-value LSD radix sort of (ordered f, index); the first pass reads f directly
    // (and detects NaN / the highest vertex), the last pass writes rank[index]
#ifndef DMS_ORDER_ITEMS
#define DMS_ORDER_ITEMS 12
#endif
    // beside the 3D gradient, tiles of 16 items per thread (c4 44.66 -> 44.38 ms); on the
    // full grid (1D / 2D, or alone) 12 (16: c5a 9.04 -> 9.37, c5b 21.0 -> 22.2 ms)
    if (order_cap > 0)
        radix_sort<uint32_t, uint32_t, 16>(c->okeys[0], c->ovals[0], c->okeys[1], c->ovals[1], c->N, 0, 32, c->ss, c->st,
                                           &c->launches, c->rank, c->f, c->err, c->kmax, order_cap);
    else
        radix_sort<uint32_t, uint32_t, DMS_ORDER_ITEMS>(c->okeys[0], c->ovals[0], c->okeys[1], c->ovals[1], c->N, 0, 32, c->ss,
                                                        c->st, &c->launches, c->rank, c->f, c->err, c->kmax, order_cap);
    CU(cudaGetLastError());
    c->have_order = true;
    c->order_fresh = true;
    c->have_crit = c->have_d[0] = c->have_d[1] = c->have_d1 = c->have_gen = c->have_ign = c->dtop_short = false;  // the gradient does not depend on ranks
    return DMS_OK;
}

// concurrent = true: the order is enqueued on the second stream after the caller's
// stream (the field is ready), and the caller's stream waits for it only when ranks are
// needed (dms_critical's sort keys).  The order is memory-bound and the gradient kernel
// ALU-bound, so they overlap.
dms_status run_order(dms_ctx* c, int32_t* d_rank, bool concurrent = false) {
    if (!concurrent) {
        c->order_pending = false;
        return run_order_on_stream(c, d_rank);
    }
    CU(cudaEventRecord(c->ev_in, c->st));
    CU(cudaStreamWaitEvent(c->st2, c->ev_in, 0));
    cudaStream_t main = c->st;
    c->st = c->st2;
    dms_status s = run_order_on_stream(c, d_rank, true);
    c->st = main;
    if (s) return s;
    if (!c->os_deferred) CU(cudaEventRecord(c->ev_order, c->st2));  // (else by run_order_rest)
    c->order_pending = true;
    return DMS_OK;
}

dms_status join_order(dms_ctx* c) {
    if (!c->have_order) return run_order(c, nullptr);
    if (c->order_pending) {
        CU(cudaStreamWaitEvent(c->st, c->ev_order, 0));
        c->order_pending = false;
    }
    return DMS_OK;
}

// one gradient launch over the vertices [v0, v1) (the record counters are zeroed by the
// first launch of a pass, v0 == 0)
dms_status launch_gradient(dms_ctx* c, int64_t v0, int64_t v1) {
    const int64_t ntiles = ceil_div(v1 - v0, kBlock);
    if (v0 == 0) CU(cudaMemsetAsync(c->totals, 0, 4 * sizeof(unsigned long long), c->st));
    if (v1 <= v0) return DMS_OK;
    GradArgs A;
    A.v0 = v0;
    A.v1 = v1;
    A.f = c->f;
    A.Lx = (int32_t)c->L[0];
    A.Ly = (int32_t)c->L[1];
    A.Lz = (int32_t)c->L[2];
    A.divx.init((uint32_t)c->L[0]);
    A.divy.init((uint32_t)c->L[1]);
    A.N = c->N;
    A.tab = c->dtab;
    A.lut3 = c->dlut3;
    A.grad = c->grad;
    for (int k = 0; k < 4; k++) {
        A.crit_id[k] = c->cid[0][k];
        A.crit_key[k] = c->ckey[0][k];
        A.cap[k] = c->cap[k];
        A.ncell[k] = c->ncell[k];
    }
    A.totals = c->totals;
    A.err = c->err;
    A.cw = c->cw;
    A.cw2 = c->cw2;
    // 1D: the per-CTA record tables for the path union-finds (single launch over the line)
    c->t1_valid = c->ndim == 1 && c->t1base[0] && v0 == 0 && v1 == c->N;
    for (int k = 0; k < 2; k++) {
        A.t1base[k] = c->t1_valid ? c->t1base[k] : nullptr;
        A.t1cnt[k] = c->t1_valid ? c->t1cnt[k] : nullptr;
    }
    A.vc = c->vc;
    StageTimer tm(c, 5);
    if (c->cplx == DMS_COMPLEX_5TET) {  // the five-tetrahedra complex (tet5.cuh)
        T5Args B;
        B.f = c->f;
        B.Lx = A.Lx;
        B.Ly = A.Ly;
        B.Lz = A.Lz;
        B.N = c->N;
        B.v0 = v0;
        B.v1 = v1;
        B.tab = c->dt5;
        B.grad = static_cast<uint8_t*>(c->grad);
        for (int k = 0; k < 4; k++) {
            B.crit_id[k] = A.crit_id[k];
            B.crit_key[k] = A.crit_key[k];
            B.cap[k] = A.cap[k];
        }
        B.totals = c->totals;
        B.err = c->err;
        k_gradient_t5<<<(unsigned)(2 * ceil_div(v1 - v0, 2 * kT5Block)), kT5Block, 0, c->st>>>(B);  // CTA pairs per window
    } else if (c->ndim >= 2) {
        static const int lut_env = getenv("DMS_LUT2") ? atoi(getenv("DMS_LUT2")) : 1;
        // 3D: pools of 8 x 128 vertices per CTA, expanded in work order
        // DMS_GRAD_PAD: unused dynamic shared memory per 3D gradient CTA (bytes), to leave
        // SM room for the order's kernels beside it (A/B knob, default 0)
        static const int pad_env = getenv("DMS_GRAD_PAD") ? atoi(getenv("DMS_GRAD_PAD")) : 0;
        // DMS_GRAD_FAST=0: the queue-driven expansion instead of the closed form (A/B)
        static const int fast_env = getenv("DMS_GRAD_FAST") ? atoi(getenv("DMS_GRAD_FAST")) : 1;
        if (c->ndim == 3 && fast_env)
            k_gradient_pool<3, 8, 1, true><<<(unsigned)ceil_div(v1 - v0, 8 * kBlockG), kBlockG, (size_t)pad_env, c->st>>>(A);
        else if (c->ndim == 3)
            k_gradient_pool<3, 8><<<(unsigned)ceil_div(v1 - v0, 8 * kBlockG), kBlockG, (size_t)pad_env, c->st>>>(A);
        else if (c->lut2 && lut_env)
            k_gradient_lut2<<<(unsigned)std::min<int64_t>(ceil_div(v1 - v0, kBlock), c->sms * 8), kBlock, 0, c->st>>>(
                A, c->lut2, c->lut2off);
        else k_gradient_pool<2, 8><<<(unsigned)ceil_div(v1 - v0, 8 * kBlockG), kBlockG, 0, c->st>>>(A);
    } else {
        k_gradient1<<<(unsigned)ceil_div(v1 - v0, (int64_t)kBlock * kG1), kBlock, 0, c->st>>>(A);
    }
    c->launches++;
    CU(cudaGetLastError());
    return DMS_OK;
}

dms_status run_gradient(dms_ctx* c, void* d_grad) {
    // each gradient pass consumes the order computed since the previous one; a second
    // gradient pass without a new dms_order means a new field, so the order (ranks,
    // f*) is recomputed lazily into the library's own buffer
    if (!c->order_fresh) c->have_order = false;
    c->order_fresh = false;
    c->grad = d_grad ? d_grad : c->grad_scratch;
    StageTimer tm(c, 1);
    dms_status s = launch_gradient(c, 0, c->N);
    if (s) return s;
    c->have_grad = true;
    c->have_crit = c->have_d[0] = c->have_d[1] = c->have_d1 = c->have_gen = c->have_ign = c->dtop_short = false;
    return DMS_OK;
}

int bits_for(int64_t n) {
    int b = 0;
    while (b < 40 && ((int64_t)1 << b) < n) b++;
    return b;
}

const int64_t* crit_ids(dms_ctx* c, int k) { return c->cid[1][k]; }            // lexicographic order
const int64_t* crit_ids_emitted(dms_ctx* c, int k) { return c->cid[0][k]; }    // emission order
const uint32_t* crit_perm(dms_ctx* c, int k) { return c->cidx[c->cur[k]][k]; }  // sorted pos -> emission idx

dms_status d0_trace(dms_ctx* c);
dms_status dtop_trace(dms_ctx* c);
bool dtop1d_short(const dms_ctx* c);
dms_status run_dtop_from_d0(dms_ctx* c);

dms_status run_critical(dms_ctx* c) {
    if (!c->have_grad) {
        dms_status s = run_gradient(c, nullptr);
        if (s) return s;
    }
    dms_status s = join_order(c);  // ranks (and the NaN flag of the order pass) needed from here
    if (s) return s;
    StageTimer tm(c, 2);
    unsigned long long tot[4] = {0, 0, 0, 0};
    CU(cudaMemcpyAsync(tot, c->totals, sizeof tot, cudaMemcpyDeviceToHost, c->st));
    s = read_err(c);
    if (s) return s;
    bool overflow = false;
    for (int k = 0; k <= c->ndim; k++)
        if ((int64_t)tot[k] > c->cap[k]) { c->cap[k] = (int64_t)tot[k] + 1024; overflow = true; }
    if (overflow) {  // rare: grow the record buffers and recompute
        s = alloc_crit(c);
        if (s) return s;
        s = launch_gradient(c, 0, c->N);
        if (s) return s;
    }
    for (int k = 0; k <= c->ndim; k++) c->ncrit[k] = (int64_t)tot[k];
    // the diagrams' tracing needs the emitted critical cells but no ranks: in the run_all
    // flows it starts now on the diagram lanes, beside the sorts below
    c->traced[0] = c->traced[1] = false;
    // (measured: c2 1.23 -> 1.11 ms; the full configs within +-0.05 ms, the traces and the
    // sorts then contend -- so on for fields below 2^23 vertices; DMS_EARLY_TRACE=0/1 forces)
    static const int early_env = getenv("DMS_EARLY_TRACE") ? atoi(getenv("DMS_EARLY_TRACE")) : -1;
    static const int conc_env2 = getenv("DMS_CONCURRENT") ? atoi(getenv("DMS_CONCURRENT")) : 1;
    const bool early = early_env >= 0 ? early_env != 0 : c->N < (int64_t(1) << 23);
    if (c->early_traces && early && conc_env2 && c->lane3.st && c->lane4.st) {
        CU(cudaEventRecord(c->ev_grad, c->st));
        for (int w = 0; w < 2; w++) {
            if (w == 1 && dtop1d_short(c)) continue;  // (D_{d-1} is listed from D0)
            Lane& L = w == 0 ? c->lane3 : c->lane4;
            CU(cudaStreamWaitEvent(L.st, c->ev_grad, 0));
            LaneSwap ls(c, L);
            s = w == 0 ? d0_trace(c) : dtop_trace(c);
            if (s) return s;
            CU(cudaEventRecord(c->ev_trace[w], c->st));
            c->traced[w] = true;
        }
    }
    const int kbits = 12 + bits_for(c->N);
    static const int k32_env = getenv("DMS_CRIT_KEY32") ? atoi(getenv("DMS_CRIT_KEY32")) : 1;
    for (int k = 0; k <= c->ndim; k++) {
        k_iota<<<grid_for(c->ncrit[k]), kBlock, 0, c->st>>>(c->cidx[0][k], c->ncrit[k]);
        c->launches++;
        static const int bm_env = getenv("DMS_CRIT_BITMAP") ? atoi(getenv("DMS_CRIT_BITMAP")) : 1;
        if ((k == 0 || c->ndim == 1) && bm_env && c->ncrit[k] > 0) {
            // one cell per star: distinct rank keys -> positions by a rank bitmap (diag.cuh)
            const int64_t nw = (c->N + 31) / 32, m = c->ncrit[k];
            if (!c->bm) {
                CU(dalloc(&c->bm, nw));
                CU(dalloc(&c->bmcnt, nw));
                CU(dalloc(&c->bmpre, nw));
            }
            uint32_t* r = reinterpret_cast<uint32_t*>(c->ckey[1][k]);
            CU(cudaMemsetAsync(c->bm, 0, nw * sizeof(unsigned), c->st));
            k_bm_set<<<grid_for(m), kBlock, 0, c->st>>>(c->ckey[0][k], m, c->rank, r, c->bm);
            k_bm_popc<<<grid_for(nw), kBlock, 0, c->st>>>(c->bm, nw, c->bmcnt);
            scan_excl(c->bmcnt, c->bmpre, nw, c->ss, c->st, &c->launches);
            k_bm_place<<<grid_for(m), kBlock, 0, c->st>>>(r, m, c->bm, c->bmpre, c->cidx[1][k]);
            c->cur[k] = 1;
            k_gather_ids<<<grid_for(m), kBlock, 0, c->st>>>(c->cid[0][k], crit_perm(c, k), m, c->cid[1][k]);
            c->launches += 5;
            continue;
        }
        if ((k == 0 || c->ndim == 1) && k32_env) {
            // one cell per star (see below): sort 32-bit ranks, half the key bytes per pass;
            // the keys go to the second buffer (ka), the first one is the ping-pong buffer
            uint32_t* ka = reinterpret_cast<uint32_t*>(c->ckey[1][k]);
            uint32_t* kb = reinterpret_cast<uint32_t*>(c->ckey[0][k]);
            k_rekey32<<<grid_for(c->ncrit[k]), kBlock, 0, c->st>>>(c->ckey[0][k], c->ncrit[k], c->rank, ka);
            c->cur[k] = radix_sort<uint32_t, uint32_t, DMS_ORDER_ITEMS>(ka, c->cidx[0][k], kb, c->cidx[1][k], c->ncrit[k], 0,
                                                                        bits_for(c->N), c->ss, c->st, &c->launches);
            k_gather_ids<<<grid_for(c->ncrit[k]), kBlock, 0, c->st>>>(c->cid[0][k], crit_perm(c, k), c->ncrit[k],
                                                                     c->cid[1][k]);
            c->launches += 2;
            continue;
        }
        static const int ms_env = getenv("DMS_CRIT_RUNS") ? atoi(getenv("DMS_CRIT_RUNS")) : 1;
        if (ms_env && bm_env && c->ncrit[k] > 0) {
            // several cells per star: star runs by the rank bitmap, each run sorted by G
            const int64_t nw = (c->N + 31) / 32, m = c->ncrit[k];
            if (!c->bm) {
                CU(dalloc(&c->bm, nw));
                CU(dalloc(&c->bmcnt, nw));
                CU(dalloc(&c->bmpre, nw));
            }
            if (m + 1 > c->ms_cap) {
                for (uint32_t** q : {&c->ms_sidx, &c->ms_slot, &c->ms_cnt, &c->ms_base}) { cudaFree(*q); *q = nullptr; }
                cudaFree(c->ms_stage);
                const int64_t cap = 2 * m + 1024;
                for (uint32_t** q : {&c->ms_sidx, &c->ms_slot, &c->ms_cnt, &c->ms_base}) CU(dalloc(q, cap));
                CU(dalloc(&c->ms_stage, cap));
                c->ms_cap = cap;
            }
            uint32_t* r = reinterpret_cast<uint32_t*>(c->ckey[1][k]);
            CU(cudaMemsetAsync(c->bm, 0, nw * sizeof(unsigned), c->st));
            CU(cudaMemsetAsync(c->ms_cnt, 0, m * sizeof(uint32_t), c->st));
            k_bm_set<<<grid_for(m), kBlock, 0, c->st>>>(c->ckey[0][k], m, c->rank, r, c->bm);
            k_bm_popc<<<grid_for(nw), kBlock, 0, c->st>>>(c->bm, nw, c->bmcnt);
            scan_excl(c->bmcnt, c->bmpre, nw, c->ss, c->st, &c->launches);
            k_ms_count<<<grid_for(m), kBlock, 0, c->st>>>(r, m, c->bm, c->bmpre, c->ms_sidx, c->ms_cnt, c->ms_slot);
            // stars present <= m; unused counts are 0, so scanning all m is exact
            scan_excl(c->ms_cnt, c->ms_base, m, c->ss, c->st, &c->launches);
            k_ms_place<<<grid_for(m), kBlock, 0, c->st>>>(c->ckey[0][k], m, c->ms_sidx, c->ms_slot, c->ms_base, c->ms_stage);
            k_ms_fix<<<grid_for(m), kBlock, 0, c->st>>>(c->ms_stage, m, c->ms_base, c->ms_cnt, c->cidx[1][k]);
            c->cur[k] = 1;
            k_gather_ids<<<grid_for(m), kBlock, 0, c->st>>>(c->cid[0][k], crit_perm(c, k), m, c->cid[1][k]);
            c->launches += 6;
            continue;
        }
        k_rekey<<<grid_for(c->ncrit[k]), kBlock, 0, c->st>>>(c->ckey[0][k], c->ncrit[k], c->rank);
        c->launches++;
        // the low 12 bits (G) only order cells of one star: C_0 holds at most one cell per
        // star (x itself), and in 1D so does C_1 (the second lower edge), so their keys
        // sort on the rank bits alone; edge keys have G's low 8 bits zero, triangle keys
        // its low 4 (key_edge / key_tri) -- fewer 8-bit passes
        // (the five-tetrahedra keys use every G bit: tet5.cuh t5_key)
        const int bit0 = (k == 0 || c->ndim == 1) ? 12 : c->cplx ? 0 : (k == 1 ? 8 : (k == 2 ? 4 : 0));
        c->cur[k] = radix_sort<uint64_t, uint32_t, 8>(c->ckey[0][k], c->cidx[0][k], c->ckey[1][k], c->cidx[1][k],
                                                     c->ncrit[k], bit0, kbits, c->ss, c->st, &c->launches);
        // lexicographically sorted ids = emitted ids gathered through the permutation
        k_gather_ids<<<grid_for(c->ncrit[k]), kBlock, 0, c->st>>>(c->cid[0][k], crit_perm(c, k), c->ncrit[k],
                                                                 c->cid[1][k]);
        c->launches++;
    }
    CU(cudaGetLastError());
    c->have_crit = true;
    // 1D: spatial order of C_0 / C_1 from the gradient's per-CTA tables (path1d.cuh)
    c->have_pmap = false;
    // DMS_PATH1D=1: the closed form (correct, measured slower on c5b: 4.1 vs 3.1 ms per
    // union-find alone -- DESIGN.md 8b), so the contraction rounds stay the default
    static const int path_env = getenv("DMS_PATH1D") ? atoi(getenv("DMS_PATH1D")) : 0;
    if (c->ndim == 1 && c->t1_valid && path_env) {
        const int64_t need = std::max(c->ncrit[0], c->ncrit[1]) + 1;
        if (need > c->cap_pmap) {
            for (int k = 0; k < 2; k++) {
                cudaFree(c->pmap[k]);
                c->pmap[k] = nullptr;
                CU(dalloc(&c->pmap[k], 2 * need + 1024));
            }
            c->cap_pmap = 2 * need + 1024;
        }
        for (int k = 0; k < 2; k++) {
            scan_excl(c->t1cnt[k], c->t1scan[k], c->t1tiles, c->ss, c->st, &c->launches);
            k_path_spatial<<<(unsigned)ceil_div(c->t1tiles * 32, kBlock), kBlock, 0, c->st>>>(c->t1base[k], c->t1cnt[k],
                                                                                          c->t1scan[k], c->t1tiles,
                                                                                          c->pmap[k]);
            c->launches++;
        }
        CU(cudaGetLastError());
        c->have_pmap = true;
    }
    return DMS_OK;
}

// 1D: the elder-rule union-find of diagram `which` in closed form on its path graph
// (path1d.cuh) instead of the contraction rounds; checked against the traced arcs (a
// mismatch falls back to the rounds in path_finish)
dms_status path_issue(dms_ctx* c, UFBuf& u, int which) {
    PathBuf& b = c->pb[which];
    const int64_t m = c->ncrit[which == 0 ? 1 : 0];
    const int64_t P = which == 0 ? c->ncrit[0] : c->ncrit[1] + 2;
    const int64_t nb = ceil_div(P, (int64_t)kPB);
    int levels = 1;
    while ((int64_t(1) << (levels - 1)) < nb) levels++;
    if (P > b.cap) {
        cudaFree(b.sage); cudaFree(b.lw); cudaFree(b.rw); cudaFree(b.dw); cudaFree(b.unres); cudaFree(b.pre); cudaFree(b.suf);
        cudaFree(b.sarc);
        const int64_t cap = 2 * P + 1024;
        CU(dalloc(&b.sarc, cap));
        CU(dalloc(&b.sage, cap)); CU(dalloc(&b.lw, cap)); CU(dalloc(&b.rw, cap)); CU(dalloc(&b.dw, cap));
        CU(dalloc(&b.unres, cap)); CU(dalloc(&b.pre, cap)); CU(dalloc(&b.suf, cap));
        b.cap = cap;
    }
    if ((int64_t)levels * nb > b.capb) {
        cudaFree(b.npre); cudaFree(b.nsuf); cudaFree(b.bnd); cudaFree(b.tmin); cudaFree(b.tspan);
        const int64_t cap = 2 * (int64_t)levels * nb + 1024;
        CU(dalloc(&b.npre, cap)); CU(dalloc(&b.nsuf, cap)); CU(dalloc(&b.bnd, cap)); CU(dalloc(&b.tmin, cap));
        CU(dalloc(&b.tspan, cap));
        b.capb = cap;
    }
    if (!b.bad) {
        CU(dalloc(&b.bad, 1));
        if (cudaMallocHost(&b.h_bad, sizeof(int)) != cudaSuccess) return fail(c, DMS_ERR_OOM, "pinned");
    }
    PathArgs A;
    A.P = P;
    A.nb = nb;
    A.node_map = c->pmap[which == 0 ? 0 : 1];
    A.arc_map = c->pmap[which == 0 ? 1 : 0];
    A.node_off = which == 0 ? 0 : 1;
    A.virt = which == 0 ? -1 : (int32_t)c->ncrit[1];
    A.key = u.key;
    A.age = u.age;
    A.arc_a = u.arc_a;
    A.arc_b = u.arc_b;
    A.bad = b.bad;
    A.sage = b.sage;
    A.sarc = b.sarc;
    A.lw = b.lw;
    A.rw = b.rw;
    A.dw = b.dw;
    A.unres = b.unres;
    A.pre = b.pre;
    A.suf = b.suf;
    A.npre = b.npre;
    A.nsuf = b.nsuf;
    A.bnd = b.bnd;
    A.tmin = b.tmin;
    A.tspan = b.tspan;
    A.levels = levels;
    A.out = u.out;
    CU(cudaMemsetAsync(b.bad, 0, sizeof(int), c->st));
    k_path_check<<<grid_for(P), kBlock, 0, c->st>>>(A);
    k_path_local<<<grid_for(nb, kPT), kPT, 0, c->st>>>(A);
    for (int k = 1; k < levels; k++) k_path_sparse<<<grid_for(nb), kBlock, 0, c->st>>>(A, k);
    k_fill_i32<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, -1);
    k_path_resolve<<<grid_for(P), kBlock, 0, c->st>>>(A);
    k_path_emit<<<grid_for(P), kBlock, 0, c->st>>>(A);
    c->launches += 5 + (levels - 1);
    CU(cudaMemcpyAsync(b.h_bad, b.bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CU(cudaGetLastError());
    b.used = true;
    return DMS_OK;
}


// union-find over arcs (processing order), see diag.cuh
// u.arc_a / u.arc_b / u.key (per arc) and u.age (per node) are in emission order
// issue: init + the cooperative rounds; the convergence status lands in pinned memory
dms_status uf_issue(dms_ctx* c, UFBuf& u, int64_t m, int64_t nodes, int karcs, int rev) {
    const unsigned gi = grid_for(std::max(m, nodes));
    k_uf_init<<<gi, kBlock, 0, c->st>>>(u.parent, u.best, nodes, u.arc_a, u.arc_b, u.key, m, u.out, u.rec0);
    c->launches++;
    if (m == 0) return DMS_OK;
    int hm[4] = {(int)m, 0, 0, 0};  // nlive[2], status, cur
    CU(cudaMemcpyAsync(u.nlive, hm, sizeof hm, cudaMemcpyHostToDevice, c->st));
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_uf_coop, kBlock, 0);
    const int64_t resident = (int64_t)sms * std::max(per, 1) / (c->half ? 2 : 1);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(m), resident));
    UFArgs U;
    U.parent = u.parent;
    U.best = u.best;
    U.out = u.out;
    U.rec0 = u.rec0;
    U.rec1 = u.rec1;
    U.nlive = u.nlive;
    U.status = u.nlive + 2;
    U.cur_out = u.nlive + 3;
    U.trace = u.trace;
    U.key = u.key;
    U.age = u.age;
    // DMS_UF_MAX_ROUNDS (tests only): cap the parallel rounds to exercise the sequential
    // fallback tail that a pathological input would take
    static const int rounds_env = getenv("DMS_UF_MAX_ROUNDS") ? atoi(getenv("DMS_UF_MAX_ROUNDS")) : 4096;
    U.max_rounds = std::max(1, rounds_env);
    // same-address contention on best[] comes with arc-dense graphs (3D: ~4 arcs per node,
    // the big components collect most arcs): pre-reduce per warp there (measured)
    static const int agg_env = getenv("DMS_AGG") ? atoi(getenv("DMS_AGG")) : -1;
    const bool dense = (double)m > 3.0 * (double)nodes;
    U.agg = agg_env >= 0 ? agg_env : (dense ? 2 : 0);
    // dense graphs (most arcs close cycles): reveal the arcs in key-ordered batches
    static const int batch_env = getenv("DMS_UFBATCH") ? atoi(getenv("DMS_UFBATCH")) : -1;
    const int nb = batch_env >= 0 ? batch_env : (dense ? 16 : 0);  // (sweep: DESIGN.md 8b)
    U.src = u.rsrc;
    U.nsrc = (int)m;
    U.batch = nb > 0 ? (int)std::max<int64_t>(kUFTail, (m + nb - 1) / nb) : 0;
    if (U.batch) {
        k_uf_src<<<grid_for(m), kBlock, 0, c->st>>>(u.arc_a, u.arc_b, crit_perm(c, karcs), m, rev, u.rsrc);
        c->launches++;
        int hz[2] = {0, 0};  // the live list starts empty
        CU(cudaMemcpyAsync(u.nlive, hz, sizeof hz, cudaMemcpyHostToDevice, c->st));
    }
    void* args[] = {&U};
    u.last_m = m;
    u.last_grid = grid;
    u.last_batch = U.batch;
    CU(cudaLaunchCooperativeKernel((void*)k_uf_coop, grid, kBlock, args, 0, c->st));
    c->launches++;
    CU(cudaMemcpyAsync(u.h_status, u.nlive + 2, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    return DMS_OK;
}

// finish: wait for the rounds; a pathological input that did not converge within
// max_rounds gets the sequential tail here
dms_status uf_finish(dms_ctx* c, UFBuf& u, int64_t m) {
    if (m == 0) return DMS_OK;
    CU(cudaStreamSynchronize(c->st));
    if (*u.h_status < 0) return DMS_OK;
    // pathological input (no convergence within max_rounds): sequential tail over the
    // undecided arcs in processing order (gather them, sort by key, then one thread)
    k_flag_undecided<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.flags);
    scan_excl(u.flags, u.pos, m, c->ss, c->st, &c->launches);
    k_gather_undecided<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.pos, u.list);
    uint32_t hp[2];
    CU(cudaMemcpyAsync(&hp[0], u.pos + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(&hp[1], u.flags + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    const int64_t nl = (int64_t)hp[0] + hp[1];
    k_gather_keys<<<grid_for(nl), kBlock, 0, c->st>>>(u.list, nl, u.key, u.inv_a);
    const int where = radix_sort<uint32_t, uint32_t, 12>(u.inv_a, reinterpret_cast<uint32_t*>(u.list), u.flags,
                                                         reinterpret_cast<uint32_t*>(u.live2), nl, 0, 32, c->ss,
                                                         c->st, &c->launches);
    const int32_t* sorted = where ? u.live2 : u.list;
    k_uf_tail<<<1, 32, 0, c->st>>>(u.arc_a, u.arc_b, sorted, nl, u.parent, u.out, u.age);
    c->launches += 4;
    CU(cudaGetLastError());
    return DMS_OK;
}

// stable compaction count: pos = exclusive scan of flags; returns the total
dms_status flag_scan(dms_ctx* c, UFBuf& u, int64_t m, int want_unpaired, int64_t* total) {
    *total = 0;
    if (m == 0) return DMS_OK;
    k_flag_ge0<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.flags, want_unpaired);
    c->launches++;
    scan_excl(u.flags, u.pos, m, c->ss, c->st, &c->launches);
    uint32_t h[2];
    CU(cudaMemcpyAsync(&h[0], u.pos + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(&h[1], u.flags + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    *total = (int64_t)h[0] + h[1];
    return DMS_OK;
}

// async: the count stays on the device (read after the next synchronisation, see
// unpaired_count), so the host does not wait here
dms_status emit_unpaired(dms_ctx* c, int which, UFBuf& u, int64_t m, const int64_t* ids, int rev,
                         bool async = false) {
    c->nunp_async[which] = false;
    if (async && m > 0) {
        k_flag_ge0<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.flags, 1);
        c->launches++;
        scan_excl(u.flags, u.pos, m, c->ss, c->st, &c->launches);
        if (m + 1 > c->cap_unp[which]) {  // grow only: capacity for every arc
            cudaFree(c->unp[which]);
            c->unp[which] = nullptr;
            CU(dalloc(&c->unp[which], 2 * m + 1024));
            c->cap_unp[which] = 2 * m + 1024;
        }
        k_emit_unpaired_dev<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.pos, u.flags, ids, c->unp[which], rev);
        c->launches++;
        CU(cudaMemcpyAsync(&u.h_cnt[0], u.pos + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        CU(cudaMemcpyAsync(&u.h_cnt[1], u.flags + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        c->nunp_async[which] = true;
        return DMS_OK;
    }
    int64_t n = 0;
    dms_status s = flag_scan(c, u, m, 1, &n);
    if (s) return s;
    if (n + 1 > c->cap_unp[which]) {  // grow only: no allocation inside a steady-state step
        cudaFree(c->unp[which]);
        c->unp[which] = nullptr;
        CU(dalloc(&c->unp[which], 2 * n + 1024));
        c->cap_unp[which] = 2 * n + 1024;
    }
    c->nunp[which] = n;
    if (n) {
        k_emit_unpaired<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.pos, n, ids, c->unp[which], rev);
        c->launches++;
    }
    return DMS_OK;
}

// union-find inputs in emission order: arc keys from the arcs' sort permutation, node
// ages from the nodes' sort permutation (rev: descending processing order)
void uf_keys_ages(dms_ctx* c, UFBuf& u, int karcs, int64_t m, int knodes, int64_t n, int rev) {
    if (m) k_uf_keys<<<grid_for(m), kBlock, 0, c->st>>>(crit_perm(c, karcs), m, rev, u.key);
    k_uf_ages<<<grid_for(n + 1), kBlock, 0, c->st>>>(crit_perm(c, knodes), n, rev, u.age);
    c->launches += 2;
}

// out (emission order) -> processing order, in place (buffer swap)
void out_to_processing(dms_ctx* c, UFBuf& u, int karcs, int64_t m, int rev) {
    if (!m) return;
    k_permute1<<<grid_for(m), kBlock, 0, c->st>>>(u.out, crit_perm(c, karcs), m, rev, u.outp);
    c->launches++;
    std::swap(u.out, u.outp);
}

// D0 part 1 (Sec. 5.1(a,b)): the unstable sets, traced from the emitted critical cells
// (no ranks needed, so it can run beside the critical sort)
dms_status d0_trace(dms_ctx* c) {
    c->t_diag[0] = stage_begin(c);
    UFBuf& u = c->uf[0];
    const int64_t m = c->ncrit[1], n0 = c->ncrit[0];
    dms_status s = alloc_uf(c, u, m, n0);
    if (s) return s;
    Geo3 g = geo(c);
    // nodes = minima, numbered in emission (spatial) order
    k_node_map<<<grid_for(n0), kBlock, 0, c->st>>>(crit_ids_emitted(c, 0), n0, c->node_of0);
    c->launches++;
    if (m) {
        StageTimer t6(c, 6);
        if (c->cplx == DMS_COMPLEX_5TET)
            k_d0_arcs_t5<<<grid_for(m), kBlock, 0, c->st>>>(t5geo(c), c->dt5, static_cast<const uint8_t*>(c->grad),
                                                           crit_ids_emitted(c, 1), m, c->node_of0, u.arc_a, u.arc_b);
        else
            k_d0_arcs<<<grid_for(m), kBlock, 0, c->st>>>(g, crit_ids_emitted(c, 1), m, c->node_of0, u.arc_a, u.arc_b);
        c->launches++;
    }
    return DMS_OK;
}

dms_status d0_issue(dms_ctx* c) {
    UFBuf& u = c->uf[0];
    const int64_t m = c->ncrit[1], n0 = c->ncrit[0];
    dms_status s;
    if (c->traced[0]) {  // traced beside the critical sort (run_critical)
        CU(cudaStreamWaitEvent(c->st, c->ev_trace[0], 0));
        c->traced[0] = false;
    } else if ((s = d0_trace(c))) {
        return s;
    }
    {
        StageTimer t8(c, 8);
        uf_keys_ages(c, u, 1, m, 0, n0, 0);
        c->pb[0].used = false;
        s = (c->have_pmap && m > 0) ? path_issue(c, u, 0) : uf_issue(c, u, m, n0, 1, 0);
        if (s) return s;
    }
    return DMS_OK;
}

// the union-find of diagram `which` done: the rounds' finish, or the path check (a
// mismatch reruns it as rounds)
dms_status uf_or_path_finish(dms_ctx* c, UFBuf& u, int which, int64_t m, int64_t nodes, int karcs, int rev) {
    PathBuf& b = c->pb[which];
    if (!b.used) return uf_finish(c, u, m);
    CU(cudaStreamSynchronize(c->st));
    if (!*b.h_bad) return DMS_OK;
    b.used = false;
    dms_status s = uf_issue(c, u, m, nodes, karcs, rev);
    return s ? s : uf_finish(c, u, m);
}

dms_status d0_finish(dms_ctx* c) {
    UFBuf& u = c->uf[0];
    const int64_t m = c->ncrit[1];
    Geo3 g = geo(c);
    dms_status s = uf_or_path_finish(c, u, 0, m, c->ncrit[0], 1, 0);
    if (s) return s;
    out_to_processing(c, u, 1, m, 0);
    c->npairs_async[0] = 0;
    if (m > 0) {  // no host wait: pair count read on the device, and by the host after the next sync
        k_flag_ge0<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.flags, 0);
        c->launches++;
        scan_excl(u.flags, u.pos, m, c->ss, c->st, &c->launches);
        if (m + 1 > c->cap_pairs[0]) {
            cudaFree(c->pairs[0]);
            c->pairs[0] = nullptr;
            CU(dalloc(&c->pairs[0], 2 * m + 1024));
            c->cap_pairs[0] = 2 * m + 1024;
        }
        k_emit_d0<<<grid_for(m), kBlock, 0, c->st>>>(g, u.out, m, u.pos, crit_ids_emitted(c, 0), crit_ids(c, 1),
                                                    c->pairs[0]);
        // Sec. 6: the global minimum (the oldest node, first of C_0) never dies
        k_emit_inf_dev<<<1, 32, 0, c->st>>>(g, 0, crit_ids(c, 0), c->kmax, c->pairs[0], u.pos, u.flags, m);
        c->launches += 2;
        CU(cudaMemcpyAsync(&u.h_cnt[2], u.pos + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        CU(cudaMemcpyAsync(&u.h_cnt[3], u.flags + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        c->npairs_async[0] = 2;  // np + the infinite class
        s = emit_unpaired(c, 0, u, m, crit_ids(c, 1), 0, true);
        if (s) return s;
        CU(cudaGetLastError());
        stage_end(c, 3, c->t_diag[0]);
        c->t_diag[0] = nullptr;
        c->have_d[0] = true;
        return DMS_OK;
    }
    int64_t np = 0;
    s = flag_scan(c, u, m, 0, &np);
    if (s) return s;
    if (np + 1 > c->cap_pairs[0]) {
        cudaFree(c->pairs[0]);
        c->pairs[0] = nullptr;
        CU(dalloc(&c->pairs[0], 2 * np + 1024));
        c->cap_pairs[0] = 2 * np + 1024;
    }
    if (np) {
        k_emit_d0<<<grid_for(m), kBlock, 0, c->st>>>(g, u.out, m, u.pos, crit_ids_emitted(c, 0), crit_ids(c, 1),
                                                    c->pairs[0]);
        c->launches++;
    }
    // Sec. 6: the global minimum (the oldest node, first of C_0) never dies
    k_emit_inf_k<<<1, 32, 0, c->st>>>(g, 0, crit_ids(c, 0), c->kmax, c->pairs[0] + np);
    c->launches++;
    c->npairs[0] = np + 1;
    s = emit_unpaired(c, 0, u, m, crit_ids(c, 1), 0, true);
    if (s) return s;
    CU(cudaGetLastError());
    stage_end(c, 3, c->t_diag[0]);
    c->t_diag[0] = nullptr;
    c->have_d[0] = true;
    return DMS_OK;
}

// D_{d-1} part 1 (Sec. 5.2): the stable sets on the dual gradient (no ranks needed)
dms_status dtop_trace(dms_ctx* c) {
    c->t_diag[1] = stage_begin(c);
    const int d = c->ndim;
    UFBuf& u = c->uf[1];
    const int64_t m = c->ncrit[d - 1], nd = c->ncrit[d];
    dms_status s = alloc_uf(c, u, m, nd + 1);
    if (s) return s;
    Geo3 g = geo(c);
    // nodes = critical d-simplices in emission order, plus the virtual maximum nd
    k_node_map<<<grid_for(nd), kBlock, 0, c->st>>>(crit_ids_emitted(c, d), nd, c->node_oftop);
    c->launches++;
    if (m && c->cplx == DMS_COMPLEX_5TET) {
        StageTimer t7(c, 7);
        k_dtop_arcs_t5<<<grid_for(2 * m), kBlock, 0, c->st>>>(t5geo(c), c->dt5, static_cast<const uint8_t*>(c->grad),
                                                             crit_ids_emitted(c, d - 1), m, c->node_oftop, (int32_t)nd,
                                                             u.arc_a, u.arc_b);
        c->launches++;
    } else if (m) {
        StageTimer t7(c, 7);
        if (d >= 2) {
            // persistent work-queue chases, 2 jobs per arc (ascending paths of very uneven
            // length), memoised where the job ids fit the 24-bit stamps
            static const int memo_env = getenv("DMS_MEMO") ? atoi(getenv("DMS_MEMO")) : 1;
            const bool memo = memo_env && 2 * m + 1 < (1 << 24);
            int dev = 0, sms = 148, per = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (d == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dtop_arcs_q<3, true>, kBlock, 0);
            else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dtop_arcs_q<2, true>, kBlock, 0);
            const unsigned grid = (unsigned)std::max<int64_t>(
                1, std::min<int64_t>(grid_for(2 * m), (int64_t)sms * std::max(per, 1)));
            CU(cudaMemsetAsync(c->tile_ctr, 0, sizeof(int), c->st));
            const int64_t* ids = crit_ids_emitted(c, d - 1);
            if (memo) {
                const int64_t ncells = c->N * (d == 3 ? 6 : 2);
                if (!c->chase_mark) {
                    CU(dalloc(&c->chase_mark, ncells));
                    CU(cudaMemsetAsync(c->chase_mark, 0, ncells * sizeof(uint32_t), c->st));
                    c->chase_gen = 0;
                }
                if (++c->chase_gen == 256) {  // stamps wrap: clear them
                    CU(cudaMemsetAsync(c->chase_mark, 0, ncells * sizeof(uint32_t), c->st));
                    c->chase_gen = 1;
                }
                int32_t* res = reinterpret_cast<int32_t*>(u.rec0);  // 2m int32 (rec0: 4m, free until the union-find)
                if (d == 3)
                    k_dtop_arcs_q<3, true><<<grid, kBlock, 0, c->st>>>(g, ids, (int)(2 * m), c->node_oftop, (int32_t)nd,
                                                                      u.arc_a, u.arc_b, c->tile_ctr, c->chase_mark,
                                                                      c->chase_gen, res);
                else
                    k_dtop_arcs_q<2, true><<<grid, kBlock, 0, c->st>>>(g, ids, (int)(2 * m), c->node_oftop, (int32_t)nd,
                                                                      u.arc_a, u.arc_b, c->tile_ctr, c->chase_mark,
                                                                      c->chase_gen, res);
                k_resolve_joins<<<grid_for(2 * m), kBlock, 0, c->st>>>(res, (int)(2 * m), u.arc_a, u.arc_b);
                c->launches++;
            } else if (d == 3) {
                k_dtop_arcs_q<3, false><<<grid, kBlock, 0, c->st>>>(g, ids, (int)(2 * m), c->node_oftop, (int32_t)nd,
                                                                    u.arc_a, u.arc_b, c->tile_ctr, nullptr, 0, nullptr);
            } else {
                k_dtop_arcs_q<2, false><<<grid, kBlock, 0, c->st>>>(g, ids, (int)(2 * m), c->node_oftop, (int32_t)nd,
                                                                    u.arc_a, u.arc_b, c->tile_ctr, nullptr, 0, nullptr);
            }
        } else {
            k_dtop_arcs<<<grid_for(m), kBlock, 0, c->st>>>(g, crit_ids_emitted(c, d - 1), m, c->node_oftop, (int32_t)nd,
                                                          u.arc_a, u.arc_b);
        }
        c->launches++;
    }
    return DMS_OK;
}

dms_status dtop_issue(dms_ctx* c) {
    const int d = c->ndim;
    UFBuf& u = c->uf[1];
    const int64_t m = c->ncrit[d - 1], nd = c->ncrit[d];
    dms_status s;
    if (c->traced[1]) {  // traced beside the critical sort (run_critical)
        CU(cudaStreamWaitEvent(c->st, c->ev_trace[1], 0));
        c->traced[1] = false;
    } else if ((s = dtop_trace(c))) {
        return s;
    }
    {
        StageTimer t9(c, 9);
        uf_keys_ages(c, u, d - 1, m, d, nd, 1);
        c->pb[1].used = false;
        s = (c->have_pmap && m > 0) ? path_issue(c, u, 1) : uf_issue(c, u, m, nd + 1, d - 1, 1);
        if (s) return s;
    }
    return DMS_OK;
}

dms_status dtop_finish(dms_ctx* c) {
    const int d = c->ndim;
    UFBuf& u = c->uf[1];
    const int64_t m = c->ncrit[d - 1];
    Geo3 g = geo(c);
    dms_status s = uf_or_path_finish(c, u, 1, m, c->ncrit[d] + 1, d - 1, 1);
    if (s) return s;
    out_to_processing(c, u, d - 1, m, 1);
    c->npairs_async[1] = 0;
    if (d >= 2 && m > 0) {  // no host wait (no infinite records for d >= 2, Sec. 6)
        k_flag_ge0<<<grid_for(m), kBlock, 0, c->st>>>(u.out, m, u.flags, 0);
        c->launches++;
        scan_excl(u.flags, u.pos, m, c->ss, c->st, &c->launches);
        if (m + 1 > c->cap_pairs[1]) {
            cudaFree(c->pairs[1]);
            c->pairs[1] = nullptr;
            CU(dalloc(&c->pairs[1], 2 * m + 1024));
            c->cap_pairs[1] = 2 * m + 1024;
        }
        k_emit_dtop<<<grid_for(m), kBlock, 0, c->st>>>(g, u.out, m, u.pos, crit_ids(c, d - 1),
                                                      crit_ids_emitted(c, d), c->pairs[1]);
        c->launches++;
        CU(cudaMemcpyAsync(&u.h_cnt[2], u.pos + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        CU(cudaMemcpyAsync(&u.h_cnt[3], u.flags + (m - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st));
        c->npairs_async[1] = 1;  // np, no infinite records
        s = emit_unpaired(c, 1, u, m, crit_ids(c, d - 1), 1, true);
        if (s) return s;
        CU(cudaGetLastError());
        stage_end(c, 4, c->t_diag[1]);
        c->t_diag[1] = nullptr;
        c->have_d[1] = true;
        return DMS_OK;
    }
    int64_t np = 0;
    s = flag_scan(c, u, m, 0, &np);
    if (s) return s;
    // pairs first (their positions are in the scan buffers), then the unpaired list
    // (which rescans); in 1D the unpaired minima (<= m - np) follow the pairs as infinite
    // classes
    const int64_t need = (d == 1 ? m : np) + 1;
    if (need > c->cap_pairs[1]) {
        cudaFree(c->pairs[1]);
        c->pairs[1] = nullptr;
        CU(dalloc(&c->pairs[1], 2 * need + 1024));
        c->cap_pairs[1] = 2 * need + 1024;
    }
    if (np) {
        k_emit_dtop<<<grid_for(m), kBlock, 0, c->st>>>(g, u.out, m, u.pos, crit_ids(c, d - 1),
                                                      crit_ids_emitted(c, d), c->pairs[1]);
        c->launches++;
    }
    s = emit_unpaired(c, 1, u, m, crit_ids(c, d - 1), 1, d >= 2);  // 1D needs the count here
    if (s) return s;
    const int64_t ninf = d == 1 ? c->nunp[1] : 0;  // Sec. 6: in 1D the unpaired minimum is infinite
    for (int64_t i = 0; i < ninf; i++) {
        k_emit_inf_k<<<1, 32, 0, c->st>>>(g, 0, c->unp[1] + i, c->kmax, c->pairs[1] + np + i);
        c->launches++;
    }
    c->npairs[1] = np + ninf;
    CU(cudaGetLastError());
    stage_end(c, 4, c->t_diag[1]);
    c->t_diag[1] = nullptr;
    c->have_d[1] = true;
    return DMS_OK;
}

// D_{d-1} in the "ignore" boundary mode (PAPER.md 2822-2825, App. A 2927-2949; reading
// Z7): the exact mode's arcs with the half-arcs to the virtual maximum dropped, the same
// union-find in decreasing order; the global maximum stays unpaired (its class is D0's
// infinite one, Sec. 6); no infinite records.  The exact results are left untouched.
dms_status run_dtop_ignore(dms_ctx* c) {
    const int d = c->ndim;
    UFBuf& e = c->uf[1];
    UFBuf& u = c->uf_ign;
    const int64_t m = c->ncrit[d - 1], nd = c->ncrit[d];
    dms_status s = alloc_uf(c, u, m, nd + 1);
    if (s) return s;
    Geo3 g = geo(c);
    k_arcs_drop_virtual<<<grid_for(std::max(m, nd + 1)), kBlock, 0, c->st>>>(e.arc_a, e.arc_b, e.key, m, (int32_t)nd,
                                                                          e.age, nd + 1, u.arc_a, u.arc_b, u.key,
                                                                          u.age);
    c->launches++;
    if ((s = uf_issue(c, u, m, nd + 1, d - 1, 1))) return s;
    if ((s = uf_finish(c, u, m))) return s;
    out_to_processing(c, u, d - 1, m, 1);
    int64_t np = 0;
    if ((s = flag_scan(c, u, m, 0, &np))) return s;
    if (np + 1 > c->cap_ign) {
        cudaFree(c->pairs_ign);
        c->pairs_ign = nullptr;
        CU(dalloc(&c->pairs_ign, 2 * np + 1024));
        c->cap_ign = 2 * np + 1024;
    }
    if (np) {
        k_emit_dtop<<<grid_for(m), kBlock, 0, c->st>>>(g, u.out, m, u.pos, crit_ids(c, d - 1), crit_ids_emitted(c, d),
                                                      c->pairs_ign);
        c->launches++;
    }
    CU(cudaGetLastError());
    c->npairs_ign = np;
    c->have_ign = true;
    return DMS_OK;
}

dms_status run_d0(dms_ctx* c) {
    if (!c->have_crit) {
        dms_status s = run_critical(c);
        if (s) return s;
    }
    dms_status s = d0_issue(c);
    return s ? s : d0_finish(c);
}

dms_status run_dtop(dms_ctx* c) {
    if (!c->have_crit) {
        dms_status s = run_critical(c);
        if (s) return s;
    }
    dms_status s = dtop_issue(c);
    return s ? s : dtop_finish(c);
}

// DMS_DTOP1D=0: the dual union-find in 1D too (A/B; the ignore mode always runs it)
bool dtop1d_short(const dms_ctx* c) {
    static const int env = getenv("DMS_DTOP1D") ? atoi(getenv("DMS_DTOP1D")) : 1;
    return c->ndim == 1 && env != 0;
}

// 1D, exact mode: D_{d-1} = D0's records in decreasing birth order (k_dtop_from_d0)
dms_status run_dtop_from_d0(dms_ctx* c) {
    dms_status s;
    if (!c->have_d[0] && (s = run_d0(c))) return s;
    cudaEvent_t t0 = stage_begin(c);
    const int64_t n0 = c->ncrit[0];  // |C_0| - 1 finite pairs + the infinite class (a line is connected)
    if (n0 + 1 > c->cap_pairs[1]) {
        cudaFree(c->pairs[1]);
        c->pairs[1] = nullptr;
        CU(dalloc(&c->pairs[1], 2 * n0 + 1024));
        c->cap_pairs[1] = 2 * n0 + 1024;
    }
    if (c->cap_unp[1] < 1) {
        cudaFree(c->unp[1]);
        c->unp[1] = nullptr;
        CU(dalloc(&c->unp[1], 1024));
        c->cap_unp[1] = 1024;
    }
    k_dtop_from_d0<<<grid_for(n0), kBlock, 0, c->st>>>(c->pairs[0], n0, c->node_of0, c->uf[0].age, c->pairs[1],
                                                      crit_ids(c, 0), c->unp[1]);
    c->launches++;
    CU(cudaGetLastError());
    c->npairs[1] = n0;
    c->npairs_async[1] = 0;
    c->nunp[1] = 1;
    c->nunp_async[1] = false;
    stage_end(c, 4, t0);
    c->have_d[1] = true;
    c->dtop_short = true;
    return DMS_OK;
}

// D0 on the second lane beside D_{d-1} (both only read the gradient and the critical
// lists): issue both, then finish both, so the host's count reads for one overlap the
// other's kernels; the cooperative union-find grids take half the GPU each (two
// cooperative grids must be co-resident together); the persistent chase grid stays
// full (it never waits on other work, and halving it measured slower).
dms_status run_diagrams(dms_ctx* c) {
    static const int conc_env = getenv("DMS_CONCURRENT") ? atoi(getenv("DMS_CONCURRENT")) : 1;
    if (dtop1d_short(c)) {  // 1D: one union-find on the whole GPU, D_{d-1} listed from D0
        dms_status s = run_d0(c);
        return s ? s : run_dtop_from_d0(c);
    }
    if (!conc_env || !c->lane3.st) {
        dms_status s = run_d0(c);
        return s ? s : run_dtop(c);
    }
    CU(cudaEventRecord(c->ev_crit, c->st));
    CU(cudaStreamWaitEvent(c->lane3.st, c->ev_crit, 0));
    c->half = true;
    dms_status s;
    {
        LaneSwap ls(c, c->lane3);
        s = d0_issue(c);
    }
    if (!s) s = dtop_issue(c);
    if (!s) {
        LaneSwap ls(c, c->lane3);
        s = d0_finish(c);
    }
    if (!s) s = dtop_finish(c);
    c->half = false;
    if (s) return s;
    CU(cudaEventRecord(c->ev_d0, c->lane3.st));  // the caller's stream sees D0's results
    CU(cudaStreamWaitEvent(c->st, c->ev_d0, 0));
    return DMS_OK;
}


// ------------------------------------------------------------------ D1 (d1.cuh)

}  // namespace
static int64_t unpaired_count(dms_ctx* c, int which);
namespace {

dms_status d1_grow_arena(dms_ctx* c, unsigned long long need) {
    D1Buf& b = c->d1;
    if (need <= b.arena_cap) return DMS_OK;
    unsigned long long cap = std::max<unsigned long long>(need, 2 * b.arena_cap);
    unsigned long long* a = nullptr;
    CU(dalloc(&a, (int64_t)cap));
    if (b.arena) {
        CU(cudaMemcpyAsync(a, b.arena, b.arena_cap * 8, cudaMemcpyDeviceToDevice, c->st));
        CU(cudaStreamSynchronize(c->st));
        cudaFree(b.arena);
    }
    b.arena = a;
    b.arena_cap = cap;
    return DMS_OK;
}

dms_status d1_alloc(dms_ctx* c, int64_t n0, int64_t nsig) {
    D1Buf& b = c->d1;
    if (!b.tab) {
        D1Tab h;
        build_d1_tab(c->htab, &h);
        CU(dalloc(&b.tab, 1));
        CU(cudaMemcpy(b.tab, &h, sizeof(D1Tab), cudaMemcpyHostToDevice));
    }
    if (!b.ctr) {
        CU(dalloc(&b.ctr, 24));
        if (cudaMallocHost(&b.h_ctr, 24 * sizeof(int32_t)) != cudaSuccess) return fail(c, DMS_ERR_OOM, "pinned");
    }
    if (c->N > b.capN) {
        cudaFree(b.order);
        CU(dalloc(&b.order, c->N));
        b.capN = c->N;
    }
    if (n0 + 1 > b.cap0) {
        const int64_t cap = 2 * (n0 + 1) + 1024;
        for (int32_t** q : {&b.owner}) { cudaFree(*q); CU(dalloc(q, cap)); }
        for (uint32_t** q : {&b.flags, &b.pos}) { cudaFree(*q); CU(dalloc(q, cap)); }
        cudaFree(b.claim);
        CU(dalloc(&b.claim, cap));
        cudaFree(b.un1);
        CU(dalloc(&b.un1, cap));
        int64_t h = 1024;
        while (h < 2 * cap) h *= 2;
        cudaFree(b.hkey);
        cudaFree(b.hval);
        CU(dalloc(&b.hkey, h));
        CU(dalloc(&b.hval, h));
        b.hcap = h;
        b.cap0 = cap;
    }
    if (nsig + 1 > b.capsig) {
        const int64_t cap = 2 * (nsig + 1) + 1024;
        for (int32_t** q : {&b.stop, &b.done, &b.col_len, &b.big, &b.act[0], &b.act[1]}) { cudaFree(*q); CU(dalloc(q, cap)); }
        cudaFree(b.col_off);
        CU(dalloc(&b.col_off, cap));
        cudaFree(b.status);
        CU(dalloc(&b.status, cap));
        cudaFree(b.pairs);
        CU(dalloc(&b.pairs, cap));
        cudaFree(b.gen_off);
        CU(dalloc(&b.gen_off, cap + 1));
        cudaFree(b.taint);
        CU(dalloc(&b.taint, cap));
        cudaFree(b.first_bad);
        CU(dalloc(&b.first_bad, cap));
        cudaFree(b.best);
        CU(dalloc(&b.best, cap));
        cudaFree(b.nadd);
        CU(dalloc(&b.nadd, cap));
        cudaFree(b.snaps);
        b.capsnaps = std::max<int64_t>(1 << 20, 4 * cap);
        CU(dalloc(&b.snaps, b.capsnaps));
        cudaFree(b.deps);
        b.capdeps = std::max<int64_t>(1 << 20, 4 * cap);
        CU(dalloc(&b.deps, b.capdeps));
        b.capsig = cap;
    }
    static const long long arena_env = getenv("DMS_D1_ARENA") ? atoll(getenv("DMS_D1_ARENA")) : 0;
    const unsigned long long want = arena_env > 0 ? (unsigned long long)arena_env
                                                  : std::max<unsigned long long>(1ull << 20, 48ull * (unsigned long long)nsig);
    return d1_grow_arena(c, std::max<unsigned long long>(want, 3ull * nsig + 64));
}

// copying collection of the arena: only the current column of every sigma is live
// (owners' columns included); the new arena doubles when the live part exceeds a quarter
dms_status d1_compact(dms_ctx* c, bool grow) {
    D1Buf& b = c->d1;
    const int64_t n = b.nsig;
    if (n == 0) return DMS_OK;
    k_d1_abs_len<<<grid_for(n), kBlock, 0, c->st>>>(b.col_len, n, b.flags);
    scan_excl(b.flags, b.pos, n, c->ss, c->st, &c->launches);
    uint32_t h[2];
    CU(cudaMemcpyAsync(&h[0], b.pos + (n - 1), 4, cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(&h[1], b.flags + (n - 1), 4, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    const unsigned long long live = (unsigned long long)h[0] + h[1];
    unsigned long long cap = grow ? 2 * b.arena_cap : b.arena_cap;
    while (live > cap / 4) cap *= 2;
    unsigned long long* a = nullptr;
    CU(dalloc(&a, (int64_t)cap));
    k_d1_compact<<<(unsigned)ceil_div(n * 32, kBlock), kBlock, 0, c->st>>>(b.col_off, b.col_len, b.pos, n, b.arena, a);
    c->launches += 2;
    CU(cudaMemcpyAsync(b.ctr + 4, &live, 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
    cudaFree(b.arena);
    b.arena = a;
    b.arena_cap = cap;
    *reinterpret_cast<unsigned long long*>(b.h_ctr + 4) = live;
    return DMS_OK;
}

D1Args d1_args(dms_ctx* c, int phase) {
    D1Buf& b = c->d1;
    D1Args A;
    A.g = geo(c);
    A.tab = b.tab;
    A.rank = c->rank;
    A.order = b.order;
    A.hkey = b.hkey;
    A.hval = b.hval;
    A.hmask = (uint32_t)(b.hcap - 1);
    A.owner = b.owner;
    A.claim = b.claim;
    A.stop = b.stop;
    A.done = b.done;
    A.col_off = b.col_off;
    A.col_len = b.col_len;
    A.status = b.status;
    A.arena = b.arena;
    A.arena_top = reinterpret_cast<unsigned long long*>(b.ctr + 4);
    A.arena_cap = b.arena_cap;
    A.active = nullptr;
    A.nactive = 0;
    A.big = b.big;
    A.nbig = b.ctr + 0;
    A.grab = b.ctr + 1;
    A.err = b.ctr + 3;
    A.dbg = reinterpret_cast<long long*>(b.ctr + 6);
    A.tag = 0;
    A.phase = phase;
    static const int lcap_env = getenv("DMS_D1_LCAP") ? atoi(getenv("DMS_D1_LCAP")) : kD1Cap;
    A.lcap = std::max(4, std::min(kD1Cap, lcap_env));
    static const int adds_env = getenv("DMS_D1_ADDS") ? atoi(getenv("DMS_D1_ADDS")) : 32;
    A.adds = std::max(0, std::min(kBigAddSmall, adds_env));
    A.deps = b.deps;
    A.ndeps = b.ctr + 14;
    A.deps_cap = b.capdeps;
    A.nadd = b.nadd;
    A.snaps = b.snaps;
    A.nsnaps = b.ctr + 16;
    A.snaps_cap = b.capsnaps;
    A.prof = b.stats ? reinterpret_cast<unsigned long long*>(b.stats + 3 * b.capsig) : nullptr;
    A.st_steps = b.stats ? b.stats : nullptr;
    A.st_adds = b.stats ? b.stats + b.capsig : nullptr;
    A.st_pushed = b.stats ? b.stats + 2 * b.capsig : nullptr;
    return A;
}

// rounds of one phase until no sigma is active (d1.cuh); the host reads the active
// count (and the arena / invariant flags) once per round
dms_status d1_rounds(dms_ctx* c, int phase, int64_t nact) {
    D1Buf& b = c->d1;
    int cur = 0;
    int r = 0;
    static const int d1_ctas = getenv("DMS_D1_CTAS") ? atoi(getenv("DMS_D1_CTAS")) : 8;
    static const bool stats = getenv("DMS_D1_STATS") && atoi(getenv("DMS_D1_STATS"));
    static bool attr = false;
    if (!attr) {
        CU(cudaFuncSetAttribute(k_d1_bigc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmem)));
        attr = true;
    }
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    if (stats) {
        for (auto& x : e) cudaEventCreate(&x);
        if (!b.stats) CU(dalloc(&b.stats, 3 * b.capsig + 64));
        CU(cudaMemsetAsync(b.stats, 0, (3 * b.capsig + 64) * sizeof(unsigned), c->st));
    }
    while (nact > 0) {
        if (r > 1000000) return fail(c, DMS_ERR_INVARIANT, "D1: no progress");
        D1Args A = d1_args(c, phase);
        A.active = b.act[cur];
        A.nactive = (int32_t)nact;
        A.tag = (unsigned long long)(0xffffffffu - (uint32_t)r) << 32;
        CU(cudaMemsetAsync(b.ctr, 0, 4 * sizeof(int32_t), c->st));
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nact, 128), (int64_t)c->sms * d1_ctas);
        if (stats) cudaEventRecord(e[0], c->st);
        k_d1_round<<<grid, 128, 0, c->st>>>(A);
        if (stats) cudaEventRecord(e[1], c->st);
        k_d1_bigc<<<c->sms * 3, kBigT, sizeof(BigSmem), c->st>>>(A);
        if (stats) cudaEventRecord(e[2], c->st);
        k_d1_resolve<<<grid_for(nact), kBlock, 0, c->st>>>(A, b.act[cur ^ 1], b.ctr + 2);
        c->launches += 3;
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(b.h_ctr, b.ctr, 16 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
        CU(cudaStreamSynchronize(c->st));
        if (b.h_ctr[3] & 30) {
            const long long* d = reinterpret_cast<const long long*>(b.h_ctr + 6);
            char m[200];
            std::snprintf(m, sizeof m, "D1 phase %d round %d: propagation invariant %d broken (sigma %lld tau %llx edge %lld owner %lld)",
                          phase, r, b.h_ctr[3] & 30, d[0], (unsigned long long)d[1], d[2], d[3]);
            return fail(c, DMS_ERR_INVARIANT, m);
        }
        if (stats) {
            float m0 = 0, m1 = 0;
            cudaEventElapsedTime(&m0, e[0], e[1]);
            cudaEventElapsedTime(&m1, e[1], e[2]);
            std::fprintf(stderr, "[d1] phase %d round %d active %lld big %d round %.3f ms big %.3f ms arena %llu\n", phase, r,
                         (long long)nact, b.h_ctr[0], m0, m1, *reinterpret_cast<unsigned long long*>(b.h_ctr + 4));
        }
        nact = b.h_ctr[2];
        cur ^= 1;
        r++;
        // arena more than half used (or full: the sigmas that did not fit are retried):
        // collect it, doubling when the live columns need it
        // (phase 1 keeps every stored column -- the restart snapshots of the generator
        // pass -- so it grows the arena instead of collecting it)
        if ((b.h_ctr[3] & 1) || *reinterpret_cast<unsigned long long*>(b.h_ctr + 4) > b.arena_cap / 2) {
            dms_status s;
            // growing keeps the snapshots while the doubled arena (plus the copy) fits in
            // a third of the free device memory; beyond that the snapshots are given up
            // (the tainted 2-saddles then restart from their boundaries) and phase 1
            // collects like phase 2
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            if (phase == 1 && b.snaps_ok && 2 * b.arena_cap * 8 > fr / 3) b.snaps_ok = false;
            if (phase == 1 && b.snaps_ok) {
                const unsigned long long used = std::min<unsigned long long>(
                    *reinterpret_cast<unsigned long long*>(b.h_ctr + 4), b.arena_cap);
                s = d1_grow_arena(c, 2 * b.arena_cap);
                if (!s) {
                    CU(cudaMemcpyAsync(b.ctr + 4, &used, 8, cudaMemcpyHostToDevice, c->st));
                    CU(cudaStreamSynchronize(c->st));
                    *reinterpret_cast<unsigned long long*>(b.h_ctr + 4) = used;
                }
            } else {
                s = d1_compact(c, (b.h_ctr[3] & 1) != 0);
            }
            if (s) return s;
        }
    }
    if (stats) {
        for (auto& x : e) cudaEventDestroy(x);
        std::vector<unsigned> h(3 * b.nsig);
        for (int q = 0; q < 3; q++)
            CU(cudaMemcpy(h.data() + q * b.nsig, b.stats + q * b.capsig, b.nsig * sizeof(unsigned), cudaMemcpyDeviceToHost));
        std::vector<int64_t> idx(b.nsig);
        for (int64_t i = 0; i < b.nsig; i++) idx[i] = i;
        auto work = [&](int64_t i) { return (double)h[i] + h[2 * b.nsig + i]; };
        std::sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return work(x) > work(y); });
        double tot_s = 0, tot_p = 0, tot_a = 0;
        for (int64_t i = 0; i < b.nsig; i++) { tot_s += h[i]; tot_a += h[b.nsig + i]; tot_p += h[2 * b.nsig + i]; }
        std::fprintf(stderr, "[d1] phase %d totals: steps %.0f adds %.0f pushed %.0f\n", phase, tot_s, tot_a, tot_p);
        unsigned long long pr[16];
        CU(cudaMemcpy(pr, b.stats + 3 * b.capsig, sizeof pr, cudaMemcpyDeviceToHost));
        const char* nm[8] = {"serial", "refill", "mergeP", "addS", "addB", "stop", "abort", "-"};
        for (int q = 0; q < 7; q++)
            std::fprintf(stderr, "[d1]   bigc %-7s %12.3f Mcycles  n %llu\n", nm[q], pr[q] / 1e6, pr[8 + q]);
        for (int64_t k = 0; k < std::min<int64_t>(12, b.nsig); k++) {
            const int64_t i = idx[k];
            std::fprintf(stderr, "[d1]   sigma %lld steps %u adds %u pushed %u\n", (long long)i, h[i], h[b.nsig + i], h[2 * b.nsig + i]);
        }
    }
    b.rounds[phase - 1] = r;
    return DMS_OK;
}

// D1 pairs (phase 1) and, with want_gen, the generators (phase 2)
dms_status run_d1(dms_ctx* c, bool want_gen) {
    if (c->ndim != 3) return fail(c, DMS_ERR_ARG, "D1 by PairCriticalSimplices is built for 3D fields");
    if (c->cplx != DMS_COMPLEX_FREUDENTHAL)
        return fail(c, DMS_ERR_STATE, "D1 on the GPU is built for the Freudenthal complex (the 5-tet one: oracle only)");
    if (!c->have_d[0] || !c->have_d[1]) {
        dms_status s = run_diagrams(c);
        if (s) return s;
    }
    CU(cudaStreamSynchronize(c->st));
    D1Buf& b = c->d1;
    const int64_t n0 = unpaired_count(c, 0), nsig = unpaired_count(c, 1);
    dms_status s = d1_alloc(c, n0, nsig);
    if (s) return s;
    b.n0 = n0;
    b.nsig = nsig;
    const Geo3 g = geo(c);
    if (!c->have_d1) {
        StageTimer tm(c, 10);
        k_d1_invert<<<grid_for(c->N), kBlock, 0, c->st>>>(c->rank, c->N, b.order);
        CU(cudaMemsetAsync(b.hkey, 0, b.hcap * 8, c->st));
        if (n0) k_d1_hash<<<grid_for(n0), kBlock, 0, c->st>>>(g, c->rank, c->unp[0], n0, b.hkey, b.hval, (uint32_t)(b.hcap - 1));
        CU(cudaMemsetAsync(b.owner, 0xff, n0 * sizeof(int32_t), c->st));
        CU(cudaMemsetAsync(b.claim, 0xff, n0 * sizeof(unsigned long long), c->st));
        unsigned long long top = 3ull * nsig;
        CU(cudaMemcpyAsync(b.ctr + 4, &top, 8, cudaMemcpyHostToDevice, c->st));
        if (nsig) k_d1_init<<<grid_for(nsig), kBlock, 0, c->st>>>(g, c->rank, c->unp[1], nsig, b.arena, b.col_off, b.col_len, b.act[0], b.done, b.nadd);
        c->launches += 3;
        CU(cudaGetLastError());
        *reinterpret_cast<unsigned long long*>(b.h_ctr + 4) = top;
        CU(cudaMemsetAsync(b.ctr + 14, 0, sizeof(int32_t), c->st));
        CU(cudaMemsetAsync(b.ctr + 16, 0, sizeof(int32_t), c->st));
        static const long long snap_budget_env = getenv("DMS_D1_SNAP_BUDGET") ? atoll(getenv("DMS_D1_SNAP_BUDGET")) : -1;
        b.snaps_ok = snap_budget_env != 0;
        if ((s = d1_rounds(c, 1, nsig))) return s;
        if (nsig) {
            k_d1_emit<<<grid_for(nsig), kBlock, 0, c->st>>>(g, b.stop, b.owner, c->unp[0], c->unp[1], nsig, b.pairs, b.ctr + 3);
            c->launches++;
        }
        // 1-saddles no 2-saddle claimed: infinite D1 classes (none on a grid, a ball)
        b.nun1 = 0;
        if (n0) {
            k_d1_unowned<<<grid_for(n0), kBlock, 0, c->st>>>(b.owner, n0, b.flags);
            scan_excl(b.flags, b.pos, n0, c->ss, c->st, &c->launches);
            k_d1_emit_unowned<<<grid_for(n0), kBlock, 0, c->st>>>(b.flags, b.pos, c->unp[0], n0, b.un1);
            c->launches += 2;
            uint32_t h[2];
            CU(cudaMemcpyAsync(&h[0], b.pos + (n0 - 1), 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaMemcpyAsync(&h[1], b.flags + (n0 - 1), 4, cudaMemcpyDeviceToHost, c->st));
            int32_t e = 0;
            CU(cudaMemcpyAsync(&e, b.ctr + 3, 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaStreamSynchronize(c->st));
            if (e & 30) return fail(c, DMS_ERR_INVARIANT, "D1: a 2-saddle does not own its stop");
            b.nun1 = (int64_t)h[0] + h[1];
        }
        c->have_d1 = true;
    }
    if (want_gen && !c->have_gen) {
        StageTimer tm(c, 11);
        // taint: only the sigmas whose phase-1 column may differ from the sequential
        // algorithm's are propagated again (d1.cuh k_d1_taint_*)
        int32_t nd = 0, nsn = 0;
        CU(cudaMemcpyAsync(&nd, b.ctr + 14, 4, cudaMemcpyDeviceToHost, c->st));
        CU(cudaMemcpyAsync(&nsn, b.ctr + 16, 4, cudaMemcpyDeviceToHost, c->st));
        CU(cudaStreamSynchronize(c->st));
        static const int all_env = getenv("DMS_D1_RERUN_ALL") ? atoi(getenv("DMS_D1_RERUN_ALL")) : 0;
        static const int snap_env = getenv("DMS_D1_SNAPSHOTS") ? atoi(getenv("DMS_D1_SNAPSHOTS")) : 1;
        const bool use_snaps = snap_env && !all_env && nd <= b.capdeps && b.snaps_ok;
        if (nsig) {
            if (nd > b.capdeps || all_env) {
                k_fill_u32<<<grid_for(nsig), kBlock, 0, c->st>>>(b.taint, nsig, 1u);
                c->launches++;
            } else {
                CU(cudaMemsetAsync(b.first_bad, 0xff, nsig * sizeof(uint32_t), c->st));
                if (nd) k_d1_taint_direct<<<grid_for(nd), kBlock, 0, c->st>>>(b.deps, nd, b.owner, b.first_bad);
                c->launches++;
                for (int it = 0; nd && it < 100000; it++) {
                    CU(cudaMemsetAsync(b.ctr + 15, 0, sizeof(int32_t), c->st));
                    k_d1_taint_prop<<<grid_for(nd), kBlock, 0, c->st>>>(b.deps, nd, b.first_bad, b.ctr + 15);
                    c->launches++;
                    int32_t ch = 0;
                    CU(cudaMemcpyAsync(&ch, b.ctr + 15, 4, cudaMemcpyDeviceToHost, c->st));
                    CU(cudaStreamSynchronize(c->st));
                    if (!ch) break;
                }
                k_d1_taint_flags<<<grid_for(nsig), kBlock, 0, c->st>>>(b.first_bad, nsig, b.taint);
                c->launches++;
                if (use_snaps) {
                    CU(cudaMemsetAsync(b.best, 0, nsig * sizeof(unsigned long long), c->st));
                    const int64_t ns = std::min<int64_t>(nsn, b.capsnaps);
                    if (ns) k_d1_snap_pick<<<grid_for(ns), kBlock, 0, c->st>>>(b.snaps, ns, b.first_bad, b.best);
                    c->launches++;
                }
            }
            scan_excl(b.taint, b.pos, nsig, c->ss, c->st, &c->launches);
            uint32_t h[2];
            CU(cudaMemcpyAsync(&h[0], b.pos + (nsig - 1), 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaMemcpyAsync(&h[1], b.taint + (nsig - 1), 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaStreamSynchronize(c->st));
            b.ntaint = (int64_t)h[0] + h[1];
            unsigned long long top = *reinterpret_cast<unsigned long long*>(b.h_ctr + 4);
            if (top + 3ull * b.ntaint + 1024 > b.arena_cap) {  // grow (the snapshots must stay put)
                if ((s = d1_grow_arena(c, 2 * (top + 3ull * b.ntaint + 1024)))) return s;
            }
            k_d1_init_tainted<<<grid_for(nsig), kBlock, 0, c->st>>>(g, c->rank, c->unp[1], nsig, b.taint, b.pos, top,
                                                                   b.arena, b.col_off, b.col_len, b.act[0], b.done,
                                                                   use_snaps ? b.best : nullptr, b.snaps);
            c->launches++;
            top += 3ull * b.ntaint;
            CU(cudaMemcpyAsync(b.ctr + 4, &top, 8, cudaMemcpyHostToDevice, c->st));
            *reinterpret_cast<unsigned long long*>(b.h_ctr + 4) = top;
        }
        if ((s = d1_rounds(c, 2, b.ntaint))) return s;
        b.ngen = 0;
        if (nsig) {
            k_d1_gen_len<<<grid_for(nsig), kBlock, 0, c->st>>>(b.col_len, nsig, b.flags);
            scan_excl(b.flags, b.pos, nsig, c->ss, c->st, &c->launches);
            uint32_t h[2];
            CU(cudaMemcpyAsync(&h[0], b.pos + (nsig - 1), 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaMemcpyAsync(&h[1], b.flags + (nsig - 1), 4, cudaMemcpyDeviceToHost, c->st));
            CU(cudaStreamSynchronize(c->st));
            const int64_t ng = (int64_t)h[0] + h[1];
            if (ng + 1 > b.capgen) {
                cudaFree(b.gen);
                CU(dalloc(&b.gen, 2 * ng + 1024));
                b.capgen = 2 * ng + 1024;
            }
            k_d1_gen_emit<<<(unsigned)ceil_div(nsig * 32, kBlock), kBlock, 0, c->st>>>(g, b.order, b.col_off, b.col_len, b.pos, nsig, b.arena, b.gen_off, b.gen);
            c->launches += 2;
            b.ngen = ng;
        } else {
            CU(cudaMemsetAsync(b.gen_off, 0, 8, c->st));
        }
        CU(cudaGetLastError());
        c->have_gen = true;
    }
    return DMS_OK;
}

}  // namespace

// counts left on the device by the asynchronous emissions, read once the caller's stream
// has been synchronised
static int64_t pair_count(dms_ctx* c, int which) {
    if (c->npairs_async[which] > 0) {
        c->npairs[which] = (int64_t)c->uf[which].h_cnt[2] + c->uf[which].h_cnt[3] + c->npairs_async[which] - 1;
        c->npairs_async[which] = 0;
    }
    return c->npairs[which];
}

static int64_t unpaired_count(dms_ctx* c, int which) {
    if (c->nunp_async[which]) {
        c->nunp[which] = (int64_t)c->uf[which].h_cnt[0] + c->uf[which].h_cnt[1];
        c->nunp_async[which] = false;
    }
    return c->nunp[which];
}

// ====================================================================== C ABI

extern "C" {

dms_status dms_create(const int64_t dims[3], int ndim, const float* d_f, void* stream, dms_ctx** out) {
    return dms_create2(dims, ndim, d_f, stream, DMS_COMPLEX_FREUDENTHAL, out);
}

dms_status dms_create2(const int64_t dims[3], int ndim, const float* d_f, void* stream, dms_complex cplx,
                       dms_ctx** out) {
    if (!dims || !d_f || !out) return DMS_ERR_ARG;
    *out = nullptr;
    if (cplx != DMS_COMPLEX_FREUDENTHAL && cplx != DMS_COMPLEX_5TET) return DMS_ERR_ARG;
    if (ndim < 1 || ndim > 3) return DMS_ERR_DEGENERATE;
    if (cplx == DMS_COMPLEX_5TET && ndim != 3) return DMS_ERR_ARG;
    int64_t N = 1;
    for (int i = 0; i < ndim; i++) {
        if (dims[i] < 2) return DMS_ERR_DEGENERATE;
        N *= dims[i];
        if (N >= ((int64_t)1 << 31)) return DMS_ERR_TOO_LARGE;
    }
    dms_ctx* c = new (std::nothrow) dms_ctx();
    if (!c) return DMS_ERR_OOM;
    c->ndim = ndim;
    for (int i = 0; i < 3; i++) c->L[i] = i < ndim ? dims[i] : 1;
    c->N = N;
    c->f = d_f;
    c->st = (cudaStream_t)stream;
    c->cplx = cplx;
    const int64_t per[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 3, 2, 0}, {1, 7, 12, 6}};
    const int64_t per5[4] = {1, 6, 10, 5};  // tet5.cuh
    for (int k = 0; k < 4; k++) c->ncell[k] = cplx == DMS_COMPLEX_5TET ? per5[k] : per[ndim][k];
    if (c->ncell[ndim] * N >= ((int64_t)1 << 31)) { delete c; return DMS_ERR_TOO_LARGE; }
    // the five-tetrahedra ids of triangles reach 10 N (the gradient's byte offsets 16 N)
    if (cplx == DMS_COMPLEX_5TET && 16 * N >= ((int64_t)1 << 35)) { delete c; return DMS_ERR_TOO_LARGE; }
    if (!build_star_tables(ndim, c->L, &c->htab)) { delete c; return DMS_ERR_INVARIANT; }
    auto bail = [&](dms_status s) { dms_destroy(c); return s; };
#define CA(call) do { if ((call) != cudaSuccess) return bail(DMS_ERR_OOM); } while (0)
    CA(dalloc(&c->dtab, 1));
    if (cudaMemcpy(c->dtab, &c->htab, sizeof(StarTab), cudaMemcpyHostToDevice) != cudaSuccess) return bail(DMS_ERR_CUDA);
    if (cplx == DMS_COMPLEX_5TET) {
        T5Tab* ht = new (std::nothrow) T5Tab;
        if (!ht) return bail(DMS_ERR_OOM);
        const bool ok = build_t5_tables(ht);
        cudaError_t e = ok ? cudaMalloc(&c->dt5, sizeof(T5Tab)) : cudaSuccess;
        if (ok && e == cudaSuccess) e = cudaMemcpy(c->dt5, ht, sizeof(T5Tab), cudaMemcpyHostToDevice);
        delete ht;
        if (!ok) return bail(DMS_ERR_INVARIANT);
        if (e != cudaSuccess) return bail(DMS_ERR_CUDA);
    }
    {
        ChaseTab ct;
        build_chase_tables(c->htab, &ct);
        CA(dalloc(&c->dctab, 1));
        if (cudaMemcpy(c->dctab, &ct, sizeof(ChaseTab), cudaMemcpyHostToDevice) != cudaSuccess) return bail(DMS_ERR_CUDA);
    }
    if (ndim == 3 && cplx == DMS_COMPLEX_FREUDENTHAL) {
        GradLut gl;
        build_grad_lut(c->htab, &gl);
        CA(dalloc(&c->dlut3, 1));
        if (cudaMemcpy(c->dlut3, &gl, sizeof(GradLut), cudaMemcpyHostToDevice) != cudaSuccess) return bail(DMS_ERR_CUDA);
    }
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev);
    }
    CA(dalloc(&c->rank_scratch, N));
    if (ndim == 1) {
        c->t1tiles = ceil_div(N, (int64_t)kBlock * kG1);
        for (int k = 0; k < 2; k++) {
            CA(dalloc(&c->t1base[k], c->t1tiles));
            CA(dalloc(&c->t1cnt[k], c->t1tiles));
            CA(dalloc(&c->t1scan[k], c->t1tiles));
        }
    }
    CA(cudaMalloc(&c->grad_scratch, dms_gradient_bytes(c)));
    for (int b = 0; b < 2; b++) { CA(dalloc(&c->okeys[b], N)); CA(dalloc(&c->ovals[b], N)); }
    {
        // the order by sample sort while the mean bucket (N / B, B <= 16384 buckets)
        // stays <= 8192 keys, i.e. N <= 2^27; LSD radix sort otherwise and below 2^16
        static const int samp_env = getenv("DMS_ORDER_SAMPLE") ? atoi(getenv("DMS_ORDER_SAMPLE")) : 0;
        int B = 2;
        while (B < kOrdMaxB && (int64_t)B * kOrdMeanMax < N) B <<= 1;
        if (samp_env && N >= (1 << 16) && (int64_t)B * kOrdMeanMax >= N) {
            c->ord_B = B;
            c->ord_S = B * kOrdOversample;
            CA(dalloc(&c->ord_keys, N));
            CA(dalloc(&c->ord_bid, N));
            for (int b = 0; b < 2; b++) { CA(dalloc(&c->ord_skeys[b], c->ord_S)); CA(dalloc(&c->ord_svals[b], c->ord_S)); }
            CA(dalloc(&c->ord_spl, B));
            CA(dalloc(&c->ord_counts, (int64_t)B * c->sms));
            CA(dalloc(&c->ord_offs, (int64_t)B * c->sms));
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_ord_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kOrdMaxB * 12);
                cudaFuncSetAttribute(k_ord_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kOrdMaxB * 4);
                cudaFuncSetAttribute(k_ord_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, kOrdBucketSmem);
                attr = true;
            }
        }
    }
    const int64_t max_tiles = ceil_div(N, (int64_t)kBlock * 8);
    CA(dalloc(&c->ss.counts, max_tiles * kRadix));
    CA(dalloc(&c->ss.counts_scan, max_tiles * kRadix));
    CA(dalloc(&c->ss.status, ceil_div(std::max<int64_t>(max_tiles * kRadix, N), (int64_t)kBlock * kScanItems) + 1));
    CA(dalloc(&c->ss.tile_ctr, 1));
    c->ss.max_tiles = max_tiles;
    CA(dalloc(&c->tile_ctr, 1));
    CA(dalloc(&c->totals, 4));
    CA(dalloc(&c->err, 1));
    CA(dalloc(&c->kmax, 1));
    CA(dalloc(&c->remaining, 1));
    if (cudaMallocHost(&c->h_pinned, 64) != cudaSuccess) return bail(DMS_ERR_OOM);
    {
        // the order's (short, memory-bound) kernels get the highest priority so that their
        // CTAs are scheduled first as the (long, ALU-bound) gradient CTAs retire
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi) != cudaSuccess) return bail(DMS_ERR_CUDA);
    }
    {
        Lane& L = c->lane3;
        if (cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking) != cudaSuccess) return bail(DMS_ERR_CUDA);
        CA(dalloc(&L.ss.counts, max_tiles * kRadix));
        CA(dalloc(&L.ss.counts_scan, max_tiles * kRadix));
        CA(dalloc(&L.ss.status, ceil_div(std::max<int64_t>(max_tiles * kRadix, N), (int64_t)kBlock * kScanItems) + 1));
        CA(dalloc(&L.ss.tile_ctr, 1));
        L.ss.max_tiles = max_tiles;
        CA(dalloc(&L.tile_ctr, 1));
        if (cudaMallocHost(&L.h_pinned, 64) != cudaSuccess) return bail(DMS_ERR_OOM);
    }
    {
        Lane& L = c->lane4;
        if (cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking) != cudaSuccess) return bail(DMS_ERR_CUDA);
        CA(dalloc(&L.ss.counts, max_tiles * kRadix));
        CA(dalloc(&L.ss.counts_scan, max_tiles * kRadix));
        CA(dalloc(&L.ss.status, ceil_div(std::max<int64_t>(max_tiles * kRadix, N), (int64_t)kBlock * kScanItems) + 1));
        CA(dalloc(&L.ss.tile_ctr, 1));
        L.ss.max_tiles = max_tiles;
        CA(dalloc(&L.tile_ctr, 1));
        if (cudaMallocHost(&L.h_pinned, 64) != cudaSuccess) return bail(DMS_ERR_OOM);
    }
    for (cudaEvent_t* e : {&c->ev_grad, &c->ev_trace[0], &c->ev_trace[1]})
        if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return bail(DMS_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_crit, cudaEventDisableTiming) != cudaSuccess) return bail(DMS_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_d0, cudaEventDisableTiming) != cudaSuccess) return bail(DMS_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess) return bail(DMS_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->ev_order, cudaEventDisableTiming) != cudaSuccess) return bail(DMS_ERR_CUDA);
    CA(dalloc(&c->node_of0, N));
    CA(dalloc(&c->node_oftop, c->ncell[ndim] * N));
    // DMS_CRIT_CAP (tests only): a small initial record capacity exercises the overflow
    // path (grow the buffers, recompute the gradient)
    static const int64_t cap_env = getenv("DMS_CRIT_CAP") ? atoll(getenv("DMS_CRIT_CAP")) : -1;
    for (int k = 0; k <= ndim; k++) c->cap[k] = cap_env >= 0 ? cap_env : N / 2 + 1024;
    if (alloc_crit(c) != DMS_OK) return bail(DMS_ERR_OOM);
    {  // 2D: the dual chases read one packed word per vertex (DMS_CHASEWORD=0: the gradient words)
        // and the D0 descent a compact vertex-code array (DMS_VCODES=0: the gradient words).
        // 3D: the 16-byte gradient word holds both (hi half = chase word, vertex code in lo).
        static const int cw_env = getenv("DMS_CHASEWORD") ? atoi(getenv("DMS_CHASEWORD")) : 1;
        if (ndim == 2 && cw_env) CA(dalloc(&c->cw2, N));
        static const int vc_env = getenv("DMS_VCODES") ? atoi(getenv("DMS_VCODES")) : 1;
        if (ndim == 2 && vc_env) CA(dalloc(&c->vc, N));
    }
    if (ndim == 2) {  // 2D: the ProcessLowerStars table of all 1957 star patterns
        int acc = 0;
        for (int L = 0; L < 64; L++) {
            c->lut2off.off[L] = (uint16_t)acc;
            acc += fact_small(__builtin_popcount(L));
        }
        if (acc != kLut2) return bail(DMS_ERR_INVARIANT);
        CA(dalloc(&c->lut2, kLut2));
        k_build_lut2<<<(unsigned)ceil_div(kLut2, kBlockG), kBlockG, 0, c->st>>>(c->dtab, c->lut2off, c->lut2);
        if (cudaGetLastError() != cudaSuccess) return bail(DMS_ERR_CUDA);
    }
    if (cudaMemsetAsync(c->err, 0, sizeof(int), c->st) != cudaSuccess) return bail(DMS_ERR_CUDA);
#undef CA
    *out = c;
    return DMS_OK;
}

size_t dms_gradient_bytes(const dms_ctx* c) {
    if (!c) return 0;
    const size_t per = c->ndim == 3 ? 16 : (c->ndim == 2 ? 2 : 1);
    return per * (size_t)c->N;
}

dms_status dms_order(dms_ctx* c, int32_t* d_rank) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_rank) return DMS_ERR_ARG;
    if ((s = clear_err(c))) return s;
    return run_order(c, d_rank);
}

dms_status dms_gradient(dms_ctx* c, void* d_grad) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_grad) return DMS_ERR_ARG;
    if (!c->order_fresh && (s = clear_err(c))) return s;  // (after dms_order: one flag for the pass)
    return run_gradient(c, d_grad);
}

dms_status dms_critical(dms_ctx* c, int64_t h_count[4], const int64_t* d_ids_out[4]) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!h_count || !d_ids_out) return DMS_ERR_ARG;
    if (!c->have_crit) {
        s = run_critical(c);
        if (s) return s;
    }
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    for (int k = 0; k < 4; k++) {
        h_count[k] = k <= c->ndim ? c->ncrit[k] : 0;
        d_ids_out[k] = k <= c->ndim ? crit_ids(c, k) : nullptr;
    }
    return DMS_OK;
}

dms_status dms_diagram0(dms_ctx* c, const dms_pair** d_pairs, int64_t* h_n) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_pairs || !h_n) return DMS_ERR_ARG;
    if (!c->have_d[0]) {
        s = run_d0(c);
        if (s) return s;
    }
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    *d_pairs = reinterpret_cast<const dms_pair*>(c->pairs[0]);
    *h_n = pair_count(c, 0);
    return DMS_OK;
}

dms_status dms_diagram_top(dms_ctx* c, dms_boundary mode, const dms_pair** d_pairs, int64_t* h_n) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_pairs || !h_n) return DMS_ERR_ARG;
    if (mode != DMS_BOUNDARY_EXACT && mode != DMS_BOUNDARY_IGNORE) return DMS_ERR_ARG;
    if (!c->have_d[1]) {
        s = (dtop1d_short(c) && mode == DMS_BOUNDARY_EXACT) ? run_dtop_from_d0(c) : run_dtop(c);
        if (s) return s;
    }
    if (mode == DMS_BOUNDARY_IGNORE) {
        if (c->dtop_short) {  // the ignore mode drops arcs of the dual union-find: run it now
            if ((s = run_dtop(c))) return s;
            c->dtop_short = false;
        }
        if (!c->have_ign) {
            if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
            if ((s = run_dtop_ignore(c))) return s;
        }
        if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
        *d_pairs = reinterpret_cast<const dms_pair*>(c->pairs_ign);
        *h_n = c->npairs_ign;
        return DMS_OK;
    }
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    *d_pairs = reinterpret_cast<const dms_pair*>(c->pairs[1]);
    *h_n = pair_count(c, 1);
    return DMS_OK;
}

// the unpaired count, after the caller's stream has been synchronised
dms_status dms_unpaired_saddles(dms_ctx* c, int which, const int64_t** d_ids, int64_t* h_n) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_ids || !h_n || which < 0 || which > 2) return DMS_ERR_ARG;
    if (which == 2) {
        if (!c->have_d1 && (s = run_d1(c, false))) return s;
        if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
        *d_ids = c->d1.un1;
        *h_n = c->d1.nun1;
        return DMS_OK;
    }
    if (!c->have_d[which]) {
        s = which == 0 ? run_d0(c) : (dtop1d_short(c) ? run_dtop_from_d0(c) : run_dtop(c));
        if (s) return s;
    }
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    *d_ids = c->unp[which];
    *h_n = unpaired_count(c, which);
    return DMS_OK;
}

dms_status dms_diagram1(dms_ctx* c, const dms_pair** d_pairs, int64_t* h_n) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_pairs || !h_n) return DMS_ERR_ARG;
    if (!c->have_d1 && (s = run_d1(c, false))) return s;
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    *d_pairs = reinterpret_cast<const dms_pair*>(c->d1.pairs);
    *h_n = c->d1.nsig;
    return DMS_OK;
}

dms_status dms_generators(dms_ctx* c, const int64_t** d_off, const int64_t** d_edges, int64_t* h_n) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!d_off || !d_edges || !h_n) return DMS_ERR_ARG;
    if ((!c->have_d1 || !c->have_gen) && (s = run_d1(c, true))) return s;
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    *d_off = c->d1.gen_off;
    *d_edges = c->d1.gen;
    *h_n = c->d1.nsig;
    return DMS_OK;
}

// DMS_CHECK_INVARIANTS=1 (debug): after a full pass, check the identities every result
// must satisfy: the ranks are a permutation, the Euler
// characteristic of the grid (a ball) is 1, every minimum dies once in D0 (one infinite
// class), every top cell once in D_{d-1} (exact mode), and the saddle counts left for D1
// agree on both sides of the sandwich.  A violation -> DMS_ERR_INVARIANT.
__global__ void k_check_perm(const int32_t* __restrict__ rank, int64_t n, unsigned* bits, unsigned long long* bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t r = rank[i];
    if (r < 0 || r >= n) { atomicAdd(bad, 1ull); return; }
    const unsigned old = atomicOr(bits + (r >> 5), 1u << (r & 31));
    if (old & (1u << (r & 31))) atomicAdd(bad, 1ull);
}
static dms_status check_invariants(dms_ctx* c) {
    static const int env = getenv("DMS_CHECK_INVARIANTS") ? atoi(getenv("DMS_CHECK_INVARIANTS")) : 0;
    if (!env) return DMS_OK;
    CU(cudaStreamSynchronize(c->st));
    const int d = c->ndim;
    char m[200];
    int64_t chi = 0;
    for (int k = 0; k <= d; k++) chi += (k & 1) ? -c->ncrit[k] : c->ncrit[k];
    if (chi != 1) {
        std::snprintf(m, sizeof m, "invariant: Euler characteristic %lld != 1", (long long)chi);
        return fail(c, DMS_ERR_INVARIANT, m);
    }
    const int64_t p0 = pair_count(c, 0), pt = pair_count(c, 1);
    const int64_t u0 = unpaired_count(c, 0), ut = unpaired_count(c, 1);
    bool ok = p0 == c->ncrit[0] && u0 == c->ncrit[1] - (c->ncrit[0] - 1);
    if (d >= 2) ok = ok && pt == c->ncrit[d] && ut == c->ncrit[d - 1] - c->ncrit[d];
    if (d == 1) ok = ok && pt == c->ncrit[0];
    if (d == 2) ok = ok && u0 == pt;  // C_1 = D0 deaths + D1 (= D_{d-1}) births
    if (d == 3) ok = ok && u0 == ut;  // |D1| from both sides of the sandwich
    if (!ok) {
        std::snprintf(m, sizeof m, "invariant: diagram counts (C %lld %lld %lld %lld, D0 %lld, Dtop %lld, unpaired %lld %lld)",
                      (long long)c->ncrit[0], (long long)c->ncrit[1], (long long)c->ncrit[2], (long long)c->ncrit[3],
                      (long long)p0, (long long)pt, (long long)u0, (long long)ut);
        return fail(c, DMS_ERR_INVARIANT, m);
    }
    unsigned* bits = nullptr;
    unsigned long long* bad = nullptr;
    CU(dalloc(&bits, (c->N + 31) / 32 + 2));
    CU(cudaMemsetAsync(bits, 0, ((c->N + 31) / 32 + 2) * sizeof(unsigned), c->st));
    bad = reinterpret_cast<unsigned long long*>(bits + ((c->N + 31) / 32));
    k_check_perm<<<grid_for(c->N), kBlock, 0, c->st>>>(c->rank, c->N, bits, bad);
    c->launches++;
    unsigned long long hb = 0;
    CU(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    cudaFree(bits);
    if (hb) {
        std::snprintf(m, sizeof m, "invariant: rank is not a permutation (%llu collisions)", hb);
        return fail(c, DMS_ERR_INVARIANT, m);
    }
    return DMS_OK;
}

dms_status dms_run_all(dms_ctx* c, int32_t* d_rank, void* d_grad) {
    dms_status s = check_sticky(c);
    if (s) return s;
    static const int oseq_env = getenv("DMS_ORDER_SEQ") ? atoi(getenv("DMS_ORDER_SEQ")) : -1;
    if ((s = clear_err(c))) return s;
    // the order beside the gradient on a second stream (the one-sweep order on a small
    // grid hides behind the ALU-bound 3D gradient: c4 22.18 vs 25.12 ms order first;
    // DMS_ORDER_SEQ=0/1 forces either)
    const bool seq = oseq_env >= 0 ? oseq_env != 0 : false;
    // DMS_ORDER_SPLIT=k (3D): only the first k digit passes run beside the gradient; the
    // rest follow it on the full grid, beside the diagrams' tracing (A/B)
    static const int split_env = getenv("DMS_ORDER_SPLIT") ? atoi(getenv("DMS_ORDER_SPLIT")) : 0;
    c->os_defer_from = (!seq && c->ndim == 3 && split_env > 0 && split_env < 4) ? split_env : 4;
    s = run_order(c, d_rank, !seq);
    c->os_defer_from = 4;
    if (s) return s;
    if ((s = run_gradient(c, d_grad))) return s;
    if ((s = run_order_rest(c))) return s;
    c->early_traces = true;
    s = run_critical(c);
    c->early_traces = false;
    if (s) return s;
    if ((s = run_diagrams(c))) return s;
    return check_invariants(c);
}

dms_status dms_run_all_host(dms_ctx* c, const float* h_f, int32_t* d_rank, void* d_grad) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (!h_f) return DMS_ERR_ARG;
    // Upload in K slabs of whole planes (z in 3D, y in 2D, runs in 1D) on the second
    // stream; the gradient of slab i starts once slab i+1 (its upper halo plane) is in,
    // so the transfer hides behind the ALU-bound gradient.  The vertex order (which
    // needs every value) follows the last slab on the same stream.
    // 8..16 slabs of >= 32 MB (measured: 16 helps the 268-537 MB fields, hurts 64 MB)
    const int K = (int)std::min<int64_t>(kSlabs, std::max<int64_t>(8, c->N * 4 / (32 << 20)));
    for (int i = 0; i < K; i++)
        if (!c->ev_slab[i]) CU(cudaEventCreateWithFlags(&c->ev_slab[i], cudaEventDisableTiming));
    const int64_t plane = c->ndim == 3 ? c->L[0] * c->L[1] : (c->ndim == 2 ? c->L[0] : 1);
    const int64_t nplanes = c->N / plane;
    int64_t b[kSlabs + 1];
    for (int i = 0; i <= K; i++) b[i] = plane * (nplanes * i / K);
    if ((s = clear_err(c))) return s;
    CU(cudaEventRecord(c->ev_in, c->st));  // earlier work on the field is done
    CU(cudaStreamWaitEvent(c->st2, c->ev_in, 0));
    float* fdev = const_cast<float*>(c->f);
    for (int i = 0; i < K; i++) {
        if (b[i + 1] > b[i])
            CU(cudaMemcpyAsync(fdev + b[i], h_f + b[i], (size_t)(b[i + 1] - b[i]) * sizeof(float),
                               cudaMemcpyHostToDevice, c->st2));
        CU(cudaEventRecord(c->ev_slab[i], c->st2));
    }
    // the vertex order on the second stream, after the last slab: by then only the tail of
    // the gradient is left, so its persistent grid takes 2 CTAs per SM instead of the 1 of
    // the device-input path (c4 e2e: 1 / full grid / 2 per SM = 26.9 / 24.7 / 24.0 ms)
    {
        cudaStream_t main = c->st;
        c->st = c->st2;
        c->order_ctas_beside = 2;
        s = run_order_on_stream(c, d_rank, true);
        c->order_ctas_beside = 1;
        c->st = main;
        if (s) return s;
        CU(cudaEventRecord(c->ev_order, c->st2));
        c->order_pending = true;
    }
    c->grad = d_grad ? d_grad : c->grad_scratch;
    {
        StageTimer tm(c, 1);
        for (int i = 0; i < K; i++) {
            CU(cudaStreamWaitEvent(c->st, c->ev_slab[std::min(i + 1, K - 1)], 0));
            if ((s = launch_gradient(c, b[i], b[i + 1]))) return s;
        }
    }
    c->have_grad = true;
    c->order_fresh = false;
    c->have_crit = c->have_d[0] = c->have_d[1] = c->have_d1 = c->have_gen = c->have_ign = c->dtop_short = false;
    c->early_traces = true;
    s = run_critical(c);
    c->early_traces = false;
    if (s) return s;
    if ((s = run_diagrams(c))) return s;
    return check_invariants(c);
}

dms_status dms_sync(dms_ctx* c) {
    dms_status s = check_sticky(c);
    if (s) return s;
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(c, DMS_ERR_CUDA, "sync");
    return read_err(c);
}

int64_t dms_decode_pairs(const int64_t dims[3], int ndim, const void* h_words, int64_t v0, int64_t v1,
                         int64_t* h_triples, int64_t cap) {
    if (!dims || !h_words || !h_triples || ndim < 1 || ndim > 3 || v0 < 0 || v1 < v0) return -1;
    int64_t L[3] = {1, 1, 1};
    for (int i = 0; i < ndim; i++) L[i] = dims[i];
    StarTab T;
    if (!build_star_tables(ndim, L, &T)) return -1;
    const int64_t per[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 3, 2, 0}, {1, 7, 12, 6}};
    const int64_t* nc = per[ndim];
    int64_t n = 0;
    auto put = [&](int64_t a, int64_t b, int64_t c3) {
        if (n < cap) { h_triples[3 * n] = a; h_triples[3 * n + 1] = b; h_triples[3 * n + 2] = c3; }
        n++;
    };
    auto anc = [&](int64_t v, const int8_t o[3]) { return v + o[0] + L[0] * o[1] + L[0] * L[1] * o[2]; };
    for (int64_t v = v0; v < v1; v++) {
        const int64_t i = v - v0;
        if (ndim == 1) {
            const uint8_t w = reinterpret_cast<const uint8_t*>(h_words)[i];
            if (w == 0) put(0, v, v - 1);
            else if (w == 1) put(0, v, v);
            continue;
        }
        int vcode;
        uint64_t lo = 0, hi = 0;
        if (ndim == 3) {
            lo = reinterpret_cast<const uint64_t*>(h_words)[2 * i];
            hi = reinterpret_cast<const uint64_t*>(h_words)[2 * i + 1];
            vcode = (int)((lo >> 56) & 15);
            if (vcode == 15) vcode = -1;
        } else {
            const uint16_t w = reinterpret_cast<const uint16_t*>(h_words)[i];
            vcode = w & 7;
            if (vcode == 7) vcode = -1;
            lo = (uint64_t)(w >> 3);
        }
        if (vcode >= 0) put(0, v, nc[1] * anc(v, T.e_anc[vcode]) + T.e_k[vcode]);
        if (ndim == 3) {  // lo: a nibble per edge slot (1 + third vertex of the paired triangle); hi: tet codes
            for (int e = 0; e < T.ne; e++) {
                const int u = (int)((lo >> (4 * e)) & 15) - 1;
                if (u < 0) continue;
                const int t = T.tri_of[e][u];
                put(1, nc[1] * anc(v, T.e_anc[e]) + T.e_k[e], nc[2] * anc(v, T.t_anc[t]) + T.t_k[t]);
            }
            for (int q = 0; q < T.nq; q++) {
                const int code = (int)((hi >> (2 * q)) & 3);
                if (!code) continue;
                const int t = T.tet_tri[q][code - 1];
                put(2, nc[2] * anc(v, T.t_anc[t]) + T.t_k[t], nc[3] * anc(v, T.q_anc[q]) + T.q_k[q]);
            }
            continue;
        }
        for (int t = 0; t < T.nt; t++) {
            const int code = (int)((lo >> (2 * t)) & 3);
            if (!code) continue;
            const int e = code == 1 ? T.tri_a[t] : T.tri_b[t];
            put(1, nc[1] * anc(v, T.e_anc[e]) + T.e_k[e], nc[2] * anc(v, T.t_anc[t]) + T.t_k[t]);
        }
    }
    return n;
}

int64_t dms_decode_pairs2(const int64_t dims[3], int ndim, dms_complex cplx, const void* h_words, int64_t v0,
                          int64_t v1, int64_t* h_triples, int64_t cap) {
    if (cplx == DMS_COMPLEX_FREUDENTHAL) return dms_decode_pairs(dims, ndim, h_words, v0, v1, h_triples, cap);
    if (cplx != DMS_COMPLEX_5TET || !dims || !h_words || !h_triples || ndim != 3 || v0 < 0 || v1 < v0) return -1;
    const int64_t Lx = dims[0], Ly = dims[1], Lz = dims[2], N = Lx * Ly * Lz;
    if (v1 > N) return -1;
    T5Tab* T = new (std::nothrow) T5Tab;
    if (!T || !build_t5_tables(T)) { delete T; return -1; }
    const uint8_t* w = static_cast<const uint8_t*>(h_words);
    int64_t n = 0;
    auto put = [&](int64_t a, int64_t b, int64_t c3) {
        if (n < cap) { h_triples[3 * n] = a; h_triples[3 * n + 1] = b; h_triples[3 * n + 2] = c3; }
        n++;
    };
    // id of the cell spanned by the lattice points pts (tet5.cuh, reading Z21)
    auto id_of = [&](const int64_t (*pts)[3], int np) -> int64_t {
        int64_t a[3] = {pts[0][0], pts[0][1], pts[0][2]};
        for (int i = 1; i < np; i++)
            for (int ax = 0; ax < 3; ax++) a[ax] = std::min(a[ax], pts[i][ax]);
        int m[4];
        for (int i = 0; i < np; i++) m[i] = (int)((pts[i][0] - a[0]) | ((pts[i][1] - a[1]) << 1) | ((pts[i][2] - a[2]) << 2));
        std::sort(m, m + np);
        const int p = (int)((a[0] + a[1] + a[2]) & 1), k = np - 1;
        for (int i = 0; i < T->cnt[k]; i++) {
            bool eq = true;
            for (int j = 0; j < np; j++) eq = eq && T->ids[p][k][i][j] == m[j];
            if (eq) return (int64_t)T->cnt[k] * (a[0] + Lx * (a[1] + Ly * a[2])) + i;
        }
        return -1;
    };
    for (int64_t v = v0; v < v1; v++) {
        const int64_t x = v % Lx, y = (v / Lx) % Ly, z = v / (Lx * Ly);
        const int p = (int)((x + y + z) & 1);
        const int vc = w[v];
        if (vc != 0xff) {
            const T5Star& S = T->star[p];
            if (vc >= S.ne) { delete T; return -1; }
            put(0, v, 6 * (v + S.e_anc[vc][0] + Lx * S.e_anc[vc][1] + Lx * Ly * S.e_anc[vc][2]) + S.e_k[vc]);
        }
        for (int k = 2; k <= 3; k++) {
            const int64_t base = k == 2 ? N + 10 * v : 11 * N + 5 * v;
            for (int i = 0; i < T->cnt[k]; i++) {
                int64_t pts[4][3];
                bool inside = true;
                for (int j = 0; j <= k; j++) {
                    const int mm = T->ids[p][k][i][j];
                    pts[j][0] = x + (mm & 1);
                    pts[j][1] = y + ((mm >> 1) & 1);
                    pts[j][2] = z + ((mm >> 2) & 1);
                    inside = inside && pts[j][0] < Lx && pts[j][1] < Ly && pts[j][2] < Lz;
                }
                if (!inside) continue;
                const int code = w[base + i];
                if (code > k) continue;  // critical, or the tail of a vector
                int64_t fp[3][3];
                int q = 0;
                for (int j = 0; j <= k; j++)
                    if (j != code) { fp[q][0] = pts[j][0]; fp[q][1] = pts[j][1]; fp[q][2] = pts[j][2]; q++; }
                put(k - 1, id_of(fp, k), (int64_t)T->cnt[k] * v + i);
            }
        }
    }
    delete T;
    return n;
}

dms_status dms_copy(dms_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!c || (!dst && bytes) || (!src && bytes)) return DMS_ERR_ARG;
    if (!bytes) return DMS_OK;
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->st));
    CU(cudaStreamSynchronize(c->st));
    return DMS_OK;
}

dms_status dms_set_timing(dms_ctx* c, int enable) {
    if (!c) return DMS_ERR_ARG;
    cudaStreamSynchronize(c->st);
    clear_events(c);
    c->timing = enable != 0;
    return DMS_OK;
}

dms_status dms_stage_ms(dms_ctx* c, double ms_out[13]) {
    if (!c || !ms_out) return DMS_ERR_ARG;
    CU(cudaStreamSynchronize(c->st));
    for (int s = 0; s < 12; s++) {
        double t = 0;
        for (auto& p : c->ev[s]) {
            float x = 0;
            CU(cudaEventElapsedTime(&x, p.first, p.second));
            t += x;
        }
        ms_out[s < 6 ? s : s + 1] = t;
    }
    ms_out[6] = (double)c->ev[5].size();
    return DMS_OK;
}

int64_t dms_launch_count(const dms_ctx* c) { return c ? c->launches : 0; }

// internal diagnostics (not part of include/dms.h): live arcs per union-find round
#ifdef DMS_CHASE_STATS
int dms_internal_chase_stats(unsigned long long out[64], int reset) {
    if (reset) {
        unsigned long long z[64] = {0};
        return cudaMemcpyToSymbol(g_chase_hist, z, sizeof z) == cudaSuccess ? 0 : 1;
    }
    return cudaMemcpyFromSymbol(out, g_chase_hist, 64 * 8) == cudaSuccess ? 0 : 1;
}
#endif
int dms_internal_uf_trace2(dms_ctx* c, int which, int out[64], unsigned long long t[64]) {
    if (!c || which < 0 || which > 1 || !c->uf[which].trace) return 1;
    cudaStreamSynchronize(c->st);
    if (cudaMemcpy(out, c->uf[which].trace, 64 * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    return cudaMemcpy(t, c->uf[which].trace + 128, 64 * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}
// the last union-find launch of a diagram: arcs, cooperative grid, batch size (tests
// assert the residency-capped multi-tile rounds were reached: arcs > grid * kBlock)
int dms_internal_uf_launch(dms_ctx* c, int which, int64_t out[3]) {
    if (!c || which < 0 || which > 1 || !out) return 1;
    out[0] = c->uf[which].last_m;
    out[1] = c->uf[which].last_grid;
    out[2] = c->uf[which].last_batch;
    return 0;
}
// 1: the last union-find of diagram `which` ran in closed form on the 1D path (path1d.cuh)
int dms_internal_path_used(dms_ctx* c, int which) {
    if (!c || which < 0 || which > 1) return -1;
    return c->pb[which].used ? 1 : 0;
}

// rounds of the last D1 phases (1: pairs, 2: generators)
int dms_internal_d1_rounds(dms_ctx* c, int out[2]) {
    if (!c) return -1;
    out[0] = c->d1.rounds[0];
    out[1] = c->d1.rounds[1];
    return (int)std::min<int64_t>(c->d1.ntaint, 0x7fffffff);
}

int dms_internal_uf_trace(dms_ctx* c, int which, int out[64]) {
    if (!c || which < 0 || which > 1 || !c->uf[which].trace) return 1;
    cudaStreamSynchronize(c->st);
    return cudaMemcpy(out, c->uf[which].trace, 64 * sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}

const char* dms_last_error(const dms_ctx* c) { return c ? c->msg : "null context"; }

void dms_destroy(dms_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->st);
    if (c->st2) cudaStreamSynchronize(c->st2);
    if (c->lane3.st) cudaStreamSynchronize(c->lane3.st);
    if (c->lane4.st) cudaStreamSynchronize(c->lane4.st);
    clear_events(c);
    if (c->dt5) cudaFree(c->dt5);
    if (c->st2) cudaStreamDestroy(c->st2);
    for (cudaEvent_t e : {c->ev_grad, c->ev_trace[0], c->ev_trace[1]})
        if (e) cudaEventDestroy(e);
    for (Lane* Lp : {&c->lane3, &c->lane4}) {
        Lane& L = *Lp;
        if (L.st) cudaStreamDestroy(L.st);
        cudaFree(L.ss.counts);
        cudaFree(L.ss.counts_scan);
        cudaFree(L.ss.status);
        cudaFree(L.ss.tile_ctr);
        cudaFree(L.tile_ctr);
        if (L.h_pinned) cudaFreeHost(L.h_pinned);
    }
    for (cudaEvent_t e : {c->ev_crit, c->ev_d0})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->t_diag)
        if (e) cudaEventDestroy(e);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_order) cudaEventDestroy(c->ev_order);
    for (cudaEvent_t e : c->ev_slab)
        if (e) cudaEventDestroy(e);
    cudaFree(c->dtab);
    cudaFree(c->dlut3);
    if (c->ev_grad2) cudaEventDestroy(c->ev_grad2);
    cudaFree(c->dctab);
    cudaFree(c->rank_scratch);
    cudaFree(c->grad_scratch);
    for (int b = 0; b < 2; b++) { cudaFree(c->okeys[b]); cudaFree(c->ovals[b]); }
    for (int k = 0; k < 2; k++) {
        cudaFree(c->t1base[k]); cudaFree(c->t1cnt[k]); cudaFree(c->t1scan[k]); cudaFree(c->pmap[k]);
        PathBuf& b = c->pb[k];
        for (void* p : {(void*)b.sage, (void*)b.sarc, (void*)b.lw, (void*)b.rw, (void*)b.dw, (void*)b.bnd, (void*)b.tspan, (void*)b.unres,
                        (void*)b.pre, (void*)b.suf, (void*)b.npre, (void*)b.nsuf, (void*)b.tmin, (void*)b.bad})
            cudaFree(p);
        if (b.h_bad) cudaFreeHost(b.h_bad);
    }
    cudaFree(c->bm);
    cudaFree(c->bmcnt);
    cudaFree(c->bmpre);
    for (uint32_t* q : {c->ms_sidx, c->ms_slot, c->ms_cnt, c->ms_base}) cudaFree(q);
    cudaFree(c->ms_stage);
    cudaFree(c->os_hist);
    cudaFree(c->os_wcur);
    cudaFree(c->os_tctr);
    cudaFree(c->os_status);
    cudaFree(c->os_wbuf);
    cudaFree(c->ord_keys);
    cudaFree(c->ord_bid);
    for (int b = 0; b < 2; b++) { cudaFree(c->ord_skeys[b]); cudaFree(c->ord_svals[b]); }
    cudaFree(c->ord_spl);
    cudaFree(c->ord_counts);
    cudaFree(c->ord_offs);
    cudaFree(c->ss.counts);
    cudaFree(c->ss.counts_scan);
    cudaFree(c->ss.status);
    cudaFree(c->ss.tile_ctr);
    for (int b = 0; b < 2; b++)
        for (int k = 0; k < 4; k++) { cudaFree(c->cid[b][k]); cudaFree(c->ckey[b][k]); cudaFree(c->cidx[b][k]); }
    cudaFree(c->status);
    cudaFree(c->tile_ctr);
    cudaFree(c->chase_mark);
    cudaFree(c->lut2);
    cudaFree(c->cw);
    cudaFree(c->cw2);
    cudaFree(c->vc);
    cudaFree(c->totals);
    cudaFree(c->err);
    cudaFree(c->kmax);
    cudaFree(c->remaining);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    cudaFree(c->node_of0);
    cudaFree(c->node_oftop);
    for (int b = 0; b < 2; b++) {
        UFBuf& u = c->uf[b];
        for (void* p : {(void*)u.arc_a, (void*)u.arc_b, (void*)u.rec0, (void*)u.rec1, (void*)u.rsrc, (void*)u.out, (void*)u.list,
                        (void*)u.live2, (void*)u.nlive, (void*)u.trace, (void*)u.outp, (void*)u.key,
                        (void*)u.inv_a, (void*)u.age,
                        (void*)u.parent, (void*)u.best, (void*)u.flags, (void*)u.pos})
            cudaFree(p);
        if (u.h_status) cudaFreeHost(u.h_status);
        if (u.h_cnt) cudaFreeHost(u.h_cnt);
        cudaFree(c->pairs[b]);
        cudaFree(c->unp[b]);
    }
    {
        UFBuf& u = c->uf_ign;
        for (void* p : {(void*)u.arc_a, (void*)u.arc_b, (void*)u.rec0, (void*)u.rec1, (void*)u.rsrc, (void*)u.out, (void*)u.list,
                        (void*)u.live2, (void*)u.nlive, (void*)u.trace, (void*)u.outp, (void*)u.key,
                        (void*)u.inv_a, (void*)u.age, (void*)u.parent, (void*)u.best, (void*)u.flags, (void*)u.pos})
            cudaFree(p);
        if (u.h_status) cudaFreeHost(u.h_status);
        if (u.h_cnt) cudaFreeHost(u.h_cnt);
        cudaFree(c->pairs_ign);
    }
    {
        D1Buf& b = c->d1;
        for (void* p : {(void*)b.order, (void*)b.hkey, (void*)b.hval, (void*)b.owner, (void*)b.stop, (void*)b.done,
                        (void*)b.col_len, (void*)b.big, (void*)b.act[0], (void*)b.act[1], (void*)b.claim,
                        (void*)b.col_off, (void*)b.status, (void*)b.arena, (void*)b.ctr, (void*)b.flags,
                        (void*)b.pos, (void*)b.pairs, (void*)b.un1, (void*)b.gen_off, (void*)b.gen, (void*)b.stats,
                        (void*)b.deps, (void*)b.taint, (void*)b.tab, (void*)b.first_bad, (void*)b.best,
                        (void*)b.nadd, (void*)b.snaps})
            cudaFree(p);
        if (b.h_ctr) cudaFreeHost(b.h_ctr);
    }
    delete c;
}

}  // extern "C"
