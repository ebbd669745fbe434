// Host-side check (CPU, dev tool and tests/test_star_closed_form.py): the closed-form
// lower-star expansion process_star_fast() (grad.cuh) against the queue-driven
// process_star() on random 3D lower stars -- random lower masks over the 14-slot Kuhn
// star (every subcomplex the grid can produce, boundary stars included) and random
// local orders, with 1 in 7 full spheres (interior maxima).  Both functions are the
// product's own device code compiled for the host through the shims below; the oracle
// is not involved (the GPU parity tests compare the product with the oracle).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#define __device__
#define __host__
#define __forceinline__ inline
#define __global__
static inline int __ffs(unsigned x) { return __builtin_ffs((int)x); }
static inline int __ffsll(long long x) { return __builtin_ffsll(x); }
static inline int __popc(unsigned x) { return __builtin_popcount(x); }
static inline int __popcll(unsigned long long x) { return __builtin_popcountll(x); }
static inline unsigned __umulhi(unsigned a, unsigned b) { return (unsigned)(((unsigned long long)a * b) >> 32); }
using std::max; using std::min;
#include <algorithm>
#include "star.cuh"
#include "star_build.cuh"
namespace dms {
constexpr int kBlock = 256;
#include BODY_INC  // the device helpers of grad.cuh, extracted by the test
}
using namespace dms;
// the queue-driven expansion's 2-bit triangle codes as the closed form's edge nibbles
static uint64_t ecode_of(const StarTab& S, const StarState& a) {
    uint64_t e = 0;
    for (int t = 0; t < 36; t++) {
        const int code = (int)((t < 32 ? (a.tcode_lo >> (2 * t)) : (a.tcode_hi >> (2 * (t - 32)))) & 3ull);
        if (code == 1) e |= (uint64_t)(S.tri_b[t] + 1) << (4 * S.tri_a[t]);
        if (code == 2) e |= (uint64_t)(S.tri_a[t] + 1) << (4 * S.tri_b[t]);
    }
    return e;
}
int main(int argc, char** argv) {
    const long iters = argc > 1 ? atol(argv[1]) : 2000000;
    const unsigned long long seed = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
    int64_t L[3] = {10, 10, 10};
    static StarTab S;
    if (!build_star_tables(3, L, &S)) { printf("tables\n"); return 1; }
    static GradLut G;
    build_grad_lut(S, &G);
    long nsimple = 0, ntwo = 0;
    std::mt19937_64 rng(seed);
    static uint8_t tki[kMaxNT * kBlockG];
    static uint16_t qk[kMaxNQ * kBlockG];
    static uint8_t par[kMaxNE * kBlockG], tp[kMaxNE * kBlockG];
    long bad = 0, tot = 0;
    for (long it = 0; it < iters; it++) {
        // random lower mask + random ranks
        uint32_t Le = rng() & 0x3fff;
        if (it % 7 == 0) Le = 0x3fff;
        int n = __builtin_popcount(Le);
        if (!n) continue;
        int perm[14]; for (int i = 0; i < n; i++) perm[i] = i;
        std::shuffle(perm, perm + n, rng);
        uint64_t R = 0, IV = 0; int delta = 0;
        for (int s = 0, i = 0; s < 14; s++) if ((Le >> s) & 1) { R |= (uint64_t)perm[i] << (4*s); IV |= (uint64_t)s << (4*perm[i]); if (!perm[i]) delta = s; i++; }
        uint64_t ta = 0, tb = 0; uint32_t qa = 0, qb = 0, qc = 0;
        for (int s = 0; s < 14; s++) if ((Le >> s) & 1) { ta |= S.tri_amask[s]; tb |= S.tri_bmask[s]; qa |= S.tet_amask[s]; qb |= S.tet_bmask[s]; qc |= S.tet_cmask[s]; }
        StarState a{}, b{};
        a.Le = b.Le = Le; a.Lt = b.Lt = ta & tb; a.Lq = b.Lq = qa & qb & qc; a.vcode = b.vcode = -1;
        for (uint64_t m = a.Lt; m; m &= m - 1) { int t = __builtin_ctzll(m); tki[t * kBlockG] = (uint8_t)tri_kidx(S, R, t); }
        for (uint32_t m = a.Lq; m; m &= m - 1) { int q = __builtin_ctz(m); qk[q * kBlockG] = (uint16_t)cmp_tet(S, R, q); }
        KeyCache C; C.tki = tki; C.qk = qk; C.IV = IV; C.S = &S; C.R = R;
        process_star<3, true>(S, C, R, IV, n, delta, a);
        process_star_fast(S, G, R, IV, n, b, par, tp);
        tot++;
        // stars with one local minimum of the ranks on L (not the full sphere): the simple path
        {
            int nmin = 0;
            for (int s2 = 0; s2 < 14; s2++) if ((Le >> s2) & 1) {
                bool ismin = true;
                for (int u = 0; u < 14; u++) if (((S.adj[s2] & Le) >> u) & 1) if (rk(R, u) < rk(R, s2)) ismin = false;
                nmin += ismin;
            }
            // Lt / Lq through the union masks
            const uint32_t nl = ~Le & 0x3fffu;
            const uint64_t Lt2 = ((1ull << 36) - 1) & ~(G.ort[0][nl & 127] | G.ort[1][nl >> 7]);
            const uint32_t Lq2 = ((1u << 24) - 1) & ~(G.orq[0][nl & 127] | G.orq[1][nl >> 7]);
            if (Lt2 != a.Lt || Lq2 != a.Lq) { if (bad < 5) printf("lut masks Le=%04x\n", Le); bad++; }
            if (nmin <= 2 && Le != 0x3fffu) {
                StarState c{};
                c.Le = Le; c.Lt = a.Lt; c.Lq = a.Lq; c.vcode = -1;
                if (nmin == 1) process_star_simple(S, G, R, IV, n, c);
                else process_star_two(S, G, R, IV, n, c);
                if (nmin == 1) nsimple++; else ntwo++;
                if (!(a.vcode == c.vcode && ecode_of(S, a) == c.ecode && a.qcode == c.qcode &&
                      a.crit_e == c.crit_e && a.crit_t == c.crit_t && a.crit_q == c.crit_q)) {
                    if (bad < 5) printf("simple mismatch Le=%04x n=%d\n", Le, n);
                    bad++;
                }
            }
        }
        bool ok = a.vcode == b.vcode && ecode_of(S, a) == b.ecode && a.qcode == b.qcode &&
                  a.crit_e == b.crit_e && a.crit_t == b.crit_t && a.crit_q == b.crit_q;
        if (!ok) {
            if (bad < 5) printf("mismatch Le=%04x n=%d: crit_e %x/%x crit_t %llx/%llx crit_q %x/%x tc %llx/%llx q %llx/%llx\n", Le, n, a.crit_e, b.crit_e,
                (unsigned long long)a.crit_t, (unsigned long long)b.crit_t, a.crit_q, b.crit_q, (unsigned long long)ecode_of(S, a), (unsigned long long)b.ecode,
                (unsigned long long)a.qcode, (unsigned long long)b.qcode);
            bad++;
        }
    }
    printf("stars %ld mismatches %ld simple %ld two %ld\n", tot, bad, nsimple, ntwo);
    return bad ? 2 : 0;
}
