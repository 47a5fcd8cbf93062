// Host simulation of the chunked exact-chain algorithm (test harness only).
// Builds with: g++ -O2 -ffp-contract=off -shared -fPIC
// Checks that offset-map prediction reproduces the sequential reference chain.
#include "../../paper_1805_07384_b200/csrc/lc_chain.cuh"
#include <vector>
#include <stdio.h>

extern "C" {

// Returns the number of chunks whose predicted start differs from the exact
// chain; *first_bad gets the first such chunk (-1 if none).  mode 0 = scan the
// maps sequentially, mode 1 = compose them in a balanced tree first.
int64_t sim_predict(const double *x, int64_t n, double eb, int64_t nbh, int L,
                    int mode, int64_t *first_bad, int64_t *n_events)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = (double)(nbh - 1); Q.max_m1 = Q.max_m + 1.0; Q.inv = 1.0 / Q.delta;
    const int64_t nc = (n - 1 + L - 1) / L;
    std::vector<double> guess(nc), rend(nc);
    std::vector<OffMap> maps(nc);
    const double x0 = x[0];
    int64_t events = 0, flagged = 0;
    *n_events = 0;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L;
        double g;
        if (c == 0) g = x0;
        else {
            const double Qn = floor((x[s] - x0) / Q.delta + 0.5);
            g = x0 + Qn * Q.delta;
        }
        guess[c] = g;
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L;
        const int64_t e = (s + L < n - 1) ? s + L : n - 1;
        double r = guess[c];
        OffMap H = lc_map_identity(lc_ulp(r));
        LcFlags F; lc_flags_init(F, r);
        int anyesc = 0;
        const double g0 = r;
        double rs = r;                               // chain value before the first flagged step
        int jj = 0;
        for (int64_t i = s + 1; i <= e; ++i) {
            uint32_t code; double inc; int esc; double pe;
            const double rn = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
            if (esc) { H = lc_map_const(0.0); anyesc = 1; }
            else {
                const bool f = lc_flag_test(F, r, inc, rn);  // every step, as the kernels do
                rs = (f && F.mask == 0u) ? r : rs;
                F.mask |= (unsigned)f << (jj & 31);
                if (inc != 0.0) {
                    const int kb = H.kind;
                    const double Bb = H.B;
                    lc_map_step(H, r, inc, rn);
                    if (H.kind != kb || H.B != Bb) ++events;
                }
            }
            r = rn;
            ++jj;
        }
        {   // the flag tracker + replay must reproduce the step-by-step map exactly
            OffMap H2 = anyesc ? lc_map_const(0.0) : lc_map_identity(lc_ulp(g0));
            if (!anyesc && F.mask) {                 // replay the first to the last flagged step
                const int j0 = __builtin_ctz(F.mask), j1 = 31 - __builtin_clz(F.mask);
                double r2 = rs;
                for (int j2 = j0; j2 <= j1; ++j2) {
                    uint32_t code; double inc; int esc; double pe;
                    const double rn = lc_step(Q, x[s + 1 + j2], r2, &code, &esc, &inc, &pe);
                    if (((F.mask >> j2) & 1u) && inc != 0.0) lc_map_step(H2, r2, inc, rn);
                    r2 = rn;
                }
                flagged += __builtin_popcount(F.mask);
            }
            {
                if (H2.kind != H.kind || lc_bits(H2.y) != lc_bits(H.y) || lc_bits(H2.t0) != lc_bits(H.t0) ||
                    lc_bits(H2.t1) != lc_bits(H.t1) || lc_bits(H2.B) != lc_bits(H.B))
                    *n_events = -1000000000;
            }
        }
        rend[c] = r;
        if (c + 1 < nc) lc_map_shift_out(H, r - guess[c + 1]);
        maps[c] = H;
    }
    // predicted D at each chunk start
    std::vector<double> D(nc);
    D[0] = 0.0;
    if (mode == 0) {
        for (int64_t c = 0; c + 1 < nc; ++c) D[c + 1] = lc_map_eval(maps[c], D[c]);
    } else {
        // inclusive prefix via Hillis-Steele composition (tests associativity)
        std::vector<OffMap> pre(maps), tmp(nc);
        for (int64_t off = 1; off < nc; off <<= 1) {
            for (int64_t c = 0; c < nc; ++c)
                tmp[c] = (c >= off) ? lc_map_compose(pre[c], pre[c - off]) : pre[c];
            pre.swap(tmp);
        }
        for (int64_t c = 0; c + 1 < nc; ++c) D[c + 1] = lc_map_eval(pre[c], 0.0);
    }
    // exact chain
    int64_t bad = 0; *first_bad = -1;
    double r = x0;
    for (int64_t c = 0; c < nc; ++c) {
        const double pred = guess[c] + D[c];
        if (lc_bits(pred) != lc_bits(r)) { if (*first_bad < 0) *first_bad = c; ++bad; }
        const int64_t s = c * L;
        const int64_t e = (s + L < n - 1) ? s + L : n - 1;
        for (int64_t i = s + 1; i <= e; ++i) {
            uint32_t code; double inc; int esc; double pe;
            r = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
        }
    }
    if (*n_events >= 0) *n_events = events * 1000000 + flagged;   // true map changes, flagged steps
    return bad;
}

// Exact sequential chain codes (for cross-checking lc_step with the oracle).
int64_t sim_codes(const double *x, int64_t n, double eb, int64_t nbh, uint32_t *codes, double *recon)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = (double)(nbh - 1); Q.max_m1 = Q.max_m + 1.0; Q.inv = 1.0 / Q.delta;
    double r = x[0]; recon[0] = r; int64_t ne = 0;
    for (int64_t i = 1; i < n; ++i) {
        double inc; int esc; double pe;
        r = lc_step(Q, x[i], r, &codes[i - 1], &esc, &inc, &pe);
        recon[i] = r; ne += esc;
    }
    return ne;
}
}

extern "C" {
// Brute-force check of lc_map_compose on consecutive chunk maps: returns the
// number of (pair, D) probes where compose(H2,H1)(D) != H2(H1(D)).
int64_t sim_compose_check(const double *x, int64_t n, double eb, int L, int span, int verbose)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = 32767.0; Q.max_m1 = 32768.0; Q.inv = 1.0 / Q.delta;
    const int64_t nc = (n - 1 + L - 1) / L;
    std::vector<double> guess(nc);
    std::vector<OffMap> maps(nc);
    const double x0 = x[0];
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L;
        guess[c] = c == 0 ? x0 : x0 + floor((x[s] - x0) / Q.delta + 0.5) * Q.delta;
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L, e = (s + L < n - 1) ? s + L : n - 1;
        double r = guess[c];
        OffMap H = lc_map_identity(lc_ulp(r));
        for (int64_t i = s + 1; i <= e; ++i) {
            uint32_t code; double inc; int esc; double pe;
            const double rn = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
            if (esc) H = lc_map_const(0.0);
            else if (inc != 0.0) lc_map_step(H, r, inc, rn);
            r = rn;
        }
        if (c + 1 < nc) lc_map_shift_out(H, r - guess[c + 1]);
        maps[c] = H;
    }
    int64_t bad = 0, shown = 0;
    for (int64_t c = 0; c + 1 < nc; ++c) {
        OffMap acc = maps[c];
        for (int len = 1; len < 4 && c + len < nc; ++len) {
            const OffMap nxt = maps[c + len];
            OffMap C;
            if (verbose >= 2) {             // right-associated: maps[c+len] o (... o maps[c+1]) then o maps[c]
                OffMap r2 = maps[c + len];
                for (int t = len - 1; t >= 1; --t) r2 = lc_map_compose(r2, maps[c + t]);
                C = lc_map_compose(r2, maps[c]);
            } else C = lc_map_compose(nxt, acc);
            const double v = maps[c].v > 0 ? maps[c].v : 1e-300;
            for (int k = -span; k <= span; ++k) {
                const double D = k * v;
                double ref = D;
                for (int t = 0; t <= len; ++t) ref = lc_map_eval(maps[c + t], ref);
                const double got = lc_map_eval(C, D);
                if (lc_bits(got) != lc_bits(ref)) {
                    ++bad;
                    if (verbose && shown < 4) {
                        ++shown;
                        printf("c=%ld len=%d D=%.17g ref=%.17g got=%.17g\n", (long)c, len, D, ref, got);
                        const OffMap *ms[2] = {&acc, &nxt};
                        for (int q = 0; q < 2; ++q)
                            printf("  %s kind=%d v=%.6g B=%.6g t0=%.17g t1=%.17g y=%.17g\n", q ? "H2" : "H1",
                                   ms[q]->kind, ms[q]->v, ms[q]->B, ms[q]->t0, ms[q]->t1, ms[q]->y);
                        printf("  C  kind=%d v=%.6g B=%.6g t0=%.17g t1=%.17g y=%.17g\n", C.kind, C.v, C.B, C.t0, C.t1, C.y);
                    }
                }
            }
            acc = C;
        }
    }
    return bad;
}
}
extern "C" {
// Left-fold vs balanced-tree composition: compares prefix evaluations at 0.
int64_t sim_tree_debug(const double *x, int64_t n, double eb, int L)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = 32767.0; Q.max_m1 = 32768.0; Q.inv = 1.0 / Q.delta;
    const int64_t nc = (n - 1 + L - 1) / L;
    std::vector<double> guess(nc);
    std::vector<OffMap> maps(nc);
    const double x0 = x[0];
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L;
        guess[c] = c == 0 ? x0 : x0 + floor((x[s] - x0) / Q.delta + 0.5) * Q.delta;
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L, e = (s + L < n - 1) ? s + L : n - 1;
        double r = guess[c];
        OffMap H = lc_map_identity(lc_ulp(r));
        for (int64_t i = s + 1; i <= e; ++i) {
            uint32_t code; double inc; int esc; double pe;
            const double rn = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
            if (esc) H = lc_map_const(0.0);
            else if (inc != 0.0) lc_map_step(H, r, inc, rn);
            r = rn;
        }
        if (c + 1 < nc) lc_map_shift_out(H, r - guess[c + 1]);
        maps[c] = H;
    }
    // sequential D
    std::vector<double> D(nc + 1);
    D[0] = 0;
    for (int64_t c = 0; c < nc; ++c) D[c + 1] = lc_map_eval(maps[c], D[c]);
    // compose pairs (2c, 2c+1), check the pair maps at the actual D
    int64_t bad = 0;
    for (int64_t c = 0; c + 1 < nc; c += 2) {
        OffMap C = lc_map_compose(maps[c + 1], maps[c]);
        double got = lc_map_eval(C, D[c]);
        if (lc_bits(got) != lc_bits(D[c + 2])) {
            if (bad < 3) {
                printf("pair c=%ld D=%.17g mid=%.17g ref=%.17g got=%.17g\n", (long)c, D[c], D[c+1], D[c + 2], got);
                const OffMap *ms[3] = {&maps[c], &maps[c + 1], &C};
                for (int q = 0; q < 3; ++q)
                    printf("  kind=%d v=%.6g B=%.6g t0=%.17g t1=%.17g y=%.17g\n",
                           ms[q]->kind, ms[q]->v, ms[q]->B, ms[q]->t0, ms[q]->t1, ms[q]->y);
            }
            ++bad;
        }
    }
    return bad;
}
}
extern "C" {
int64_t sim_tree_debug2(const double *x, int64_t n, double eb, int L)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = 32767.0; Q.max_m1 = 32768.0; Q.inv = 1.0 / Q.delta;
    const int64_t nc = (n - 1 + L - 1) / L;
    std::vector<double> guess(nc);
    std::vector<OffMap> maps(nc);
    const double x0 = x[0];
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L;
        guess[c] = c == 0 ? x0 : x0 + floor((x[s] - x0) / Q.delta + 0.5) * Q.delta;
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L, e = (s + L < n - 1) ? s + L : n - 1;
        double r = guess[c];
        OffMap H = lc_map_identity(lc_ulp(r));
        for (int64_t i = s + 1; i <= e; ++i) {
            uint32_t code; double inc; int esc; double pe;
            const double rn = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
            if (esc) H = lc_map_const(0.0);
            else if (inc != 0.0) lc_map_step(H, r, inc, rn);
            r = rn;
        }
        if (c + 1 < nc) lc_map_shift_out(H, r - guess[c + 1]);
        maps[c] = H;
    }
    std::vector<double> D(nc + 1);
    D[0] = 0;
    for (int64_t c = 0; c < nc; ++c) D[c + 1] = lc_map_eval(maps[c], D[c]);
    std::vector<OffMap> pre(maps), tmp(nc);
    int level = 0;
    for (int64_t off = 1; off < nc; off <<= 1, ++level) {
        for (int64_t c = 0; c < nc; ++c) {
            tmp[c] = (c >= off) ? lc_map_compose(pre[c], pre[c - off]) : pre[c];
            const int64_t lo = c - 2 * off + 1 < 0 ? 0 : c - 2 * off + 1;
            const double got = lc_map_eval(tmp[c], D[lo]);
            if (lc_bits(got) != lc_bits(D[c + 1])) {
                printf("level %d c=%ld lo=%ld Dlo=%.17g Dmid=%.17g ref=%.17g got=%.17g\n", level, (long)c, (long)lo,
                       D[lo], c >= off ? D[c - off + 1] : -1.0, D[c + 1], got);
                const OffMap *ms[3] = {&pre[c - off], &pre[c], &tmp[c]};
                const char *nm[3] = {"H1", "H2", "C "};
                for (int q = 0; q < 3; ++q)
                    printf("  %s kind=%d v=%.6g B=%.6g t0=%.17g t1=%.17g y=%.17g\n", nm[q],
                           ms[q]->kind, ms[q]->v, ms[q]->B, ms[q]->t0, ms[q]->t1, ms[q]->y);
                printf("  H1(Dlo)=%.17g  H2(H1(Dlo))=%.17g\n", lc_map_eval(pre[c-off], D[lo]), lc_map_eval(pre[c], lc_map_eval(pre[c-off], D[lo])));
                return 1;
            }
        }
        pre.swap(tmp);
    }
    return 0;
}
}
extern "C" {
// histogram of recorded events per chunk (deferred tracker), hist[0..15]
void sim_event_hist(const double *x, int64_t n, double eb, int L, int64_t *hist)
{
    LcQuant Q;
    Q.delta = 2.0 * eb; Q.eb = eb; Q.max_m = 32767.0; Q.max_m1 = 32768.0; Q.inv = 1.0 / Q.delta;
    const int64_t nc = (n - 1 + L - 1) / L;
    const double x0 = x[0];
    for (int i = 0; i < 16; ++i) hist[i] = 0;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t s = c * L, e = (s + L < n - 1) ? s + L : n - 1;
        double r = c == 0 ? x0 : x0 + floor((x[s] - x0) / Q.delta + 0.5) * Q.delta;
        LcFlags F; lc_flags_init(F, r);
        int jj = 0, anyesc = 0;
        for (int64_t i = s + 1; i <= e; ++i, ++jj) {
            uint32_t code; double inc; int esc; double pe;
            const double rn = lc_step(Q, x[i], r, &code, &esc, &inc, &pe);
            if (esc) anyesc = 1; else lc_flags_step(F, jj, r, inc, rn);
            r = rn;
        }
        const int ne = anyesc ? 0 : __builtin_popcount(F.mask);
        hist[ne < 15 ? ne : 15]++;
    }
}
}
