/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This file is the CPU checker for the B200 library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product library never links or calls it.  It is pinned against the
 * unmodified reference (oracle/_ref/libtsdref.so) and the committed golden
 * fixtures in tests/golden/ (tests/test_oracle.py).
 *
 * Build with -ffp-contract=off: the canonical reference build
 * (CMakeLists.txt: -O3, no -march) contains no FMA, and every function below
 * reproduces its IEEE-754 double operation order exactly.
 *
 * The MERLIN restatement does not re-implement the segment scan: the
 * reference proves that one pardrag(m, r^2) call returns exactly
 * {i : nn(i)^2 >= r^2} with the exact nn (tests/pardrag_test.cpp:108-135,
 * tests/acceptance_test.cpp:214-254), so orc_range_discords evaluates that set
 * directly from the brute-force nearest-neighbour profile
 * (src/drag.cpp:137-149) and orc_merlin drives it with the reference's
 * threshold schedule (src/merlin.cpp:18-132).
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
#define SIGMA_EPS 1e-12 /* include/tsdiscord/stats.hpp:11 */

static int err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---- generator: std::mt19937_64 + libstdc++ normal_distribution --------
 * src/io.cpp:110-119.  The polar method and generate_canonical<double,53>
 * follow libstdc++ (bits/random.tcc, GCC 13), the library the reference is
 * built against. */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

static double canonical(mt64* g) {
    double r = (double)mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

int orc_gen_randomwalk(int64_t n, uint64_t seed, double* out) {
    if (n < 3) return err(1, "gen_randomwalk: n must be at least 3");
    mt64 g;
    mt64_seed(&g, seed);
    int saved_ok = 0;
    double saved = 0.0;
    out[0] = 0.0;
    for (int64_t i = 1; i < n; ++i) {
        double ret;
        if (saved_ok) {
            saved_ok = 0;
            ret = saved;
        } else {
            double x, y, r2;
            do {
                x = 2.0 * canonical(&g) - 1.0;
                y = 2.0 * canonical(&g) - 1.0;
                r2 = x * x + y * y;
            } while (r2 > 1.0 || r2 == 0.0);
            const double mult = sqrt(-2 * log(r2) / r2);
            saved = x * mult;
            saved_ok = 1;
            ret = y * mult;
        }
        ret = ret * 1.0 + 0.0;
        out[i] = out[i - 1] + ret;
    }
    return 0;
}

/* ---- rolling stats: src/stats.cpp:7-36 (Eq. 4) and :38-58 (Eq. 7-8) ---- */
int orc_init_stats(const double* t, int64_t n, int64_t m, double* mu, double* sigma) {
    if (m < 2 || m > n - 1) return err(1, "init_stats: length out of range");
    const int64_t cnt = n - m + 1;
    double sum = 0.0, sum_sq = 0.0;
    for (int64_t k = 0; k < m; ++k) {
        sum += t[k];
        sum_sq += t[k] * t[k];
    }
    for (int64_t i = 0;; ++i) {
        const double mean = sum / (double)m;
        const double var = sum_sq / (double)m - mean * mean;
        mu[i] = mean;
        sigma[i] = sqrt(var > 0.0 ? var : 0.0);
        if (i + 1 >= cnt) break;
        const double o = t[i], in = t[i + m];
        sum += in - o;
        sum_sq += in * in - o * o;
    }
    return 0;
}

int orc_advance_stats(const double* t, int64_t n, int64_t m0, int64_t m1, double* mu,
                      double* sigma) {
    int rc = orc_init_stats(t, n, m0, mu, sigma);
    if (rc) return rc;
    for (int64_t m = m0; m < m1; ++m) {
        if (m + 1 > n - 1) return err(1, "advance_stats: next length out of range");
        const int64_t cnt = n - (m + 1) + 1;
        const double md = (double)m;
        for (int64_t i = 0; i < cnt; ++i) {
            const double u = mu[i], sg = sigma[i];
            const double in = t[i + m];
            const double delta = u - in;
            mu[i] = (md * u + in) / (md + 1.0);
            const double var = md / (md + 1.0) * (sg * sg + delta * delta / (md + 1.0));
            sigma[i] = sqrt(var > 0.0 ? var : 0.0);
        }
    }
    return 0;
}

/* ---- exact distance: znormalize + sq_ed (src/distance.cpp:8-33) under the
 * constant conventions of reference_sq_dist (src/pardrag.cpp:57-69) and
 * ZnormCache::dist (src/drag.cpp:24-58). ---------------------------------- */
static int znorm(const double* x, int64_t m, double* z) {
    double sum = 0.0, sum_sq = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        sum += x[i];
        sum_sq += x[i] * x[i];
    }
    const double mu = sum / (double)m;
    const double var = sum_sq / (double)m - mu * mu;
    const double sg = sqrt(var > 0.0 ? var : 0.0);
    int is_const = 1;
    if (sg < SIGMA_EPS) {
        memset(z, 0, sizeof(double) * (size_t)m);
        return 1;
    }
    for (int64_t i = 0; i < m; ++i) {
        z[i] = (x[i] - mu) / sg;
        if (z[i] != 0.0) is_const = 0;
    }
    return is_const;
}

static double sq_ed(const double* a, const double* b, int64_t m) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    return s;
}

double orc_ref_sq_dist(const double* t, int64_t n, int64_t m, int64_t i, int64_t j) {
    (void)n;
    double* zi = malloc(sizeof(double) * (size_t)m);
    double* zj = malloc(sizeof(double) * (size_t)m);
    const int ci = znorm(t + i - 1, m, zi), cj = znorm(t + j - 1, m, zj);
    double d;
    if (ci && cj) d = 0.0;
    else if (ci || cj) d = 2.0 * (double)m;
    else d = sq_ed(zi, zj, m);
    free(zi);
    free(zj);
    return d;
}

/* brute_force_nn: src/drag.cpp:137-149 (non-self: |i-j| >= m, types.cpp:22-24) */
int orc_brute_force_nn(const double* t, int64_t n, int64_t m, double* nn) {
    if (m < 3 || m > n) return err(1, "brute_force_nn: bad length");
    const int64_t cnt = n - m + 1;
    double* z = malloc(sizeof(double) * (size_t)(cnt * m));
    char* cst = malloc((size_t)cnt);
    if (!z || !cst) return err(3, "oom");
    for (int64_t i = 0; i < cnt; ++i) {
        cst[i] = (char)znorm(t + i, m, z + i * m);
        nn[i] = INFINITY;
    }
    for (int64_t i = 0; i < cnt; ++i) {
        for (int64_t j = i + m; j < cnt; ++j) {
            double d;
            if (cst[i] && cst[j]) d = 0.0;
            else if (cst[i] || cst[j]) d = 2.0 * (double)m;
            else d = sq_ed(z + i * m, z + j * m, m);
            if (d < nn[i]) nn[i] = d;
            if (d < nn[j]) nn[j] = d;
        }
    }
    free(z);
    free(cst);
    return 0;
}

/* sort order: nn_dist_sq desc, index asc (src/types.cpp:15-20) */
static int rec_cmp(const void* a, const void* b) {
    const orc_record* x = a;
    const orc_record* y = b;
    if (x->nn_dist_sq != y->nn_dist_sq) return x->nn_dist_sq > y->nn_dist_sq ? -1 : 1;
    return (x->index > y->index) - (x->index < y->index);
}

static int64_t range_from_nn(const double* nn, int64_t cnt, double r_sq, orc_record* recs,
                             int64_t cap) {
    int64_t k = 0;
    for (int64_t i = 0; i < cnt; ++i) {
        if (nn[i] >= r_sq) {
            if (k < cap) recs[k] = (orc_record){i + 1, nn[i], sqrt(nn[i])};
            ++k;
        }
    }
    qsort(recs, (size_t)(k < cap ? k : cap), sizeof(orc_record), rec_cmp);
    return k;
}

/* pardrag(m, r_sq) == {i : nn(i) >= r_sq}, exact nn, sorted. */
int64_t orc_range_discords(const double* t, int64_t n, int64_t m, double r_sq, orc_record* recs,
                           int64_t cap) {
    const int64_t cnt = n - m + 1;
    double* nn = malloc(sizeof(double) * (size_t)cnt);
    const int rc = orc_brute_force_nn(t, n, m, nn);
    if (rc) {
        free(nn);
        return -rc;
    }
    const int64_t k = range_from_nn(nn, cnt, r_sq, recs, cap);
    free(nn);
    return k;
}

/* compute_layout: src/types.cpp:26-39 */
int orc_compute_layout(int64_t n, int64_t m, int64_t seglen, int64_t out[4]) {
    if (m < 3) return err(1, "subsequence length must be at least 3");
    if (m > n - 2) return err(1, "subsequence length too large for series");
    if (seglen < m) return err(1, "segment length must be at least the subsequence length");
    if (n < seglen) return err(1, "series shorter than one segment");
    const int64_t seg_n = seglen - m + 1, cnt = n - m + 1;
    const int64_t num_seg = (cnt + seg_n - 1) / seg_n;
    out[0] = seglen;
    out[1] = seg_n;
    out[2] = num_seg;
    out[3] = num_seg * seg_n + 2 * (m - 1) - n;
    return 0;
}

/* ThresholdHistory / next_threshold: src/merlin.cpp:18-55 */
static int window_stats(const double* h, int64_t len, double* mean, double* sd) {
    if (len < 5) return err(2, "threshold history window too short");
    double s = 0.0;
    for (int64_t k = len - 5; k < len; ++k) s += h[k];
    const double mu = s / 5.0;
    double q = 0.0;
    for (int64_t k = len - 5; k < len; ++k) {
        const double d = h[k] - mu;
        q += d * d;
    }
    *mean = mu;
    *sd = sqrt(q / 5.0);
    return 0;
}

int orc_next_threshold(const double* h, int64_t len, int phase, int64_t min_len, double last_r,
                       int failed, double* out) {
    double mu, sd;
    int rc;
    switch (phase) {
        case 0: /* first */
            *out = failed ? 0.5 * last_r : 2.0 * sqrt((double)min_len);
            return 0;
        case 1: /* warmup */
            if (!failed && len < 1) return err(2, "empty history");
            *out = 0.99 * (failed ? last_r : h[len - 1]);
            return 0;
        case 2: /* steady */
            if ((rc = window_stats(h, len, &mu, &sd))) return rc;
            if (failed) {
                const double e = 0.01 * last_r;
                *out = last_r - (sd > e ? sd : e);
                return 0;
            }
            {
                const double r = mu - 2.0 * sd;
                *out = r <= 0.0 ? 0.01 * h[len - 1] : r;
            }
            return 0;
    }
    return err(2, "unreachable");
}

/* merlin_full: src/merlin.cpp:57-132 */
int orc_merlin(const double* t, int64_t n, int64_t min_len, int64_t max_len, int64_t top_k,
               int64_t seglen, int64_t workers, int64_t max_retries, int reuse_stats,
               int64_t* counts, orc_record* recs, double* final_r, int64_t* retries,
               uint8_t* failed) {
    (void)workers;
    (void)reuse_stats; /* stats only steer the scan; the range set does not depend on them */
    if (min_len < 3 || min_len > max_len || 2 * max_len > n)
        return err(1, "merlin: length range out of bounds (need 3 <= minL <= maxL <= n/2)");
    if (top_k < 1) return err(1, "merlin: topK must be positive");
    const int64_t L = max_len - min_len + 1;
    double* hist = malloc(sizeof(double) * (size_t)L);
    int64_t hlen = 0;
    int rc = 0;
    for (int64_t m = min_len; m <= max_len; ++m) {
        const int64_t k = m - min_len;
        const int phase = m == min_len ? 0 : (m < min_len + 5 ? 1 : 2);
        counts[k] = 0;
        failed[k] = 0;
        if (phase != 0 && hlen == 0) {
            failed[k] = 1;
            final_r[k] = 0.0;
            retries[k] = 0;
            continue;
        }
        int64_t lay[4];
        const int64_t sl0 = seglen > 2 * m ? seglen : 2 * m;
        if ((rc = orc_compute_layout(n, m, sl0 < n ? sl0 : n, lay))) break;
        const int64_t cnt = n - m + 1;
        double* nn = malloc(sizeof(double) * (size_t)cnt);
        orc_record* cur = malloc(sizeof(orc_record) * (size_t)cnt);
        if ((rc = orc_brute_force_nn(t, n, m, nn))) {
            free(nn);
            free(cur);
            break;
        }
        double r;
        if ((rc = orc_next_threshold(hist, hlen, phase, min_len, 0.0, 0, &r))) {
            free(nn);
            free(cur);
            break;
        }
        int64_t tries = 0, got = 0;
        int success = 0;
        for (;;) {
            const double r_sq = r > 0.0 ? r * r : 0.0;
            got = range_from_nn(nn, cnt, r_sq, cur, cnt);
            if (got >= top_k) {
                success = 1;
                break;
            }
            if (tries >= max_retries) {
                success = got > 0;
                break;
            }
            ++tries;
            if ((rc = orc_next_threshold(hist, hlen, phase, min_len, r, 1, &r))) break;
        }
        if (rc) {
            free(nn);
            free(cur);
            break;
        }
        final_r[k] = r;
        retries[k] = tries;
        if (!success) {
            failed[k] = 1;
        } else {
            const int64_t keep = got < top_k ? got : top_k;
            double mn = cur[0].nn_dist;
            for (int64_t j = 0; j < keep; ++j) {
                recs[k * top_k + j] = cur[j];
                if (cur[j].nn_dist < mn) mn = cur[j].nn_dist;
            }
            counts[k] = keep;
            hist[hlen++] = mn;
        }
        free(nn);
        free(cur);
    }
    free(hist);
    return rc;
}
