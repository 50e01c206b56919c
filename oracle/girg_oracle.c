/*
 * girg_oracle.c -- plain sequential CPU oracle for the GIRG hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see girg_oracle.h).  Not linked, imported or executed by the
 * product path; shares no code with paper_1905_06706_b200/.
 *
 * Built with: gcc -O2 -std=c99 -ffp-contract=off -fPIC -shared -lm   (no FMA contraction:
 * the canonical arithmetic of DESIGN.md "Canonical arithmetic" is evaluated literally).
 *
 * Citations "P:NNN" are lines of PAPER.md (arXiv:1905.06706).  Readings R1..R26 are listed
 * in DESIGN.md; they resolve the places where the paper is silent or garbled.
 */
#define _GNU_SOURCE
#include "girg_oracle.h"

#include <limits.h>
#include <math.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================================== */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  Key = (lo32(seed), hi32(seed)).   */
/* R17: all randomness is counter-based and keyed, so the edge set does not depend on   */
/* evaluation order (replaces the thread-local generators of P:1281-1282).              */
/* ===================================================================================== */
void or_philox4x32_10(const uint32_t ctr[4], uint64_t seed, uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u; /* Weyl key schedule */
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* uniform in [0,1) on the 2^-53 grid from two 32-bit words (hi, lo) */
double or_u53(uint32_t hi, uint32_t lo)
{
    uint64_t b = (((uint64_t)hi << 32) | (uint64_t)lo) >> 11;
    return (double)b * 0x1p-53;
}

/* TEST HOOK for the near-tie detector (O12 pin, tests/test_oracle_sampler.py): when a mode
 * bit is set, the decision variable of that kind is moved to (threshold + delta) before the
 * detector and the decision run, so a test can check that the detector fires inside its window
 * and stays silent outside it, on every decision of that kind.  Bit 1: type-I uniform
 * r := p_uv + delta (decisions with p_uv < 1).  Bit 2: type-II acceptance r_acc := p_uv/pbar +
 * delta.  Bit 4: jump quotient z := nearbyint(z) + delta*max(1,|z|).  Off (0) by default; never
 * set outside tests. */
static int or_tie_mode = 0;
static double or_tie_delta = 0.0;
void or_set_tie_hook(int mode, double delta)
{
    or_tie_mode = mode;
    or_tie_delta = delta;
}

/* ===================================================================================== */
/* Model, Sec. 2.1                                                           */
/* ===================================================================================== */

/* ===================================================================================== */
/* R26: the canonical log / exp / pow of the edge decisions.  Written with + - * / and bit   */
/* operations only (no libm), so the oracle and the CUDA library (which implements the same */
/* formulas independently) compute identical bits: T > 0 decisions cannot differ by a libm   */
/* ulp any more.  Accuracy (pinned against glibc by tests/test_oracle_model.py): log within */
/* 2 ulp, exp within 2 ulp, pow within 1e-13 relative over the decisions' range.            */
/* ===================================================================================== */
static const double OR_LN2_HI = 0x1.62e42fee00000p-1; /* 21 trailing zero bits: k*LN2_HI exact */
static const double OR_LN2_LO = 0x1.a39ef35793c76p-33;

static double or_pow2i(int k) /* 2^k for -1022 <= k <= 1023 */
{
    uint64_t b = (uint64_t)(k + 1023) << 52;
    double r;
    memcpy(&r, &b, 8);
    return r;
}

/* log x, x > 0 finite: x = m 2^k, m in [sqrt(1/2), sqrt(2)); s = (m-1)/(m+1);
 * log m = 2 atanh(s) = 2 s (1 + s^2/3 + s^4/5 + ... + s^22/23) (|s| <= 0.172, the next term is
 * below 2^-60 relative); log x = k ln2_hi + (k ln2_lo + log m) */
double or_det_log(double x)
{
    if (!(x > 0.0)) return x == 0.0 ? -INFINITY : NAN;
    if (isinf(x)) return x;
    int k = 0;
    uint64_t b;
    memcpy(&b, &x, 8);
    if (((b >> 52) & 0x7ff) == 0) { /* subnormal: scale into the normal range */
        x = x * 0x1p54;
        k = -54;
        memcpy(&b, &x, 8);
    }
    k += (int)((b >> 52) & 0x7ff) - 1023;
    b = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
    double m;
    memcpy(&m, &b, 8); /* m in [1, 2) */
    if (m > 0x1.6a09e667f3bcdp+0) { /* sqrt(2) */
        m = m * 0.5;
        k += 1;
    }
    double f = m - 1.0;
    double s = f / (m + 1.0);
    double z = s * s;
    double p = 0x1.642c8590b2164p-5;        /* 1/23 */
    p = p * z + 0x1.8618618618618p-5;       /* 1/21 */
    p = p * z + 0x1.af286bca1af28p-5;       /* 1/19 */
    p = p * z + 0x1.e1e1e1e1e1e1ep-5;       /* 1/17 */
    p = p * z + 0x1.1111111111111p-4;       /* 1/15 */
    p = p * z + 0x1.3b13b13b13b14p-4;       /* 1/13 */
    p = p * z + 0x1.745d1745d1746p-4;       /* 1/11 */
    p = p * z + 0x1.c71c71c71c71cp-4;       /* 1/9 */
    p = p * z + 0x1.2492492492492p-3;       /* 1/7 */
    p = p * z + 0x1.999999999999ap-3;       /* 1/5 */
    p = p * z + 0x1.5555555555555p-2;       /* 1/3 */
    double logm = (2.0 * s) + (2.0 * s) * (z * p);
    double kd = (double)k;
    return kd * OR_LN2_HI + (kd * OR_LN2_LO + logm);
}

/* exp t: k = round-half-even(t / ln2), r = (t - k ln2_hi) - k ln2_lo (|r| <= 0.35),
 * exp r = sum_{i <= 13} r^i / i! (Horner), times 2^k (two exact-or-IEEE-rounded multiplies) */
double or_det_exp(double t)
{
    if (isnan(t)) return t;
    if (t > 709.78) return INFINITY;
    if (t < -745.2) return 0.0;
    double kd = nearbyint(t * 0x1.71547652b82fep+0); /* 1/ln2 */
    int k = (int)kd;
    double r = (t - kd * OR_LN2_HI) - kd * OR_LN2_LO;
    double p = 0x1.6124613a86d09p-33;       /* 1/13! */
    p = p * r + 0x1.1eed8eff8d898p-29;      /* 1/12! */
    p = p * r + 0x1.ae64567f544e4p-26;      /* 1/11! */
    p = p * r + 0x1.27e4fb7789f5cp-22;      /* 1/10! */
    p = p * r + 0x1.71de3a556c734p-19;      /* 1/9! */
    p = p * r + 0x1.a01a01a01a01ap-16;      /* 1/8! */
    p = p * r + 0x1.a01a01a01a01ap-13;      /* 1/7! */
    p = p * r + 0x1.6c16c16c16c17p-10;      /* 1/6! */
    p = p * r + 0x1.1111111111111p-7;       /* 1/5! */
    p = p * r + 0x1.5555555555555p-5;       /* 1/4! */
    p = p * r + 0x1.5555555555555p-3;       /* 1/3! */
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    if (k >= -1022 && k <= 1023) return p * or_pow2i(k);
    if (k > 1023) return (p * or_pow2i(1023)) * or_pow2i(k - 1023);
    return (p * or_pow2i(k + 200)) * or_pow2i(-200);
}

/* x^y for x > 0, finite y: exp(y log x) with the two functions above */
double or_det_pow(double x, double y) { return or_det_exp(y * or_det_log(x)); }

/* P:264-265 "weights ... following a power law with exponent beta>2"; R4 fixes the Pareto
 * law P(w >= x) = x^(1-beta), w_min = 1, by inverse transform w = (1-U)^(-1/(beta-1)).
 * U comes from Philox counter (v, 0, 0, 1), words (o0, o1). */
double or_weight_of_uniform(double U, double beta)
{
    return pow(1.0 - U, -1.0 / (beta - 1.0));
}

int or_weights(uint64_t n, double beta, uint64_t seed, double *w)
{
    if (n == 0 || n >= (1ull << 32) || !(beta > 2.0) || !isfinite(beta) || !w) return OR_EINVAL;
    for (uint64_t v = 0; v < n; v++) {
        uint32_t ctr[4] = {(uint32_t)v, 0u, 0u, 1u}, o[4];
        or_philox4x32_10(ctr, seed, o);
        w[v] = or_weight_of_uniform(or_u53(o[0], o[1]), beta);
    }
    return OR_OK;
}

/* P:269-270 "x_v ... drawn uniformly and independently at random" on T^d.
 * Coordinate 2k of vertex v uses Philox counter (v, k, 0, 2) words (o0,o1); 2k+1 uses (o2,o3).
 * Layout: structure of arrays, x[k*n + v]. */
int or_positions(uint64_t n, int d, uint64_t seed, double *x)
{
    if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5 || !x) return OR_EINVAL;
    for (uint64_t v = 0; v < n; v++) {
        for (int k = 0; 2 * k < d; k++) {
            uint32_t ctr[4] = {(uint32_t)v, (uint32_t)k, 0u, 2u}, o[4];
            or_philox4x32_10(ctr, seed, o);
            x[(uint64_t)(2 * k) * n + v] = or_u53(o[0], o[1]);
            if (2 * k + 1 < d) x[(uint64_t)(2 * k + 1) * n + v] = or_u53(o[2], o[3]);
        }
    }
    return OR_OK;
}

/* P:265-266 "Let W be their sum".  R3: W is the exactly rounded (round-to-nearest-even)
 * value of the real sum, so that it does not depend on a summation order.  Written as a
 * Kulisch accumulator: every finite double is an integer multiple of 2^-1074. */
#define OR_ACC_WORDS 72 /* 2304 bits >= 1074 + 1024 + 64 carry bits */
double or_exact_sum(const double *w, uint64_t n)
{
    uint32_t acc[OR_ACC_WORDS];
    memset(acc, 0, sizeof(acc));
    for (uint64_t v = 0; v < n; v++) {
        uint64_t bits;
        memcpy(&bits, &w[v], 8);
        uint64_t E = (bits >> 52) & 0x7ffu, frac = bits & ((1ull << 52) - 1);
        uint64_t m = E ? (frac | (1ull << 52)) : frac; /* value = m * 2^(pos - 1074) */
        uint64_t pos = E ? E - 1 : 0;
        /* add m << pos into acc (m < 2^53 spans at most 3 words) */
        uint64_t word = pos / 32, sh = pos % 32;
        uint64_t carry = 0;
        unsigned __int128 wide = (unsigned __int128)m << sh; /* < 2^85 */
        uint64_t part[3];
        part[0] = (uint64_t)(wide & 0xffffffffu);
        part[1] = (uint64_t)((wide >> 32) & 0xffffffffu);
        part[2] = (uint64_t)(wide >> 64);
        for (uint64_t k = word; k < OR_ACC_WORDS; k++) {
            uint64_t add = (k - word < 3) ? part[k - word] : 0;
            uint64_t s = (uint64_t)acc[k] + add + carry;
            acc[k] = (uint32_t)s;
            carry = s >> 32;
            if (k - word >= 2 && carry == 0) break;
        }
    }
    /* round to nearest even: find the top set bit t; value = acc * 2^-1074 */
    int t = -1;
    for (int k = OR_ACC_WORDS - 1; k >= 0 && t < 0; k--)
        if (acc[k]) {
            for (int b = 31; b >= 0; b--)
                if ((acc[k] >> b) & 1u) { t = 32 * k + b; break; }
        }
    if (t < 0) return 0.0;
#define OR_BIT(i) ((i) < 0 ? 0u : ((acc[(i) / 32] >> ((i) % 32)) & 1u))
    uint64_t mant = 0;
    int lo = t - 52 < 0 ? 0 : t - 52;
    for (int b = t; b >= lo; b--) mant = (mant << 1) | OR_BIT(b);
    if (t <= 52) return ldexp((double)mant, -1074);
    int rnd = (int)OR_BIT(t - 53);
    int sticky = 0;
    for (int b = t - 54; b >= 0 && !sticky; b--) sticky = (int)OR_BIT(b);
#undef OR_BIT
    if (rnd && (sticky || (mant & 1u))) {
        mant++;
        if (mant == (1ull << 53)) { mant >>= 1; t++; }
    }
    return ldexp((double)mant, t - 52 - 1074);
}

/* ||x-y|| = max_i min(|x_i-y_i|, 1-|x_i-y_i|) (L-infinity on the torus).
 * xu, xv point at coordinate 0 with the stride handled by the caller (contiguous d values). */
double or_torus_dist(const double *xu, const double *xv, int d)
{
    double dist = 0.0;
    for (int k = 0; k < d; k++) {
        double a = fabs(xu[k] - xv[k]);
        double t = a < 1.0 - a ? a : 1.0 - a;
        if (t > dist) dist = t;
    }
    return dist;
}

/* ||x_u - x_v||^d evaluated left to right: dist, dist*dist, (dist*dist)*dist, ... */
double or_dpow(double dist, int d)
{
    double D = dist;
    for (int k = 1; k < d; k++) D = D * dist;
    return D;
}

/* Eq. 1 in the kappa form of R1: p = min(1, (q/D)^(1/T)), q = (w_u*w_v)*s, s = kappa/W.
 * D = 0 gives ratio = +inf, p = 1 (R15). */
double or_prob(double wu, double wv, double s, double D, double T)
{
    double q = (wu * wv) * s;
    double ratio = q / D;
    if (ratio >= 1.0) return 1.0;
    return or_det_pow(ratio, 1.0 / T); /* R26 */
}

/* threshold model P:282-286 in the kappa form of R1: edge iff ||x_u-x_v||^d <= q (inclusive). */
int or_thresh_edge(double wu, double wv, double s, double D)
{
    double q = (wu * wv) * s;
    return D <= q;
}

/* ===================================================================================== */
/* Morton codes, Sec. 4.4 and Sec. 5.2: bitwise interleave, the   */
/* first coordinate most significant in each d-bit group ("a_3 b_3 a_2 b_2 ...").         */
/* ===================================================================================== */
uint32_t or_morton_encode(const uint32_t *coord, int d, int level)
{
    uint64_t code = 0;
    for (int b = level - 1; b >= 0; b--)
        for (int k = 0; k < d; k++) code = (code << 1) | ((coord[k] >> b) & 1u);
    return (uint32_t)code;
}

void or_morton_decode(uint32_t code, int d, int level, uint32_t *coord)
{
    for (int k = 0; k < d; k++) coord[k] = 0;
    for (int b = 0; b < level; b++)
        for (int k = 0; k < d; k++) {
            int bit = b * d + (d - 1 - k);
            coord[k] |= ((code >> bit) & 1u) << b;
        }
}

/* Lemma 1 proof P:994-996: "coordinates of the cell containing a given vertex is obtained
 * ... by rounding": c_k = floor(x_k * 2^level) (exact: scaling by a power of two). */
uint32_t or_cell_of_point(const double *x, int d, int level)
{
    uint32_t c[5];
    for (int k = 0; k < d; k++) c[k] = (uint32_t)floor(ldexp(x[k], level));
    return or_morton_encode(c, d, level);
}

/* per-dimension torus gap in cells */
static uint32_t or_gap(uint32_t a, uint32_t b, int level)
{
    uint32_t side = 1u << level;
    uint32_t g = a > b ? a - b : b - a;
    return g < side - g ? g : side - g;
}

/* Fig. 2a caption P:422-424: neighbouring cells (a cell is its own neighbour), on the torus.
 * R8: at levels 0 and 1 every pair is a neighbour pair. */
int or_are_neighbors(uint32_t A, uint32_t B, int d, int level)
{
    return or_delta_max(A, B, d, level) <= 1;
}

int or_delta_max(uint32_t A, uint32_t B, int d, int level)
{
    if (level == 0) return 0;
    uint32_t ca[5], cb[5];
    or_morton_decode(A, d, level, ca);
    or_morton_decode(B, d, level, cb);
    uint32_t m = 0;
    for (int k = 0; k < d; k++) {
        uint32_t g = or_gap(ca[k], cb[k], level);
        if (g > m) m = g;
    }
    return (int)m;
}

/* ===================================================================================== */
/* Weight buckets and levels, Sec. 4.1                                        */
/* ===================================================================================== */
/* Buckets ("layers") are factor-2 weight ranges.  R5: layer of v is
 * ilogb(w_v) - e_min; the bucket bound is wbar_i = 2^(e_min+i+1) (exclusive).
 * CL(i,j): deepest level whose cells are larger than the connection threshold of
 * the bucket bounds; R6: max{l in [0, Lmax] : 2^(-d l) >= qbar_ij}, qbar_ij = (wbar_i wbar_j) s.
 * I(i): deepest CL(i,.) over nonempty partners.  R7: Lmax = min(Ln+1, floor(32/d))
 * with Ln the smallest L such that 2^(dL) >= n. */
static int or_levels_s(const double *w, uint64_t n, int d, double kappa, double s_override, or_levels_t *lv);
int or_levels(const double *w, uint64_t n, int d, double kappa, or_levels_t *lv)
{
    return or_levels_s(w, n, d, kappa, 0.0, lv);
}

/* s_override > 0 replaces s = kappa/W (the HRG's dominating GIRG fixes s itself, R25) */
static int or_levels_s(const double *w, uint64_t n, int d, double kappa, double s_override, or_levels_t *lv)
{
    memset(lv, 0, sizeof(*lv));
    int emin = INT_MAX, emax = INT_MIN;
    for (uint64_t v = 0; v < n; v++) {
        if (!(w[v] > 0.0) || !isfinite(w[v])) return OR_EINVAL;
        int e = ilogb(w[v]);
        if (e < emin) emin = e;
        if (e > emax) emax = e;
    }
    if (emin < -500 || emax > 500) return OR_ERANGE;
    if (emax - emin + 1 > 64) return OR_ERANGE;
    lv->e_min = emin;
    lv->L = emax - emin + 1;
    for (uint64_t v = 0; v < n; v++) lv->cnt[ilogb(w[v]) - emin]++;
    lv->W = or_exact_sum(w, n);
    lv->s = s_override > 0.0 ? s_override : kappa / lv->W;
    int Ln = 0;
    while (ldexp(1.0, d * Ln) < (double)n) Ln++;
    lv->Lmax = Ln + 1 < 32 / d ? Ln + 1 : 32 / d;
    lv->maxCL = 0;
    for (int i = 0; i < lv->L; i++) {
        lv->I[i] = 0;
        for (int j = 0; j < lv->L; j++) {
            double qbar = ldexp(1.0, 2 * emin + i + j + 2) * lv->s;
            int cl = 0;
            for (int l = lv->Lmax; l >= 0; l--)
                if (ldexp(1.0, -d * l) >= qbar) { cl = l; break; }
            lv->CL[i][j] = cl;
        }
    }
    for (int i = 0; i < lv->L; i++) {
        if (!lv->cnt[i]) continue;
        for (int j = 0; j < lv->L; j++) {
            if (!lv->cnt[j]) continue;
            if (lv->CL[i][j] > lv->I[i]) lv->I[i] = lv->CL[i][j];
            if (lv->CL[i][j] > lv->maxCL) lv->maxCL = lv->CL[i][j];
        }
    }
    return OR_OK;
}

/* ===================================================================================== */
/* Edge sampler                                                                           */
/* ===================================================================================== */
typedef struct {
    const double *w, *x;
    uint64_t n;
    int d;
    double T, invT, s;
    uint64_t seed;
    or_levels_t lv;
    /* Lemma 1 index: order[] = vertex ids sorted by (layer, Morton code at I(layer), id);
     * layer i occupies order[lstart[i] .. lstart[i+1]); P[i][C] = number of layer-i vertices
     * in cells before C at level I(i). */
    uint32_t *order;
    uint32_t *codeI; /* Morton code at I(layer) of each sorted point (order[] positions) */
    uint64_t *mpre, *mb0; /* R22 scratch: 6^d + 1 entries each */
    uint64_t lstart[65];
    uint32_t *P[64];
    /* type-II tables per (i, j, level, class) */
    double *pbar, *Lbar;
    int *clog2;
    double *pbarR, *LbarR; /* R27: per (i, j, level, class h = 2, 3, 4) */
    /* per-level bucket-pair lists: eq[l] = pairs with CL == l, ge[l] = CL >= l */
    int neq[33], nge[33];
    int eq[33][64 * 65 / 2][2];
    int ge[33][64 * 65 / 2][2];
    /* shard filter: block range [blo, bhi) at level sl, or (nranks > 0) interleaved ranks */
    int sl;
    uint64_t blo, bhi;
    uint32_t nranks, rank;
    /* type-II scheme: OR_SCHEME_EVENT (one jump sequence per distant cell pair, Alg. 1 as
     * written) or OR_SCHEME_MERGED (one sequence per (A cell, bound class), R22) */
    int scheme;
    /* output */
    uint32_t *edges;
    uint64_t cap, m;
    or_stats_t *st;
    int err;
    /* test hook: coverage mode counts every candidate pair of every event (no sampling) */
    uint32_t *cover;
} or_ctx;

#define TAB(c, i, j, l, k) ((((size_t)(i) * 64 + (j)) * 32 + (l)) * 2 + (k))
#define TAB3(c, i, j, l, k) ((((size_t)(i) * 64 + (j)) * 32 + (l)) * 3 + (k))

static void emit(or_ctx *c, uint32_t u, uint32_t v)
{
    uint32_t a = u < v ? u : v, b = u < v ? v : u;
    if (c->m < c->cap) {
        c->edges[2 * c->m] = a;
        c->edges[2 * c->m + 1] = b;
    }
    c->m++;
}

/* Lemma 1: V_i^A = order range [P_{C_1}, P_{C_{j+1}}) with C_1.. the level-I(i)
 * descendants of A.  Returns offsets relative to the layer start. */
static void vrange(const or_ctx *c, int i, uint32_t A, int l, uint64_t *lo, uint64_t *hi)
{
    int sh = c->d * (c->lv.I[i] - l);
    uint64_t a0 = (uint64_t)A << sh, a1 = ((uint64_t)A + 1) << sh;
    *lo = c->P[i][a0];
    *hi = c->P[i][a1];
}

static const double *xcoord(const or_ctx *c, uint32_t v, double *buf)
{
    for (int k = 0; k < c->d; k++) buf[k] = c->x[(uint64_t)k * c->n + v];
    return buf;
}

/* Alg. 1 line 3: emit each (u,v) in V_i^A x V_j^B with probability p_uv.
 * App. B.1: for (i,i) and (A,A) only u<v.  T>0: r keyed by the vertex pair
 * (counter (u, v, 0, 3), u<v ids, words (o0,o1)), R17. */
static void type1(or_ctx *c, int l, uint32_t A, uint32_t B, int i, int j)
{
    uint64_t a0, a1, b0, b1;
    vrange(c, i, A, l, &a0, &a1);
    vrange(c, j, B, l, &b0, &b1);
    c->st->ev1++;
    if (a1 == a0 || b1 == b0) return;
    c->st->ev1_nonempty++;
    int same = (i == j && A == B);
    const uint32_t *Va = c->order + c->lstart[i], *Vb = c->order + c->lstart[j];
    double xu[5], xv[5];
    if (c->cover) {
        for (uint64_t s = a0; s < a1; s++)
            for (uint64_t t = same ? s + 1 : b0; t < b1; t++) {
                c->cover[(uint64_t)Va[s] * c->n + Vb[t]]++;
                c->st->cand1++;
            }
        return;
    }
    for (uint64_t s = a0; s < a1; s++) {
        uint32_t u = Va[s];
        xcoord(c, u, xu);
        for (uint64_t t = same ? s + 1 : b0; t < b1; t++) {
            uint32_t v = Vb[t];
            xcoord(c, v, xv);
            c->st->cand1++;
            double D = or_dpow(or_torus_dist(xu, xv, c->d), c->d);
            int edge;
            if (c->T == 0.0) {
                edge = or_thresh_edge(c->w[u], c->w[v], c->s, D);
            } else {
                double p = or_prob(c->w[u], c->w[v], c->s, D, c->T);
                if (p >= 1.0) {
                    edge = 1;
                } else {
                    uint32_t ctr[4] = {u < v ? u : v, u < v ? v : u, 0u, 3u}, o[4];
                    or_philox4x32_10(ctr, c->seed, o);
                    double r = or_u53(o[0], o[1]);
                    if (or_tie_mode & 1) r = p + or_tie_delta;
                    c->st->rnd1++;
                    if (fabs(r - p) < 1e-12) c->st->nt1++;
                    edge = r < p;
                }
            }
            if (edge) { c->st->acc1++; emit(c, u, v); }
        }
    }
}

/* Alg. 1 lines 5-6, Sec. 4.2: candidates of V_i^A x V_j^B (row-major,
 * R10) are visited by geometric jumps with the cell-pair bound pbar and accepted with
 * probability p_uv/pbar (R14: r_acc*pbar < p_uv).  Chunking (R10): the candidate index range
 * is cut into chunks of C = 2^clog2 candidates, each an independent jump chain (exact by
 * memorylessness), at most 2^15 chunks per event.  Draw k of chunk ch uses Philox counter
 * (A, B, l | i<<5 | j<<11 | ch<<17, k): r_jump = (o0,o1), r_acc = (o2,o3). */
static void type2(or_ctx *c, int l, uint32_t A, uint32_t B, int i, int j)
{
    uint64_t a0, a1, b0, b1;
    vrange(c, i, A, l, &a0, &a1);
    vrange(c, j, B, l, &b0, &b1);
    c->st->ev2++;
    uint64_t nA = a1 - a0, nB = b1 - b0;
    uint64_t N = nA * nB;
    if (N == 0) return;
    c->st->ev2_nonempty++;
    c->st->cand2 += N;
    int cls = or_delta_max(A, B, c->d, l) - 2; /* mind = (delta_max - 1) 2^-l, R9 */
    size_t ti = TAB(c, i, j, l, cls);
    double pbar = c->pbar[ti], Lbar = c->Lbar[ti];
    if (c->cover) { /* every candidate once; and the bound must hold for each */
        const uint32_t *Va = c->order + c->lstart[i], *Vb = c->order + c->lstart[j];
        double xu[5], xv[5];
        for (uint64_t s = a0; s < a1; s++)
            for (uint64_t t = b0; t < b1; t++) {
                c->cover[(uint64_t)Va[s] * c->n + Vb[t]]++;
                double D = or_dpow(or_torus_dist(xcoord(c, Va[s], xu), xcoord(c, Vb[t], xv), c->d), c->d);
                if (or_prob(c->w[Va[s]], c->w[Vb[t]], c->s, D, c->T) > pbar) c->st->bound_viol++;
            }
        return;
    }
    if (pbar == 0.0) return;
    /* R10: chunk length C = 2^clog2 (2..4 expected landings per chunk), doubled until the
     * event has at most 2^15 chunks (the chunk index has 15 counter bits) */
    int cl2 = c->clog2[ti];
    while (((N - 1) >> cl2) >= (1ull << 15)) cl2++;
    uint64_t C = 1ull << cl2;
    uint64_t nch = (N - 1) / C + 1;
    const uint32_t *Va = c->order + c->lstart[i], *Vb = c->order + c->lstart[j];
    double xu[5], xv[5];
    for (uint64_t ch = 0; ch < nch; ch++) {
        c->st->chunks++;
        uint64_t start = ch * C, end = start + C < N ? start + C : N;
        int64_t pos = (int64_t)start - 1;
        for (uint32_t k = 0;; k++) {
            uint32_t ctr[4] = {A, B, (uint32_t)l | ((uint32_t)i << 5) | ((uint32_t)j << 11) |
                                     ((uint32_t)ch << 17), k};
            uint32_t o[4];
            or_philox4x32_10(ctr, c->seed, o);
            c->st->draws++;
            double rj = or_u53(o[0], o[1]), ra = or_u53(o[2], o[3]);
            double z = pbar == 1.0 ? 0.0 : or_det_log(1.0 - rj) / Lbar; /* R26 */
            int64_t remaining = (int64_t)end - pos - 1;
            /* jump near-tie (R21): floor(z) is an integer decided in double.  glibc's and CUDA's
             * log are each within 1 ulp of log(1-rj), the division is correctly rounded, so the
             * two z differ by < 3 ulp < 7e-16 |z|; only a z within 1e-15 |z| of an integer, and
             * small enough to matter (z < remaining + 1), is counted. */
            if ((or_tie_mode & 4) && pbar < 1.0) {
                double az0 = fabs(z);
                z = nearbyint(z) + or_tie_delta * (az0 > 1.0 ? az0 : 1.0);
            }
            if (z < (double)remaining + 1.0 && pbar < 1.0) {
                c->st->jchk++;
                double az = fabs(z);
                if (fabs(z - nearbyint(z)) < 1e-15 * (az > 1.0 ? az : 1.0)) c->st->nt2jump++;
            }
            if (z >= (double)remaining) break;
            pos += 1 + (int64_t)z;
            c->st->landings++;
            uint64_t sidx = (uint64_t)pos / nB, tidx = (uint64_t)pos % nB;
            uint32_t u = Va[a0 + sidx], v = Vb[b0 + tidx];
            double D = or_dpow(or_torus_dist(xcoord(c, u, xu), xcoord(c, v, xv), c->d), c->d);
            double p = or_prob(c->w[u], c->w[v], c->s, D, c->T);
            /* acceptance near-tie: the uniform r_acc within 1e-12 of its threshold p_uv/pbar */
            if (or_tie_mode & 2) ra = p / pbar + or_tie_delta;
            if (fabs(ra * pbar - p) < 1e-12 * pbar) c->st->nt2acc++;
            if (ra * pbar < p) { c->st->acc2++; emit(c, u, v); }
        }
    }
}

/* ---- R22: merged type-II sequences ----
 * Alg. 1 samples every distant cell pair (A,B) of a bucket pair (i,j) on level l with its own
 * geometric-jump sequence under the bound pbar(i,j,l,delta_max).  All distant
 * pairs that share A and the bound class delta_max = k have the SAME pbar, so their candidate
 * sets can be concatenated and jumped over as one sequence: each candidate is still landed on
 * independently with probability pbar (memorylessness of the geometric skips), so
 * the edge distribution is unchanged, while the per-pair terminating draws disappear.
 *   D_k(A) = { B on level l : B and A not neighbours, parent(B) and parent(A) neighbours
 *             (the distant pairs of Alg. 1), delta_max(A,B) = k, and B > A if i = j
 *             (R16) }, in increasing Morton order.
 *   candidates: row-major over V_i^A x (V_j^B for B in D_k(A), concatenated in that order).
 *   chunks: C = 2^max(0, 1 - ilogb(pbar)) candidates (2..4 expected landings, as R10), doubled
 *   until the sequence has < 2^32 chunks.  Draw r of chunk ch: Philox counter
 *   (A, ch, l | i<<5 | j<<11 | (k-2)<<17 | 1<<18, r); r_jump = (o0,o1), r_acc = (o2,o3).
 * Everything else (jump, stop test, acceptance r_acc*pbar < p_uv, near-tie log) is type2's. */
static int cmp_u32(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : x > y;
}

/* D_2(A), D_3(A) without the i = j restriction: the children of the neighbours of parent(A) (on
 * the torus) that are not neighbours of A, split by delta_max, each list in increasing Morton
 * order (parents sorted by code, then their 2^d children in child-code order). */
static void distant_cells(const or_ctx *c, int l, uint32_t A, uint32_t *out2, int *n2, uint32_t *out3,
                          int *n3)
{
    int d = c->d, np = 0;
    uint32_t ac[5], pa[5], q[5], par[243];
    or_morton_decode(A, d, l, ac);
    for (int k = 0; k < d; k++) pa[k] = ac[k] >> 1;
    uint32_t side = 1u << l, sidep = 1u << (l - 1);
    int noff = 1;
    for (int k = 0; k < d; k++) noff *= 3;
    for (int o = 0; o < noff; o++) { /* parent neighbours, offsets in {-1,0,1}^d */
        int r = o;
        for (int k = 0; k < d; k++) {
            int off = r % 3 - 1;
            r /= 3;
            q[k] = (pa[k] + sidep + (uint32_t)off) % sidep;
        }
        uint32_t P = or_morton_encode(q, d, l - 1);
        int dup = 0; /* on levels <= 2 several offsets wrap onto the same parent */
        for (int t = 0; t < np; t++)
            if (par[t] == P) { dup = 1; break; }
        if (!dup) par[np++] = P;
    }
    qsort(par, (size_t)np, sizeof(uint32_t), cmp_u32);
    *n2 = 0;
    *n3 = 0;
    for (int t = 0; t < np; t++) {
        or_morton_decode(par[t], d, l - 1, q);
        for (uint32_t ch = 0; ch < (1u << d); ch++) {
            uint32_t dm = 0;
            for (int k = 0; k < d; k++) {
                uint32_t b = 2 * q[k] + ((ch >> (d - 1 - k)) & 1u);
                uint32_t g = b > ac[k] ? b - ac[k] : ac[k] - b;
                if (side - g < g) g = side - g; /* torus gap */
                if (g > dm) dm = g;
            }
            if (dm <= 1) continue; /* a neighbour of A (type-I or a deeper level) */
            uint32_t B = (par[t] << d) | ch;
            if (dm == 2) out2[(*n2)++] = B;
            else out3[(*n3)++] = B;
        }
    }
}

/* One merged geometric-jump sequence (R22 / R27): rows = sorted positions [a0, a1) of layer i,
 * columns = the concatenation of V_j^B over the cells Bs[0..nBs) (level l, in the given order),
 * every candidate landed on with probability pbar, chunks of 2^cl2 candidates keyed by
 * Philox counter (c0, chunk, tag, draw). */
static void type2_seq(or_ctx *c, int l, uint32_t c0, uint64_t a0, uint64_t a1, int j, uint32_t tag,
                      double pbar, double Lbar, const uint32_t *Bs, int nBs)
{
    uint64_t nA = a1 - a0;
    /* prefix of |V_j^B| over the concatenation (scratch owned by merged_all) */
    uint64_t *pre = c->mpre, *b0 = c->mb0;
    pre[0] = 0;
    for (int t = 0; t < nBs; t++) {
        uint64_t lo, hi;
        vrange(c, j, Bs[t], l, &lo, &hi);
        b0[t] = lo;
        pre[t + 1] = pre[t] + (hi - lo);
    }
    uint64_t M = pre[nBs], N = nA * M;
    if (N == 0) return;
    c->st->ev2_nonempty++;
    c->st->cand2 += N;
    int i = (int)((tag >> 5) & 63u);
    const uint32_t *Va = c->order + c->lstart[i], *Vb = c->order + c->lstart[j];
    double xu[5], xv[5];
    if (c->cover) { /* every candidate once; and the bound must hold for each */
        for (uint64_t s = a0; s < a1; s++)
            for (int t = 0; t < nBs; t++)
                for (uint64_t v = b0[t]; v < b0[t] + (pre[t + 1] - pre[t]); v++) {
                    uint32_t uu = Va[s], vv = Vb[v];
                    c->cover[(uint64_t)uu * c->n + vv]++;
                    double D = or_dpow(or_torus_dist(xcoord(c, uu, xu), xcoord(c, vv, xv), c->d), c->d);
                    if (or_prob(c->w[uu], c->w[vv], c->s, D, c->T) > pbar) c->st->bound_viol++;
                }
        return;
    }
    if (pbar == 0.0) return;
    int cl2 = 0;
    cl2 = 1 - ilogb(pbar);
    if (cl2 < 0) cl2 = 0;
    if (cl2 > 62) cl2 = 62;
    while (((N - 1) >> cl2) >= (1ull << 32)) cl2++;
    uint64_t C = 1ull << cl2;
    uint64_t nch = (N - 1) / C + 1;
    for (uint64_t ch = 0; ch < nch; ch++) {
        c->st->chunks++;
        uint64_t start = ch * C, end = start + C < N ? start + C : N;
        int64_t pos = (int64_t)start - 1;
        for (uint32_t r = 0;; r++) {
            uint32_t ctr[4] = {c0, (uint32_t)ch, tag, r}, o[4];
            or_philox4x32_10(ctr, c->seed, o);
            c->st->draws++;
            double rj = or_u53(o[0], o[1]), ra = or_u53(o[2], o[3]);
            double z = pbar == 1.0 ? 0.0 : or_det_log(1.0 - rj) / Lbar; /* R26 */
            int64_t remaining = (int64_t)end - pos - 1;
            if ((or_tie_mode & 4) && pbar < 1.0) {
                double az0 = fabs(z);
                z = nearbyint(z) + or_tie_delta * (az0 > 1.0 ? az0 : 1.0);
            }
            if (z < (double)remaining + 1.0 && pbar < 1.0) { /* jump near-tie, as in type2 */
                c->st->jchk++;
                double az = fabs(z);
                if (fabs(z - nearbyint(z)) < 1e-15 * (az > 1.0 ? az : 1.0)) c->st->nt2jump++;
            }
            if (z >= (double)remaining) break;
            pos += 1 + (int64_t)z;
            c->st->landings++;
            uint64_t sidx = (uint64_t)pos / M, tidx = (uint64_t)pos % M;
            int t = 0;
            while (pre[t + 1] <= tidx) t++; /* the B cell holding concatenated index tidx */
            uint32_t u = Va[a0 + sidx], v = Vb[b0[t] + (tidx - pre[t])];
            double D = or_dpow(or_torus_dist(xcoord(c, u, xu), xcoord(c, v, xv), c->d), c->d);
            double p = or_prob(c->w[u], c->w[v], c->s, D, c->T);
            if (or_tie_mode & 2) ra = p / pbar + or_tie_delta;
            if (fabs(ra * pbar - p) < 1e-12 * pbar) c->st->nt2acc++;
            if (ra * pbar < p) { c->st->acc2++; emit(c, u, v); }
        }
    }
}

/* R22: one sequence per (A cell, class delta_max = k) over V_i^A x (V_j^B, B in Bs) */
static void type2_merged(or_ctx *c, int l, uint32_t A, int i, int j, int k, const uint32_t *Bs, int nBs)
{
    uint64_t a0, a1;
    vrange(c, i, A, l, &a0, &a1);
    size_t ti = TAB(c, i, j, l, k - 2);
    uint32_t tag = (uint32_t)l | ((uint32_t)i << 5) | ((uint32_t)j << 11) | ((uint32_t)(k - 2) << 17) | (1u << 18);
    type2_seq(c, l, A, a0, a1, j, tag, c->pbar[ti], c->Lbar[ti], Bs, nBs);
}

/* R27 (refined bound): the rows of A are split by A's children a on level
 * l+1 (contiguous in the sorted index because l+1 <= I(i), Lemma 1), and the distant cells B of A
 * are classed by their box distance from a instead of from A: h = max over dimensions of the
 * torus gap between a (one level-(l+1) cell) and B (two level-(l+1) cells), in units of
 * 2^-(l+1); a pair (u in a, v in B) is at distance >= h 2^-(l+1) (P:486-491 with a tighter
 * mind).  Classes k = 0, 1, 2 for h = 2, 3, >= 4 (bound taken at h = 2, 3, 4).  Applied where
 * ref_level() says (R27). */
#define OR_REF_X 4096 /* R27: refine a level when layer i has >= 4096 points per level-l cell on average (R27) */
static int or_ref_x = 0;  /* TEST HOOK: 0 = OR_REF_X, k > 0 = k points, -1 = every level l < CL */
void or_set_ref_x(int x) { or_ref_x = x; }

static int ref_level(const or_ctx *c, int l, int i, int j)
{
    long x = or_ref_x == 0 ? OR_REF_X : or_ref_x;
    return c->scheme == OR_SCHEME_REFINED && (c->d == 2 || c->d == 3) && l < c->lv.CL[i][j] &&
           (x < 0 || (uint64_t)c->lv.cnt[i] >= ((uint64_t)x << (c->d * l)));
}

static uint32_t half_gap(uint32_t a2, uint32_t b, uint32_t S2) /* a2: level l+1, b: level l */
{
    uint32_t dd = (2u * b + S2 - a2) % S2; /* B = [dd, dd+2) relative to a = [0, 1) */
    if (dd == 0 || dd == S2 - 1) return 0;
    uint32_t r = dd - 1, lft = S2 - dd - 2;
    return r < lft ? r : lft;
}

static void type2_refined(or_ctx *c, int l, uint32_t A, int i, int j, const uint32_t *Bs, int nBs,
                          uint32_t *cls[3])
{
    int d = c->d;
    uint32_t S2 = 2u << l, bc[5], acd[5];
    for (uint32_t e = 0; e < (1u << d); e++) {
        uint32_t a = (A << d) | e; /* child of A on level l+1 <= I(i) */
        uint64_t a0, a1;
        vrange(c, i, a, l + 1, &a0, &a1);
        if (a1 == a0) continue;
        or_morton_decode(a, d, l + 1, acd);
        int nk[3] = {0, 0, 0};
        for (int t = 0; t < nBs; t++) {
            or_morton_decode(Bs[t], d, l, bc);
            uint32_t h = 0;
            for (int k = 0; k < d; k++) {
                uint32_t g = half_gap(acd[k], bc[k], S2);
                if (g > h) h = g;
            }
            int k = h <= 2 ? 0 : (h == 3 ? 1 : 2);
            cls[k][nk[k]++] = Bs[t];
        }
        for (int k = 0; k < 3; k++) {
            size_t ti = TAB3(c, i, j, l, k);
            uint32_t tag = (uint32_t)l | ((uint32_t)i << 5) | ((uint32_t)j << 11) | ((uint32_t)k << 17) | (1u << 19);
            type2_seq(c, l, a, a0, a1, j, tag, c->pbarR[ti], c->LbarR[ti], cls[k], nk[k]);
        }
    }
}

/* shard ownership of an event whose A cell is at level l */
static uint64_t blk_of(const or_ctx *c, int l, uint32_t A)
{
    if (l >= c->sl) return (uint64_t)A >> (c->d * (l - c->sl));
    return (uint64_t)A << (c->d * (c->sl - l));
}
/* Ownership of the events of A cell A on level l for layer pair (i, j).  Block-range mode: the
 * block of A (its first descendant's when l < sl) lies in [blo, bhi).  Interleaved mode
 * (nranks > 0, SURVEY 8(e) "Balance"): rank = block mod nranks for l >= sl; a coarse event
 * (l < sl) goes to rank (A + 7 j + 13 i + 31 l) mod nranks, so that the few large coarse events
 * spread over the ranks (unsigned 32-bit arithmetic). */
static int owns(const or_ctx *c, int l, uint32_t A, int i, int j)
{
    if (c->nranks == 0) {
        uint64_t b = blk_of(c, l, A);
        return b >= c->blo && b < c->bhi;
    }
    uint32_t key = l >= c->sl ? (uint32_t)((uint64_t)A >> (c->d * (l - c->sl)))
                              : A + 7u * (uint32_t)j + 13u * (uint32_t)i + 31u * (uint32_t)l;
    return key % c->nranks == c->rank;
}

static int subtree_may_own(const or_ctx *c, int l, uint32_t A)
{
    if (c->nranks > 0) /* interleaved: one block (and rank) per subtree from the split level on */
        return l < c->sl || (uint32_t)((uint64_t)A >> (c->d * (l - c->sl))) % c->nranks == c->rank;
    if (l >= c->sl) {
        uint64_t b = blk_of(c, l, A);
        return b >= c->blo && b < c->bhi;
    }
    uint64_t b0 = (uint64_t)A << (c->d * (c->sl - l)), b1 = ((uint64_t)A + 1) << (c->d * (c->sl - l));
    return b1 > c->blo && b0 < c->bhi;
}

/* Algorithm 1, with the loop swap of Sec. 4.3: a neighbouring cell
 * pair on level l is processed by bucket pairs with CL == l, a distant pair (whose parents
 * are neighbours) by bucket pairs with CL >= l.  Ordered cell pairs; bucket pairs i <= j, and
 * for i == j only A <= B (A < B for distant pairs): R16 (App. B.1). */
static void recur(or_ctx *c, int l, uint32_t A, uint32_t B)
{
    if (c->err) return;
    c->st->visits++;
    if (!subtree_may_own(c, l, A)) return;
    if (or_are_neighbors(A, B, c->d, l)) {
        for (int k = 0; k < c->neq[l]; k++) {
            int i = c->eq[l][k][0], j = c->eq[l][k][1];
            if (i == j && A > B) continue;
            if (!owns(c, l, A, i, j)) continue;
            type1(c, l, A, B, i, j);
        }
        if (l < c->lv.maxCL) { /* Alg. 1 line 7: refine neighbours until max depth */
            uint32_t nc = 1u << c->d;
            for (uint32_t x = 0; x < nc; x++)
                for (uint32_t y = 0; y < nc; y++)
                    recur(c, l + 1, (A << c->d) | x, (B << c->d) | y);
        }
    } else if (c->T > 0.0 && c->scheme == OR_SCHEME_EVENT) {
        for (int k = 0; k < c->nge[l]; k++) {
            int i = c->ge[l][k][0], j = c->ge[l][k][1];
            if (i == j && A >= B) continue;
            if (!owns(c, l, A, i, j)) continue;
            type2(c, l, A, B, i, j);
        }
    }
}

/* R22 driver: for every level l >= 2, bucket pair (i,j) with CL(i,j) >= l, and
 * nonempty A cell of bucket i on level l (visited in Morton order through the sorted index),
 * the two merged sequences of classes delta_max = 2, 3. */
static void merged_all(or_ctx *c)
{
    int d = c->d, noff = 1;
    for (int k = 0; k < d; k++) noff *= 6;
    uint32_t *l2 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)noff);
    uint32_t *l3 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)noff);
    uint32_t *all = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)noff);
    uint32_t *cls[3];
    for (int k = 0; k < 3; k++) cls[k] = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)noff);
    c->mpre = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(noff + 1));
    c->mb0 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(noff + 1));
    for (int l = 2; l <= c->lv.maxCL; l++)
        for (int i = 0; i < c->lv.L; i++) {
            int any = 0;
            for (int pr = 0; pr < c->nge[l]; pr++) any |= c->ge[l][pr][0] == i;
            if (!any) continue;
            int sh = d * (c->lv.I[i] - l);
            const uint32_t *code = c->codeI + c->lstart[i];
            uint64_t ni = c->lstart[i + 1] - c->lstart[i];
            for (uint64_t s = 0; s < ni; s++) {
                uint32_t A = code[s] >> sh;
                if (s > 0 && (code[s - 1] >> sh) == A) continue; /* first point of the cell */
                if (!subtree_may_own(c, l, A)) continue;
                int n2, n3;
                distant_cells(c, l, A, l2, &n2, l3, &n3);
                for (int pr = 0; pr < c->nge[l]; pr++) {
                    if (c->ge[l][pr][0] != i) continue;
                    int j = c->ge[l][pr][1];
                    if (!owns(c, l, A, i, j)) continue;
                    int s2 = 0, s3 = 0; /* i == j: only B > A (R16); the lists are sorted */
                    if (i == j) {
                        while (s2 < n2 && l2[s2] <= A) s2++;
                        while (s3 < n3 && l3[s3] <= A) s3++;
                    }
                    c->st->ev2 += (uint64_t)(n2 - s2 + n3 - s3);
                    if (ref_level(c, l, i, j)) { /* R27: both classes in one Morton-ordered list */
                        int na = 0, p2 = s2, p3 = s3;
                        while (p2 < n2 || p3 < n3)
                            all[na++] = (p3 >= n3 || (p2 < n2 && l2[p2] < l3[p3])) ? l2[p2++] : l3[p3++];
                        type2_refined(c, l, A, i, j, all, na, cls);
                        continue;
                    }
                    type2_merged(c, l, A, i, j, 2, l2 + s2, n2 - s2);
                    type2_merged(c, l, A, i, j, 3, l3 + s3, n3 - s3);
                }
            }
        }
    free(l2);
    free(l3);
    free(all);
    for (int k = 0; k < 3; k++) free(cls[k]);
    free(c->mpre);
    free(c->mb0);
}

/* test hook output of the Lemma-1 index */
typedef struct {
    uint32_t *order;  /* [n] */
    uint64_t *lstart; /* [65] */
    uint32_t *P;      /* concatenated per-layer prefix arrays, layer i at P + poff[i] */
    uint64_t *poff;   /* [65] */
    uint64_t pcap;
} or_index_out;

static uint64_t now_ns(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

static int or_run_s(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                    double s_override, uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi,
                    uint32_t nranks, uint32_t rank, int scheme, uint32_t *edges, uint64_t cap,
                    uint64_t *m_out, or_stats_t *st, uint32_t *cover, or_index_out *ix);
static int or_run(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                  uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi, uint32_t nranks,
                  uint32_t rank, int scheme, uint32_t *edges, uint64_t cap, uint64_t *m_out,
                  or_stats_t *st, uint32_t *cover, or_index_out *ix)
{
    return or_run_s(w, x, n, d, T, kappa, 0.0, seed, shard_level, blk_lo, blk_hi, nranks, rank, scheme,
                    edges, cap, m_out, st, cover, ix);
}

static int or_run_s(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                    double s_override, uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi,
                    uint32_t nranks, uint32_t rank, int scheme, uint32_t *edges, uint64_t cap,
                    uint64_t *m_out, or_stats_t *st, uint32_t *cover, or_index_out *ix)
{
    or_stats_t dummy;
    if (!st) st = &dummy;
    memset(st, 0, sizeof(*st));
    if (!w || !x || !m_out || (cap && !edges)) return OR_EINVAL;
    if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5) return OR_EINVAL;
    if (!(T >= 0.0 && T < 1.0)) return OR_EINVAL;
    if (!(kappa > 0.0) || !isfinite(kappa)) return OR_EINVAL;
    if (shard_level < 0 || shard_level * d > 32 || blk_lo >= blk_hi) return OR_EINVAL;
    if (nranks > 0 && rank >= nranks) return OR_EINVAL;
    if (scheme != OR_SCHEME_EVENT && scheme != OR_SCHEME_MERGED && scheme != OR_SCHEME_REFINED) return OR_EINVAL;
    for (uint64_t i = 0; i < (uint64_t)d * n; i++)
        if (!(x[i] >= 0.0 && x[i] < 1.0)) return OR_EINVAL;

    uint64_t t0 = now_ns();
    or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
    if (!c) return OR_ENOMEM;
    int rc = or_levels_s(w, n, d, kappa, s_override, &c->lv);
    if (rc) { free(c); return rc; }
    c->w = w; c->x = x; c->n = n; c->d = d; c->T = T; c->seed = seed;
    c->invT = T > 0.0 ? 1.0 / T : 0.0;
    c->s = c->lv.s;
    c->sl = shard_level; c->blo = blk_lo; c->bhi = blk_hi; c->scheme = scheme;
    c->nranks = nranks; c->rank = rank;
    c->edges = edges; c->cap = cap; c->st = st; c->cover = cover;
    const int L = c->lv.L;

    /* ---- Lemma 1 preprocessing (App. A): per bucket, bucket sort by
     * Morton code at I(i); visiting vertices in id order makes the sort stable, i.e. ties in
     * a cell are broken by vertex id (R11). ---- */
    c->order = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *cell = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint8_t *lay = (uint8_t *)malloc(n);
    if (!c->order || !cell || !lay) { rc = OR_ENOMEM; goto done; }
    c->lstart[0] = 0;
    for (int i = 0; i < L; i++) c->lstart[i + 1] = c->lstart[i] + c->lv.cnt[i];
    for (int i = 0; i < L; i++) {
        uint64_t ncell = 1ull << (d * c->lv.I[i]);
        c->P[i] = (uint32_t *)calloc(ncell + 1, sizeof(uint32_t));
        if (!c->P[i]) { rc = OR_ENOMEM; goto done; }
    }
    for (uint64_t v = 0; v < n; v++) {
        int i = ilogb(w[v]) - c->lv.e_min;
        double xv[5];
        lay[v] = (uint8_t)i;
        cell[v] = or_cell_of_point(xcoord(c, (uint32_t)v, xv), d, c->lv.I[i]);
        c->P[i][cell[v] + 1]++; /* counts, shifted by one */
    }
    for (int i = 0; i < L; i++) { /* prefix sums P_C */
        uint64_t ncell = 1ull << (d * c->lv.I[i]);
        for (uint64_t C = 0; C < ncell; C++) c->P[i][C + 1] += c->P[i][C];
    }
    {
        /* placement in id order (stable bucket sort) */
        uint32_t *cur[64];
        for (int i = 0; i < L; i++) {
            uint64_t ncell = 1ull << (d * c->lv.I[i]);
            cur[i] = (uint32_t *)malloc(sizeof(uint32_t) * (ncell + 1));
            if (!cur[i]) { rc = OR_ENOMEM; for (int k = 0; k < i; k++) free(cur[k]); goto done; }
            memcpy(cur[i], c->P[i], sizeof(uint32_t) * (ncell + 1));
        }
        for (uint64_t v = 0; v < n; v++) {
            int i = lay[v];
            c->order[c->lstart[i] + cur[i][cell[v]]++] = (uint32_t)v;
        }
        c->codeI = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
        if (!c->codeI) { rc = OR_ENOMEM; for (int i = 0; i < L; i++) free(cur[i]); goto done; }
        for (uint64_t s = 0; s < n; s++) c->codeI[s] = cell[c->order[s]];
        for (int i = 0; i < L; i++) free(cur[i]);
    }

    /* ---- bucket-pair lists per level (Sec. 4.3), nonempty layers, i <= j ---- */
    for (int l = 0; l <= 32; l++) { c->neq[l] = 0; c->nge[l] = 0; }
    for (int i = 0; i < L; i++)
        for (int j = i; j < L; j++) {
            if (!c->lv.cnt[i] || !c->lv.cnt[j]) continue;
            int cl = c->lv.CL[i][j];
            c->eq[cl][c->neq[cl]][0] = i; c->eq[cl][c->neq[cl]][1] = j; c->neq[cl]++;
            for (int l = 2; l <= cl; l++) {
                c->ge[l][c->nge[l]][0] = i; c->ge[l][c->nge[l]][1] = j; c->nge[l]++;
            }
        }

    /* ---- type-II bounds: pbar = min(1, (qbar / mind^d)^(1/T)) with mind =
     * (delta_max - 1) 2^-l (R9); Lbar = log1p(-pbar); chunk C = 2^max(0, 1 - ilogb(pbar))
     * (2..4 expected landings per chunk), capped at 2^62 (R10). ---- */
    if (T > 0.0) {
        size_t sz = (size_t)64 * 64 * 32 * 2;
        c->pbar = (double *)calloc(sz, sizeof(double));
        c->Lbar = (double *)calloc(sz, sizeof(double));
        c->clog2 = (int *)calloc(sz, sizeof(int));
        if (!c->pbar || !c->Lbar || !c->clog2) { rc = OR_ENOMEM; goto done; }
        for (int i = 0; i < L; i++)
            for (int j = 0; j < L; j++) {
                double qbar = ldexp(1.0, 2 * c->lv.e_min + i + j + 2) * c->s;
                for (int l = 2; l <= c->lv.CL[i][j]; l++)
                    for (int k = 0; k < 2; k++) {
                        double mind_d = ldexp(1.0, -d * l + d * k); /* ((k+1) 2^-l)^d */
                        double ratio = qbar / mind_d;
                        double pb = ratio >= 1.0 ? 1.0 : pow(ratio, c->invT);
                        size_t t = TAB(c, i, j, l, k);
                        c->pbar[t] = pb;
                        c->Lbar[t] = log1p(-pb);
                        int cl2 = 0;
                        if (pb > 0.0) {
                            cl2 = 1 - ilogb(pb);
                            if (cl2 < 0) cl2 = 0;
                            if (cl2 > 62) cl2 = 62;
                        }
                        c->clog2[t] = cl2;
                    }
            }
        /* R27: classes h = 2, 3, 4: mind = h 2^-(l+1), mind^d = h^d 2^(-d(l+1)) (exact) */
        size_t sz3 = (size_t)64 * 64 * 32 * 3;
        c->pbarR = (double *)calloc(sz3, sizeof(double));
        c->LbarR = (double *)calloc(sz3, sizeof(double));
        if (!c->pbarR || !c->LbarR) { rc = OR_ENOMEM; goto done; }
        for (int i = 0; i < L; i++)
            for (int j = 0; j < L; j++) {
                double qbar = ldexp(1.0, 2 * c->lv.e_min + i + j + 2) * c->s;
                for (int l = 2; l <= c->lv.CL[i][j]; l++)
                    for (int k = 0; k < 3; k++) {
                        double hd = 1.0;
                        for (int q = 0; q < d; q++) hd *= (double)(k + 2);
                        double mind_d = ldexp(hd, -d * (l + 1));
                        double ratio = qbar / mind_d;
                        double pb = ratio >= 1.0 ? 1.0 : pow(ratio, c->invT);
                        size_t t = TAB3(c, i, j, l, k);
                        c->pbarR[t] = pb;
                        c->LbarR[t] = log1p(-pb);
                    }
            }
    }

    if (ix) { /* test hook: export the index instead of sampling */
        memcpy(ix->order, c->order, sizeof(uint32_t) * n);
        memcpy(ix->lstart, c->lstart, sizeof(uint64_t) * 65);
        uint64_t off = 0;
        for (int i = 0; i < 64; i++) {
            ix->poff[i] = off;
            if (i < L) {
                uint64_t ncell = (1ull << (d * c->lv.I[i])) + 1;
                if (off + ncell > ix->pcap) { rc = OR_ECAPACITY; goto done; }
                memcpy(ix->P + off, c->P[i], sizeof(uint32_t) * ncell);
                off += ncell;
            }
        }
        ix->poff[64] = off;
        rc = OR_OK;
        goto done;
    }
    uint64_t t1 = now_ns();
    recur(c, 0, 0u, 0u);
    if (c->T > 0.0 && c->scheme != OR_SCHEME_EVENT) merged_all(c);
    st->ns_pre = t1 - t0;
    st->ns_edges = now_ns() - t1;
    rc = c->err;
    *m_out = c->m;
    if (!rc && c->m > cap) rc = OR_ECAPACITY;

done:
    free(c->order); free(c->codeI); free(cell); free(lay);
    for (int i = 0; i < 64; i++) free(c->P[i]);
    free(c->pbar); free(c->Lbar); free(c->clog2);
    free(c->pbarR); free(c->LbarR);
    free(c);
    return rc;
}

int or_edges(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
             uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi, int scheme,
             uint32_t *edges, uint64_t cap, uint64_t *m_out, or_stats_t *st)
{
    return or_run(w, x, n, d, T, kappa, seed, shard_level, blk_lo, blk_hi, 0, 0, scheme, edges, cap,
                  m_out, st, NULL, NULL);
}

int or_edges_ranked(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                    uint64_t seed, int shard_level, uint32_t nranks, uint32_t rank, int scheme,
                    uint32_t *edges, uint64_t cap, uint64_t *m_out, or_stats_t *st)
{
    if (nranks == 0) return OR_EINVAL;
    return or_run(w, x, n, d, T, kappa, seed, shard_level, 0, 1, nranks, rank, scheme, edges, cap,
                  m_out, st, NULL, NULL);
}

/* instrumented oracle (SURVEY 8(c) "Coverage"): cover[u*n+v] += 1 for every candidate pair
 * (u in V_i^A, v in V_j^B) of every type-I and type-II event; T > 0 so both types occur. */
int or_coverage(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                int scheme, uint32_t *cover, or_stats_t *st)
{
    uint64_t m = 0;
    if (!cover || n > 20000) return OR_EINVAL;
    memset(cover, 0, sizeof(uint32_t) * n * n);
    return or_run(w, x, n, d, T, kappa, 0, 0, 0, 1, 0, 0, scheme, NULL, 0, &m, st, cover, NULL);
}

int or_index(const double *w, const double *x, uint64_t n, int d, double kappa, uint32_t *order,
             uint64_t *lstart, uint32_t *P, uint64_t *poff, uint64_t pcap)
{
    uint64_t m = 0;
    or_index_out ix = {order, lstart, P, poff, pcap};
    return or_run(w, x, n, d, 0.0, kappa, 0, 0, 0, 1, 0, 0, OR_SCHEME_EVENT, NULL, 0, &m, NULL, NULL,
                  &ix);
}

/* Cell pairs enumerated by Algorithm 1 on a full tree of depth `depth`,
 * counted per level as unordered pairs: nb[l] = neighbouring pairs (A <= B), ds[l] = distant
 * pairs with neighbouring parents (A < B); ds2/ds3 split the distant pairs by delta_max. */
static void count_rec(int d, int depth, int l, uint32_t A, uint32_t B, uint64_t *nb, uint64_t *ds,
                      uint64_t *ds2, uint64_t *ds3)
{
    if (or_are_neighbors(A, B, d, l)) {
        if (A <= B) nb[l]++;
        if (l < depth) {
            uint32_t nc = 1u << d;
            for (uint32_t x = 0; x < nc; x++)
                for (uint32_t y = 0; y < nc; y++)
                    count_rec(d, depth, l + 1, (A << d) | x, (B << d) | y, nb, ds, ds2, ds3);
        }
    } else if (A < B) {
        ds[l]++;
        if (or_delta_max(A, B, d, l) == 2) ds2[l]++;
        else ds3[l]++;
    }
}

int or_count_pairs(int d, int depth, uint64_t *nb, uint64_t *ds, uint64_t *ds2, uint64_t *ds3)
{
    if (d < 1 || d > 5 || depth < 0 || depth * d > 24) return OR_EINVAL;
    for (int l = 0; l <= depth; l++) nb[l] = ds[l] = ds2[l] = ds3[l] = 0;
    count_rec(d, depth, 0, 0u, 0u, nb, ds, ds2, ds3);
    return OR_OK;
}

/* ===================================================================================== */
/* Hyperbolic random graphs (Sec. 3.2) on the GIRG machinery (Sec. 3.3           */
/* P:341-351), R25: the HRG is sampled as an exactly thinned DOMINATING GIRG.     */
/* ===================================================================================== */
/* R = 2 log(n) + C */
double or_hrg_R(uint64_t n, double C) { return 2.0 * log((double)n) + C; }

/* theta_v uniform in [0, 2 pi), r_v with density alpha sinh(alpha r)/(cosh(alpha R)-1)
 * on [0, R).  Inverse transform of F(r) = (cosh(alpha r) - 1)/(cosh(alpha R) - 1):
 * r = acosh(1 + U (cosh(alpha R) - 1)) / alpha.  Philox counter (v, 0, 0, 7): U = (o0, o1); the
 * angle is stored as the torus position x_v = theta_v / (2 pi) = (o2, o3). */
int or_hrg_points(uint64_t n, double alpha, double C, uint64_t seed, double *r, double *x)
{
    if (n < 2 || n >= (1ull << 32) || !(alpha > 0.5) || !isfinite(alpha) || !isfinite(C) || !r || !x)
        return OR_EINVAL;
    double R = or_hrg_R(n, C);
    if (!(R > 0.0)) return OR_EINVAL;
    double K = cosh(alpha * R) - 1.0;
    for (uint64_t v = 0; v < n; v++) {
        uint32_t ctr[4] = {(uint32_t)v, 0u, 0u, 7u}, o[4];
        or_philox4x32_10(ctr, seed, o);
        double U = or_u53(o[0], o[1]);
        r[v] = acosh(1.0 + U * K) / alpha;
        x[v] = or_u53(o[2], o[3]);
    }
    return OR_OK;
}

/* cosh d(p_u, p_v) = cosh r_u cosh r_v - sinh r_u sinh r_v cos(dtheta), dtheta the
 * angular distance in [0, pi] = 2 pi * (torus distance of x_u, x_v) */
double or_hrg_cosh_dist(double ru, double rv, double xu, double xv)
{
    double a = fabs(xu - xv);
    double t = a < 1.0 - a ? a : 1.0 - a;
    return cosh(ru) * cosh(rv) - sinh(ru) * sinh(rv) * cos(6.283185307179586 * t);
}

/* T = 0: edge iff d < R, i.e. cosh d < cosh R; T > 0: p_T(d) = 1/(exp((d-R)/(2T)) + 1) */
double or_hrg_prob(double cosh_d, double R, double T)
{
    if (T == 0.0) return cosh_d < cosh(R) ? 1.0 : 0.0;
    double d = acosh(cosh_d < 1.0 ? 1.0 : cosh_d);
    return 1.0 / (exp((d - R) / (2.0 * T)) + 1.0);
}

/* R25 dominating weight: w'_v = e^((R - r_v)/2) / sqrt(1 - e^(-2 r_v)) (the GIRG weight of P:345
 * divided by sqrt(2 sinh(r_v) e^(-r_v))), and e^(R/2) at r_v = 0 (then every GIRG' pair of v
 * saturates).  With s' = e^(-R/2)/sqrt(2) every HRG probability is at most the GIRG one:
 * cosh d >= 2 sinh r_u sinh r_v sin^2(pi dx) >= 2 e^(2R) dx^2 / (w'_u w'_v)^2, so e^(-d) <=
 * 1/cosh d gives p_T(d) <= e^((R-d)/(2T)) <= (w'_u w'_v s' / dx)^(1/T), and d < R gives
 * dx < w'_u w'_v s'. */
double or_hrg_dom_weight(double r, double R)
{
    if (r <= 0.0) return exp(0.5 * R);
    return exp(0.5 * (R - r)) / sqrt(-expm1(-2.0 * r));
}

double or_hrg_dom_s(double R) { return exp(-0.5 * R) / sqrt(2.0) * (1.0 + 0x1p-30); }

int or_hrg_dom_weights(const double *r, uint64_t n, double C, double *w)
{
    if (!r || !w || n < 2) return OR_EINVAL;
    double R = or_hrg_R(n, C);
    for (uint64_t v = 0; v < n; v++) w[v] = or_hrg_dom_weight(r[v], R);
    return OR_OK;
}

/* The HRG edge set: the dominating GIRG (w', x, d = 1, T, s') sampled by the GIRG sampler (merged
 * scheme, the same keyed randomness), then every GIRG edge kept with probability p_HRG / p_GIRG
 * (T > 0: uniform from Philox counter (u, v, 0, 6), u < v, words (o0, o1), kept iff r < ratio;
 * T = 0: kept iff cosh d < cosh R).  Each pair is an edge with probability
 * p_GIRG * p_HRG / p_GIRG = p_HRG, independently: the HRG distribution exactly.
 * Near-ties (north-star rule) of the thinning decision: |r - ratio| < 1e-12 (T > 0),
 * |cosh d - cosh R| < 1e-12 cosh R (T = 0); dominance violations (ratio > 1) counted. */
int or_hrg_edges(const double *r, const double *x, const double *w, uint64_t n, double C, double T,
                 uint64_t seed, uint32_t *edges, uint64_t cap, uint64_t *m_out, or_hrg_stats_t *hst)
{
    or_hrg_stats_t dummy;
    if (!hst) hst = &dummy;
    memset(hst, 0, sizeof(*hst));
    if (!r || !x || !w || !m_out || (cap && !edges) || n < 2) return OR_EINVAL;
    if (!(T >= 0.0 && T < 1.0)) return OR_EINVAL;
    double R = or_hrg_R(n, C), sd = or_hrg_dom_s(R), coshR = cosh(R);
    uint64_t scap = 16 * n + 1024, sm = 0;
    uint32_t *sup = NULL;
    int rc;
    for (;;) {
        sup = (uint32_t *)malloc(sizeof(uint32_t) * 2 * scap);
        if (!sup) return OR_ENOMEM;
        rc = or_run_s(w, x, n, 1, T, 1.0, sd, seed, 0, 0, 1, 0, 0, OR_SCHEME_MERGED, sup, scap, &sm, NULL,
                      NULL, NULL);
        if (rc != OR_ECAPACITY) break;
        free(sup);
        scap = sm + 1;
    }
    if (rc) { free(sup); return rc; }
    hst->super_edges = sm;
    uint64_t m = 0;
    for (uint64_t k = 0; k < sm; k++) {
        uint32_t u = sup[2 * k], v = sup[2 * k + 1];
        double cd = or_hrg_cosh_dist(r[u], r[v], x[u], x[v]);
        int keep;
        if (T == 0.0) {
            if (fabs(cd - coshR) < 1e-12 * coshR) hst->nt++;
            keep = cd < coshR;
        } else {
            double ph = or_hrg_prob(cd, R, T);
            double a = fabs(x[u] - x[v]);
            double D = a < 1.0 - a ? a : 1.0 - a; /* d = 1: D = dist */
            double pg = or_prob(w[u], w[v], sd, D, T);
            double ratio = ph / pg;
            if (ratio > 1.0) hst->violations++;
            uint32_t ctr[4] = {u < v ? u : v, u < v ? v : u, 0u, 6u}, o[4];
            or_philox4x32_10(ctr, seed, o);
            double rr = or_u53(o[0], o[1]);
            if (fabs(rr - ratio) < 1e-12) hst->nt++;
            keep = rr < ratio;
        }
        if (keep) {
            if (m < cap) { edges[2 * m] = u; edges[2 * m + 1] = v; }
            m++;
        }
    }
    free(sup);
    *m_out = m;
    return m > cap ? OR_ECAPACITY : OR_OK;
}

/* O(n^2) definitions: threshold HRG edge set (d < R), the expected edge count sum p_T(d), and
 * the largest p_HRG / p_GIRG' over all pairs (dominance, must be <= 1) */
int or_hrg_bruteforce_t0(const double *r, const double *x, uint64_t n, double C, uint32_t *edges, uint64_t cap,
                         uint64_t *m_out)
{
    double coshR = cosh(or_hrg_R(n, C));
    uint64_t m = 0;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t v = u + 1; v < n; v++)
            if (or_hrg_cosh_dist(r[u], r[v], x[u], x[v]) < coshR) {
                if (m < cap) { edges[2 * m] = (uint32_t)u; edges[2 * m + 1] = (uint32_t)v; }
                m++;
            }
    *m_out = m;
    return m > cap ? OR_ECAPACITY : OR_OK;
}

double or_hrg_expected_edges(const double *r, const double *x, uint64_t n, double C, double T)
{
    double R = or_hrg_R(n, C), acc = 0.0;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t v = u + 1; v < n; v++) acc += or_hrg_prob(or_hrg_cosh_dist(r[u], r[v], x[u], x[v]), R, T);
    return acc;
}

double or_hrg_max_ratio(const double *r, const double *x, const double *w, uint64_t n, double C, double T)
{
    double R = or_hrg_R(n, C), sd = or_hrg_dom_s(R), best = 0.0;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t v = u + 1; v < n; v++) {
            double a = fabs(x[u] - x[v]);
            double D = a < 1.0 - a ? a : 1.0 - a;
            double ph = or_hrg_prob(or_hrg_cosh_dist(r[u], r[v], x[u], x[v]), R, T);
            double pg = T == 0.0 ? (double)or_thresh_edge(w[u], w[v], sd, D) : or_prob(w[u], w[v], sd, D, T);
            double ratio = ph == 0.0 ? 0.0 : (pg == 0.0 ? INFINITY : ph / pg);
            if (ratio > best) best = ratio;
        }
    return best;
}

/* ===================================================================================== */
/* Brute force (the plain definition for T=0; the expected edge count for T>0)            */
/* ===================================================================================== */
int or_bruteforce_t0(const double *w, const double *x, uint64_t n, int d, double kappa,
                     uint32_t *edges, uint64_t cap, uint64_t *m_out)
{
    if (!w || !x || !m_out || n == 0 || d < 1 || d > 5) return OR_EINVAL;
    double s = kappa / or_exact_sum(w, n);
    uint64_t m = 0;
    double xu[5], xv[5];
    for (uint64_t u = 0; u < n; u++) {
        for (int k = 0; k < d; k++) xu[k] = x[(uint64_t)k * n + u];
        for (uint64_t v = u + 1; v < n; v++) {
            for (int k = 0; k < d; k++) xv[k] = x[(uint64_t)k * n + v];
            double D = or_dpow(or_torus_dist(xu, xv, d), d);
            if (or_thresh_edge(w[u], w[v], s, D)) {
                if (m < cap) { edges[2 * m] = (uint32_t)u; edges[2 * m + 1] = (uint32_t)v; }
                m++;
            }
        }
    }
    *m_out = m;
    return m > cap ? OR_ECAPACITY : OR_OK;
}

double or_expected_edges_bf(const double *w, const double *x, uint64_t n, int d, double T,
                            double kappa)
{
    double s = kappa / or_exact_sum(w, n);
    double acc = 0.0;
    double xu[5], xv[5];
    for (uint64_t u = 0; u < n; u++) {
        for (int k = 0; k < d; k++) xu[k] = x[(uint64_t)k * n + u];
        for (uint64_t v = u + 1; v < n; v++) {
            for (int k = 0; k < d; k++) xv[k] = x[(uint64_t)k * n + v];
            double D = or_dpow(or_torus_dist(xu, xv, d), d);
            acc += T == 0.0 ? (double)or_thresh_edge(w[u], w[v], s, D) : or_prob(w[u], w[v], s, D, T);
        }
    }
    return acc;
}

/* X ~ Geometric(p) = number of pairs skipped before the next selected pair.
 * R10: floor(log(1-u) / log1p(-p)); p = 1 gives 0. */
int64_t or_geometric_skip(double p, double u)
{
    if (p >= 1.0) return 0;
    return (int64_t)floor(log(1.0 - u) / log1p(-p));
}

/* ===================================================================================== */
/* Average-degree estimation, Sec. 5.1 and App. B.2             */
/* In kappa form (R1): y_uv = 2^d kappa w_u w_v / W is the short-edge probability (Eq. 2,  */
/* P:1092-1097); E[X_uv] = g(y) (Eq. 4) for y <= 1, and 1 for y > 1          */
/* (k >= 0.5).  T = 0: E[X_uv] = min(1, y).                                       */
/* ===================================================================================== */
double or_g(double y, double T)
{
    if (y > 1.0) return 1.0;
    if (T == 0.0) return y;
    return (y - T * pow(y, 1.0 / T)) / (1.0 - T);
}

/* the plain definition: (1/n) sum_{u != v} E[X_uv]  (Eq. 5 P:1126-1127 before simplification) */
double or_f_bruteforce(const double *w, uint64_t n, int d, double T, double kappa)
{
    double W = or_exact_sum(w, n);
    double a = ldexp(kappa, d) / W;
    double acc = 0.0;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t v = 0; v < n; v++)
            if (u != v) acc += or_g((a * w[u]) * w[v], T);
    return acc / (double)n;
}

static int cmp_desc(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? 1 : (x > y ? -1 : 0);
}

/* candidates R: vertices with at least one partner v with y_uv > 1; it suffices
 * to test against the largest weight.  Returned sorted by decreasing weight. */
static double *or_R(const double *w, uint64_t n, double a, uint64_t *nr)
{
    double wmax = 0.0;
    for (uint64_t v = 0; v < n; v++) if (w[v] > wmax) wmax = w[v];
    double *r = (double *)malloc(sizeof(double) * (n ? n : 1));
    uint64_t k = 0;
    for (uint64_t v = 0; v < n; v++)
        if ((a * w[v]) * wmax > 1.0) r[k++] = w[v];
    qsort(r, k, sizeof(double), cmp_desc);
    *nr = k;
    return r;
}

/* error term over E_R: sum over ordered pairs u != v with y_uv > 1 of
 * (formula(y_uv) - 1), formula = (y - T y^(1/T))/(1-T) (Eq. 4) -- O(|R|^2) reference */
double or_ER_quadratic(const double *w, uint64_t n, int d, double T, double kappa)
{
    double W = or_exact_sum(w, n);
    double a = ldexp(kappa, d) / W;
    uint64_t nr;
    double *r = or_R(w, n, a, &nr);
    double acc = 0.0;
    for (uint64_t u = 0; u < nr; u++)
        for (uint64_t v = 0; v < nr; v++) {
            if (u == v) continue;
            double y = (a * r[u]) * r[v];
            if (y > 1.0) {
                double f = T == 0.0 ? y : (y - T * pow(y, 1.0 / T)) / (1.0 - T);
                acc += f - 1.0;
            }
        }
    free(r);
    return acc;
}

/* the same sum in O(|R|): with R sorted by weight, the partners of u in E_R form
 * a prefix of the sorted order that grows with w_u; prefix sums of w and of (sqrt(a) w)^(1/T)
 * give each vertex's contribution in O(1). */
double or_ER_linear(const double *w, uint64_t n, int d, double T, double kappa)
{
    double W = or_exact_sum(w, n);
    double a = ldexp(kappa, d) / W;
    double ra = sqrt(a);
    uint64_t nr;
    double *r = or_R(w, n, a, &nr);
    double *S1 = (double *)malloc(sizeof(double) * (nr + 1));
    double *SP = (double *)malloc(sizeof(double) * (nr + 1));
    S1[0] = 0.0; SP[0] = 0.0;
    for (uint64_t k = 0; k < nr; k++) {
        S1[k + 1] = S1[k] + r[k];
        SP[k + 1] = SP[k] + (T == 0.0 ? 0.0 : pow(ra * r[k], 1.0 / T));
    }
    double acc = 0.0;
    uint64_t m = 0; /* prefix length; grows while u goes to larger weights */
    for (uint64_t t = nr; t-- > 0;) { /* increasing weight */
        double wu = r[t];
        while (m < nr && (a * wu) * r[m] > 1.0) m++;
        uint64_t cnt = m;
        double s1 = S1[m], sp = SP[m];
        double zu = T == 0.0 ? 0.0 : pow(ra * wu, 1.0 / T);
        if (t < m) { cnt -= 1; s1 -= wu; sp -= zu; } /* exclude v = u */
        double lin = a * wu * s1;
        double f = T == 0.0 ? lin : (lin - T * zu * sp) / (1.0 - T);
        acc += f - (double)cnt;
    }
    free(S1); free(SP); free(r);
    return acc;
}

/* f(kappa) = E[average degree] in kappa form.  Same decomposition as the paper
 * (short + long edges for pairs with y <= 1, Eq. 4; pairs in E_R count 1), but
 * summed over the non-E_R pairs directly instead of "all pairs minus E_R" (R12): the literal
 * form subtracts huge, nearly equal sums when heavy pairs saturate (double loses up to ~6 digits
 * at beta = 2.2, d = 3).  With R sorted by decreasing weight, the non-E_R partners of u in R
 * are the vertices outside R plus a suffix of R, so suffix sums give each
 * vertex's contribution in O(1):
 *   f = [ (a L - T P)/(1-T) + |E_R| ] / n,   a = 2^d kappa / W,
 *   L = sum_{(u,v) not in E_R, u != v} w_u w_v,  P = sum_{(u,v) not in E_R, u != v} z_u z_v,
 *   z_u = (sqrt(a) w_u)^(1/T)  (so z_u z_v = y_uv^(1/T)).     T = 0: f = (a L + |E_R|)/n. */
double or_f(const double *w, uint64_t n, int d, double T, double kappa)
{
    double W = or_exact_sum(w, n);
    double a = ldexp(kappa, d) / W;
    double ra = sqrt(a), invT = T > 0.0 ? 1.0 / T : 0.0;
    uint64_t nr;
    double *r = or_R(w, n, a, &nr);
    double wmax = nr ? r[0] : 0.0;
    /* vertices outside R: (a w_v) wmax <= 1 */
    double Wsmall = 0.0, Zsmall = 0.0;
    for (uint64_t v = 0; v < n; v++) {
        if ((a * w[v]) * wmax > 1.0) continue;
        Wsmall += w[v];
        if (T > 0.0) Zsmall += pow(ra * w[v], invT);
    }
    double *zc = (double *)malloc(sizeof(double) * (nr + 1));
    double *S1s = (double *)malloc(sizeof(double) * (nr + 1)); /* suffix sums over R */
    double *SPs = (double *)malloc(sizeof(double) * (nr + 1));
    for (uint64_t k = 0; k < nr; k++) zc[k] = T > 0.0 ? pow(ra * r[k], invT) : 0.0;
    S1s[nr] = 0.0; SPs[nr] = 0.0;
    for (uint64_t k = nr; k-- > 0;) { S1s[k] = S1s[k + 1] + r[k]; SPs[k] = SPs[k + 1] + zc[k]; }
    double ZR = SPs[0], Lsum = 0.0, Psum = 0.0, nER = 0.0;
    for (uint64_t v = 0; v < n; v++) { /* u outside R: every partner is a non-E_R pair */
        if ((a * w[v]) * wmax > 1.0) continue;
        Lsum += w[v] * (Wsmall + S1s[0] - w[v]);
        if (T > 0.0) {
            double z = pow(ra * w[v], invT);
            Psum += z * (Zsmall + ZR - z);
        }
    }
    uint64_t m = nr; /* E_R partners of the t-th heaviest: prefix [0, m), shrinking with t */
    for (uint64_t t = 0; t < nr; t++) {
        while (m > 0 && !((a * r[t]) * r[m - 1] > 1.0)) m--;
        int self_in_prefix = t < m;
        nER += (double)(m - (uint64_t)self_in_prefix);
        double sl = Wsmall + S1s[m] - (self_in_prefix ? 0.0 : r[t]);
        double sp = Zsmall + SPs[m] - (self_in_prefix ? 0.0 : zc[t]);
        Lsum += r[t] * sl;
        Psum += zc[t] * sp;
    }
    free(zc); free(S1s); free(SPs); free(r);
    double tot = T == 0.0 ? a * Lsum + nER : (a * Lsum - T * Psum) / (1.0 - T) + nER;
    return tot / (double)n;
}

/* exponential search, then bisection in log kappa, R12:
 * start kappa0 = avg_deg (1-T) / (2^d E[w]), E[w] = (beta-1)/(beta-2); stop when
 * hi/lo - 1 < 1e-13 or after 200 bisection steps; return (lo+hi)/2. */
int or_scale_weights(const double *w, uint64_t n, double avg_deg, int d, double T, double beta,
                     double *kappa_out)
{
    if (!w || !kappa_out || n < 2 || d < 1 || d > 5) return OR_EINVAL;
    if (!(T >= 0.0 && T < 1.0) || !(beta > 2.0)) return OR_EINVAL;
    if (!(avg_deg > 0.0 && avg_deg < (double)(n - 1))) return OR_EINVAL;
    double Ew = (beta - 1.0) / (beta - 2.0);
    double k0 = avg_deg * (1.0 - T) / (ldexp(1.0, d) * Ew);
    double lo, hi;
    double f0 = or_f(w, n, d, T, k0);
    if (!isfinite(f0)) return OR_ERANGE;
    int it = 0;
    if (f0 < avg_deg) {
        lo = k0; hi = 2.0 * k0;
        while (or_f(w, n, d, T, hi) < avg_deg) {
            lo = hi; hi *= 2.0;
            if (++it > 2000) return OR_ERANGE;
        }
    } else {
        hi = k0; lo = 0.5 * k0;
        while (or_f(w, n, d, T, lo) >= avg_deg) {
            hi = lo; lo *= 0.5;
            if (++it > 2000) return OR_ERANGE;
        }
    }
    for (it = 0; it < 200 && hi / lo - 1.0 >= 1e-13; it++) {
        double mid = sqrt(lo * hi);
        double fm = or_f(w, n, d, T, mid);
        if (!isfinite(fm)) return OR_ERANGE;
        if (fm < avg_deg) lo = mid;
        else hi = mid;
    }
    *kappa_out = 0.5 * (lo + hi);
    return OR_OK;
}
