/*
 * girg_oracle.h -- the CPU ORACLE for the GIRG hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (paper_1905_06706_b200/, include/girg.h) never links, imports or executes it,
 * and this oracle shares no code, header, table or constant generator with it.
 *
 * Plain, sequential, obviously-correct C99 (compiled -O2 -ffp-contract=off, glibc libm).
 * Citations: "P:NNN" = line NNN of /root/reference/PAPER.md (arXiv:1905.06706).
 * Every reading of an ambiguous passage is listed in DESIGN.md ("Readings", R1..R26).
 *
 * Parity status of every function is pinned by tests/test_oracle_*.py; see DESIGN.md
 * section "Oracle pins".  No function here is "parity unpinned".
 */
#ifndef GIRG_ORACLE_H
#define GIRG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numeric meaning as the C ABI, defined independently) */
#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ECAPACITY (-2)
#define OR_ERANGE (-3)
#define OR_ENOMEM (-4)

/* ---- randomness (R17: counter-based, keyed; replaces P:1281 thread-local RNG) ---- */
void or_philox4x32_10(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]);
double or_u53(uint32_t hi, uint32_t lo);

/* ---- R26: canonical log / exp / pow of the edge decisions (+ - * / and bit operations only) ---- */
double or_det_log(double x);
double or_det_exp(double t);
double or_det_pow(double x, double y);

/* ---- model, Sec. 2.1 P:258-290 ---- */
int or_weights(uint64_t n, double beta, uint64_t seed, double *w);          /* P:264-265, R4 */
double or_weight_of_uniform(double U, double beta); /* inverse transform (1-U)^(-1/(beta-1)) */
int or_positions(uint64_t n, int d, uint64_t seed, double *x /* [d][n] */);
double or_exact_sum(const double *w, uint64_t n);                         /* P:265-266, R3 */
double or_torus_dist(const double *xu, const double *xv, int d);
double or_dpow(double dist, int d);                                       /* ||.||^d, left to right */
/* scaled weight product q = (w_u*w_v)*s, s = kappa/W  (R1) */
double or_prob(double wu, double wv, double s, double D, double T);       /* Eq. 1, R1 */
int or_thresh_edge(double wu, double wv, double s, double D);             /* P:282-286, R1 */

/* ---- Morton / grid, Sec. 4.4, Sec. 5.2 P:663-669 ---- */
uint32_t or_morton_encode(const uint32_t *coord, int d, int level);
void or_morton_decode(uint32_t code, int d, int level, uint32_t *coord);
uint32_t or_cell_of_point(const double *x, int d, int level); /* x: d contiguous coords */
int or_are_neighbors(uint32_t A, uint32_t B, int d, int level); /* Fig. 2a, R8 */
int or_delta_max(uint32_t A, uint32_t B, int d, int level);     /* max_k torus cell gap */

/* ---- levels, Sec. 4.1 P:440-476 ---- */
typedef struct {
    int L;           /* number of layers = e_max - e_min + 1 */
    int e_min;       /* min ilogb(w) */
    int Lmax;        /* depth cap, R7 */
    int maxCL;       /* max CL over nonempty layer pairs */
    double W, s;     /* exact sum, s = kappa/W */
    uint64_t cnt[64];
    int CL[64][64];
    int I[64];
} or_levels_t;
int or_levels(const double *w, uint64_t n, int d, double kappa, or_levels_t *lv);

/* ---- work counters and near-tie log (north-star parity rule) ---- */
typedef struct {
    uint64_t visits;          /* cell pairs visited by the recursion */
    uint64_t ev1, ev1_nonempty, cand1, acc1; /* type-I events, nonempty, candidates, edges */
    uint64_t ev2, ev2_nonempty, chunks, draws, landings, acc2; /* type-II */
    uint64_t nt1, nt2acc, nt2jump; /* near-ties: type-I r~p, type-II r_acc~p/pbar, jump z~int */
    uint64_t cand2;                /* sum of |V_i^A||V_j^B| over type-II events */
    uint64_t ns_pre, ns_edges;     /* wall time: levels + index ("Pre"), recursion ("Edges") */
    uint64_t rnd1;                 /* type-I decisions that drew a uniform (p_uv < 1) */
    uint64_t jchk;                 /* jump near-tie checks (draws with z < remaining + 1) */
    uint64_t bound_viol;           /* coverage mode: merged / refined candidates with p_uv > pbar */
} or_stats_t;

/* TEST HOOK (O12 pin): move type-I uniforms (bit 1), type-II acceptance uniforms (bit 2) or
 * jump quotients (bit 4) to threshold + delta; 0 = off (the default) */
void or_set_tie_hook(int mode, double delta);

/* type-II schemes: EVENT = one jump sequence per distant cell pair (Alg. 1 lines 5-6 as
 * written, R10); MERGED = one sequence per (A cell, bound class), the distant pairs of A with
 * the same bound concatenated (R22, exact in distribution; the product default). */
#define OR_SCHEME_EVENT 0
#define OR_SCHEME_MERGED 1
/* REFINED = MERGED, except on the levels l < CL(i,j) where layer i has >= 4096 points per level-l
 * cell on average (d = 2, 3): there the rows of A are split by A's children on level l+1 and the
 * distant cells classed by their box distance from the child (R27) */
#define OR_SCHEME_REFINED 2
/* TEST HOOK (pins of R27 at small n): the REFINED scheme's points-per-cell threshold; 0 = the
 * default (8), k > 0 = k, -1 = every level l < CL(i,j).  The library's girg_options.ref_x has the
 * same meaning. */
void or_set_ref_x(int x);

/* Edge sampler: Algorithm 1 over the Lemma-1 index, double counting
 * per App. B.1 (R16), type-II by geometric jumps (R10 / R22).
 * Shard filter: only events whose A cell's block at shard_level lies in
 * [blk_lo, blk_hi) are processed; shard_level=0, [0,1) = everything.
 * edges: [cap][2] uint32 (u<v).  Returns OR_OK / OR_ECAPACITY (m_out = true m) / errors. */
int or_edges(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
             uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi, int scheme,
             uint32_t *edges, uint64_t cap, uint64_t *m_out, or_stats_t *st);

/* Interleaved shard ownership (SURVEY 8(e) "Balance"): events whose A cell is on a level
 * l >= shard_level belong to rank (Morton block at shard_level) mod nranks; coarser events to rank
 * (A + 7 j + 13 i + 31 l) mod nranks (32-bit unsigned).  The nranks shards partition the graph. */
int or_edges_ranked(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                    uint64_t seed, int shard_level, uint32_t nranks, uint32_t rank, int scheme,
                    uint32_t *edges, uint64_t cap, uint64_t *m_out, or_stats_t *st);

/* test hooks: instrumented coverage (cover: n*n counters), Lemma-1 index export, and the
 * per-level cell-pair counts of Algorithm 1 on a full tree */
int or_coverage(const double *w, const double *x, uint64_t n, int d, double T, double kappa,
                int scheme, uint32_t *cover, or_stats_t *st);
int or_index(const double *w, const double *x, uint64_t n, int d, double kappa, uint32_t *order,
             uint64_t *lstart, uint32_t *P, uint64_t *poff, uint64_t pcap);
int or_count_pairs(int d, int depth, uint64_t *nb, uint64_t *ds, uint64_t *ds2, uint64_t *ds3);

/* ---- hyperbolic random graphs, Sec. 3.2, through the dominating GIRG of Sec. 3.3
 * P:341-351 and exact thinning (R25) ---- */
typedef struct {
    uint64_t super_edges; /* edges of the dominating GIRG */
    uint64_t nt;          /* thinning near-ties (must be 0) */
    uint64_t violations;  /* pairs with p_HRG > p_GIRG' (must be 0) */
} or_hrg_stats_t;
double or_hrg_R(uint64_t n, double C);
int or_hrg_points(uint64_t n, double alpha, double C, uint64_t seed, double *r, double *x);
double or_hrg_cosh_dist(double ru, double rv, double xu, double xv);
double or_hrg_prob(double cosh_d, double R, double T);
double or_hrg_dom_weight(double r, double R);
double or_hrg_dom_s(double R);
int or_hrg_dom_weights(const double *r, uint64_t n, double C, double *w);
int or_hrg_edges(const double *r, const double *x, const double *w, uint64_t n, double C, double T,
                 uint64_t seed, uint32_t *edges, uint64_t cap, uint64_t *m_out, or_hrg_stats_t *hst);
int or_hrg_bruteforce_t0(const double *r, const double *x, uint64_t n, double C, uint32_t *edges,
                         uint64_t cap, uint64_t *m_out);
double or_hrg_expected_edges(const double *r, const double *x, uint64_t n, double C, double T);
double or_hrg_max_ratio(const double *r, const double *x, const double *w, uint64_t n, double C, double T);

/* O(n^2) brute force, threshold model (T=0), canonical arithmetic */
int or_bruteforce_t0(const double *w, const double *x, uint64_t n, int d, double kappa,
                     uint32_t *edges, uint64_t cap, uint64_t *m_out);
/* O(n^2) sum_{u<v} p_uv  (expected edge count given w, x) */
double or_expected_edges_bf(const double *w, const double *x, uint64_t n, int d, double T,
                            double kappa);

/* ---- average-degree estimation, Sec. 5.1, App. B.2 P:1059-1158 ---- */
double or_g(double y, double T);                 /* E[X_uv] given y = 2^d kappa w_u w_v / W */
double or_f_bruteforce(const double *w, uint64_t n, int d, double T, double kappa);
double or_f(const double *w, uint64_t n, int d, double T, double kappa); /* O(n + |R|) */
double or_ER_quadratic(const double *w, uint64_t n, int d, double T, double kappa);
double or_ER_linear(const double *w, uint64_t n, int d, double T, double kappa);
int or_scale_weights(const double *w, uint64_t n, double avg_deg, int d, double T,
                     double beta, double *kappa_out);

/* single geometric skip, P:494-501 (R10): floor(log(1-u)/log1p(-p)) */
int64_t or_geometric_skip(double p, double u);

#ifdef __cplusplus
}
#endif
#endif
