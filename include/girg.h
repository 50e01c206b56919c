/*
 * girg.h -- C ABI of the B200-native GIRG edge generator (libgirg.so).
 *
 * The operations follow the problem statement of arXiv:1905.06706 ("Efficiently generating
 * geometric inhomogeneous and hyperbolic random graphs"); "P:NNN" cites a line of its text
 * (PAPER.md).  All arithmetic runs in the library's sm_100a kernels; the host side only
 * validates arguments, computes O(#layers^2) tables and launches kernels.
 *
 * Conventions shared by every entry point
 *   - Pointers named *_dev are caller-owned DEVICE buffers (e.g. torch CUDA tensors); pointers
 *     named *_host / *_out are caller-owned HOST memory.  The library never frees or retains a
 *     caller pointer after the call returns.
 *   - Scratch memory is allocated stream-ordered (cudaMallocAsync on the current device's
 *     default pool) and released before return.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is enqueued on it.
 *     Calls on different streams may run concurrently from different host threads.
 *   - Return value: GIRG_OK (0) or a negative girg_status.  Arguments are validated before any
 *     launch; no C++ exception crosses the ABI.
 *   - Layout of positions: structure of arrays, x[k*n + v] = coordinate k of vertex v, k < d.
 *   - Vertex ids are uint32, so n < 2^32.
 */
#ifndef GIRG_H
#define GIRG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GIRG_OK = 0,
    GIRG_EINVAL = -1,    /* invalid argument (value, pointer, non-finite input) */
    GIRG_ECAPACITY = -2, /* edge buffer too small; *m_out holds the true edge count */
    GIRG_ERANGE = -3,    /* input outside the representable range of the index (see below) */
    GIRG_ENOMEM = -4,    /* device allocation failed */
    GIRG_ECUDA = -5      /* a CUDA runtime error; see girg_strerror / girg_last_cuda_error */
} girg_status;

/* Optional work counters of one girg_edges call (pass NULL to skip collecting them). */
typedef struct {
    uint64_t cand1;      /* type-I candidate pairs tested */
    uint64_t ev2;        /* nonempty type-II events */
    uint64_t chunks;     /* type-II jump chains                                  */
    uint64_t draws;      /* type-II Philox draws                                 */
    uint64_t landings;   /* type-II candidates reached by a jump                 */
    uint64_t edges1;     /* edges from type-I events                             */
    uint64_t edges2;     /* edges from type-II events                            */
    uint64_t neartie1;   /* |r - p_uv| < 1e-12 at a type-I test (device-side)    */
    uint64_t neartie2;   /* |r_acc - p_uv/pbar| < 1e-12 at a type-II acceptance  */
    uint64_t layers;     /* number of weight layers (buckets)                    */
    uint64_t key_space;  /* number of index cells sum_i 2^(d I(i))               */
    uint64_t fast_fallback; /* decisions the float fast path left to the canonical double path */
    uint64_t fast_mismatch; /* fast-path decisions that differ from the canonical one (must be 0) */
    uint64_t neartie_jump;  /* jump quotient z within 1e-15 max(1,|z|) of an integer where it can
                               matter (z < remaining + 1), R21 (device-side)          */
} girg_stats;

/*
 * girg_weights -- power-law weights, P:264-265 ("weights w_1..w_n following a power law with
 * exponent beta > 2").  Pareto law with w_min = 1, P(w >= x) = x^(1-beta), by inverse transform
 * w_v = (1-U_v)^(-1/(beta-1)); U_v is the 53-bit uniform from Philox4x32-10 counter (v,0,0,1),
 * key = seed.  Output w_dev[n] (float64).  Asynchronous.
 * Errors: EINVAL if n == 0, n >= 2^32, beta <= 2 or non-finite, w_dev == NULL.
 */
int girg_weights(uint64_t n, double beta, uint64_t seed, double *w_dev, void *stream);

/*
 * girg_positions -- uniform positions on the torus T^d = [0,1)^d.  Coordinates 2k
 * and 2k+1 of vertex v are the two 53-bit uniforms of Philox4x32-10 counter (v,k,0,2).
 * Output x_dev[d*n] (SoA, float64, on the 2^-53 grid).  Asynchronous.
 * Errors: EINVAL if n == 0, n >= 2^32, d not in [1,5], x_dev == NULL.
 */
int girg_positions(uint64_t n, int d, uint64_t seed, double *x_dev, void *stream);

/*
 * girg_scale_weights -- average-degree estimation, Sec. 5.1 P:627-658 and App. B.2
 * finds kappa such that the expected average degree f(kappa) of the GIRG with
 * weights w_dev[n], dimension d and temperature T equals avg_deg (exponential search and
 * bisection on the monotone f; f evaluated exactly from the actual weights, with the
 * saturated pairs E_R handled in O(|R|)).  kappa is the constant of the kappa form used by
 * girg_edges: p_uv = min(1, (kappa w_u w_v / (W ||x_u-x_v||^d))^(1/T)), i.e. kappa = c^T for
 * Eq. 1 (App. B.2 P:1073-1075 "scaling all weights by c^T"), kappa = c^d for T = 0.
 * beta only seeds the search (kappa0 = avg_deg (1-T) / (2^d (beta-1)/(beta-2))).
 * Writes *kappa_out (host).  Synchronises `stream`.
 * Errors: EINVAL if n < 2, avg_deg not in (0, n-1), d not in [1,5], T not in [0,1),
 * beta <= 2, a weight not finite and > 0; ERANGE if f overflows (extreme T / weights).
 */
int girg_scale_weights(const double *w_dev, uint64_t n, double avg_deg, int d, double T,
                       double beta, double *kappa_out, void *stream);

/*
 * girg_edges -- sample the GIRG edge set in expected linear time: weight layers,
 * the nested Morton-ordered grid and Lemma-1 index, and per layer pair the
 * neighbouring (type-I) cell pairs tested pair by pair and the distant (type-II) cell pairs
 * sampled by geometric jumps under the cell-pair bound pbar with rejection (Sec. 4.2-4.3,
 * Algorithm 1).
 *   T = 0 : threshold model, edge iff ||x_u-x_v||^d <= kappa w_u w_v / W.
 *   T > 0 : binomial model, independent edges with p_uv = min(1,(kappa w_u w_v/(W D))^(1/T)).
 * Inputs: w_dev[n] (finite, > 0), x_dev[d*n] (each coordinate in [0,1)), 0 <= T < 1,
 * kappa > 0 finite, seed (keys all Philox draws; the edge set is a pure function of
 * (w, x, d, T, kappa, seed) and does not depend on the schedule).
 * Output: edges_dev[cap][2] uint32 pairs (u, v) with u < v, in unspecified order, no
 * duplicates, no self-loops; *m_out (host) = number of edges.  Synchronises `stream`.
 * Errors: EINVAL (bad argument / input value), ECAPACITY (m > cap: *m_out = true m, buffer
 * contents unspecified; re-running with cap >= m gives the identical set), ERANGE (more than
 * 64 weight layers, weights outside [2^-500, 2^500], d*I(i) > 31 or index cells >= 2^32-1),
 * ENOMEM, ECUDA.
 */
int girg_edges(const double *w_dev, const double *x_dev, uint64_t n, int d, double T,
               double kappa, uint64_t seed, uint32_t *edges_dev, uint64_t cap,
               uint64_t *m_out, void *stream);

/*
 * girg_edges_shard -- girg_edges restricted to the events whose A cell (the cell of the
 * lower layer) lies in Morton blocks [blk_lo, blk_hi) at level shard_level (coarser events are
 * owned by the block of their first descendant).  Shards of one graph are disjoint and their
 * union is the girg_edges result (multi-GPU partitioning).
 * shard_level = 0, blk_lo = 0, blk_hi = 1 is the whole graph.  stats_out may be NULL.
 * Errors: as girg_edges, plus EINVAL if shard_level*d > 32 or blk_lo >= blk_hi.
 */
int girg_edges_shard(const double *w_dev, const double *x_dev, uint64_t n, int d, double T,
                     double kappa, uint64_t seed, int shard_level, uint64_t blk_lo,
                     uint64_t blk_hi, uint32_t *edges_dev, uint64_t cap, uint64_t *m_out,
                     girg_stats *stats_out, void *stream);

/* type-II sampling schemes (R10 / R22 / R27).  Each gives exactly the GIRG distribution;
 * for a fixed seed they give different (each deterministic) edge sets. */
#define GIRG_SCHEME_EVENT 0  /* one geometric-jump sequence per distant cell pair: Alg. 1 lines 5-6
                                as written, chunks of 2..4 expected landings */
#define GIRG_SCHEME_MERGED 1 /* default: the distant cells of an A cell with the same bound class
                                concatenated into one sequence (memorylessness of the jumps,
                                P:494-501), chunks of 2..4 expected landings */
#define GIRG_SCHEME_REFINED 2 /* MERGED with the refined bound of DESIGN.md R27 (P:486-491 with a
                                tighter minimum distance) where it pays: for d = 2, 3, T > 0, on the
                                levels l < CL(i,j) with >= 4096 points of layer i per cell, the rows of
                                an A cell are split by A's children on level l+1 and its distant
                                cells classed by their box distance from the child (2, 3, >= 4
                                half-cells), one sequence per (child, class).  Elsewhere (and for
                                other d or T = 0) identical to MERGED */

typedef struct {
    int scheme;           /* GIRG_SCHEME_MERGED (default), GIRG_SCHEME_EVENT or GIRG_SCHEME_REFINED */
    int shard_level;      /* as girg_edges_shard; 0, [0, 1) = the whole graph */
    uint64_t blk_lo, blk_hi;
    /* interleaved multi-GPU ownership (nranks > 0; blk_lo / blk_hi are then ignored): an event
     * whose A cell is on a level l >= shard_level belongs to rank (Morton block of A at
     * shard_level) mod nranks; a coarser event (l < shard_level) to rank
     * (A + 7 j + 13 i + 31 l) mod nranks (A its Morton code on level l, (i, j) its layer pair),
     * so the few large coarse events are spread over the ranks instead of falling to the first
     * blocks.  The nranks shards of one graph are disjoint and their union is the whole graph.
     * EINVAL if rank >= nranks.  nranks = 0: block-range mode as girg_edges_shard. */
    uint32_t nranks, rank;
} girg_options;

/*
 * girg_edges_ex -- girg_edges with explicit options (NULL = defaults: merged scheme, whole
 * graph) and optional work counters (stats_out may be NULL).  Same semantics and errors as
 * girg_edges_shard, plus EINVAL for an unknown scheme.
 */
int girg_edges_ex(const double *w_dev, const double *x_dev, uint64_t n, int d, double T,
                  double kappa, uint64_t seed, const girg_options *opt, uint32_t *edges_dev,
                  uint64_t cap, uint64_t *m_out, girg_stats *stats_out, void *stream);

/*
 * girg_edges_host -- end-to-end variant with HOST buffers: copies w_host[n] and x_host[d*n]
 * to the device and runs girg_edges.  If edges_host[cap][2] is page-locked (cudaHostAlloc /
 * cudaHostRegister / torch pin_memory) the sampling kernels write the edges directly into it
 * over the bus while they run; otherwise they are copied back after the run.  Same semantics
 * and errors as girg_edges.
 */
int girg_edges_host(const double *w_host, const double *x_host, uint64_t n, int d, double T,
                    double kappa, uint64_t seed, uint32_t *edges_host, uint64_t cap,
                    uint64_t *m_out, void *stream);

/*
 * girg_edges_batch -- many independent GIRGs in one call ("batched small
 * graphs"; the paper's observation that many instances of a generator beat one parallel
 * instance for small n).  Graph g is exactly girg_edges(w_dev[g], x_dev[g], n, d, T,
 * kappa[g], seed[g], edges_dev[g], cap[g], &m_out[g], .) -- the same edge set, bit for bit.
 *   B            number of graphs (>= 1); all share n, d and T
 *   w_dev, x_dev host arrays of B device pointers: w[n] and x[d][n] (SoA) of each graph
 *   kappa, seed  host arrays [B]
 *   edges_dev    host array of B device pointers to caller-owned uint32 [cap[g]][2] buffers
 *   cap          host array [B]
 *   m_out        host array [B]: the true edge count of each graph (also when > cap[g])
 *   status_out   host array [B] or NULL: the girg_status of each graph
 *   nstreams     execution: for B >= 2 graphs of n <= 2^22 points (and B n < 2^31) the batch is
 *                FUSED -- one launch per kernel for all graphs (weight statistics, one counting
 *                sort over the concatenated cell spaces, sampling with one block row per graph)
 *                and two synchronisations in total; nstreams < 0 (or larger graphs) runs the
 *                graphs as independent girg_edges pipelines on |nstreams| internal streams, one
 *                native host thread each (0 = 8)
 *   stream       ordering: the batch starts after the work already queued on `stream` and the
 *                call returns when every graph is done (it synchronises, as girg_edges does)
 * Returns GIRG_OK if every graph succeeded, else the status of the lowest failing index
 * (GIRG_ECAPACITY included); EINVAL for B < 1 or NULL arrays.
 */
int girg_edges_batch(int B, const double *const *w_dev, const double *const *x_dev, uint64_t n,
                     int d, double T, const double *kappa, const uint64_t *seed,
                     uint32_t *const *edges_dev, const uint64_t *cap, uint64_t *m_out,
                     int *status_out, int nstreams, void *stream);

/*
 * Hyperbolic random graphs (Sec. 3.2) on the GIRG machinery (Sec. 3.3
 * P:341-351; R25).
 *
 * girg_hrg_points -- n HRG points: radius r_v with density alpha sinh(alpha r)/(cosh(alpha R)-1)
 * on [0, R), R = 2 ln(n) + C, by inverse transform of the 53-bit uniform U of Philox
 * counter (v, 0, 0, 7) words (o0, o1): r = acosh(1 + U (cosh(alpha R) - 1)) / alpha; the angle as
 * the torus position x_v = theta_v / (2 pi) = words (o2, o3); and the dominating GIRG
 * weight w'_v = e^((R - r_v)/2) / sqrt(1 - e^(-2 r_v)) (e^(R/2) at r_v = 0).  Outputs r_dev[n],
 * x_dev[n], w_dev[n] (float64, caller-owned device buffers).  Asynchronous.
 * Errors: EINVAL if n < 2, n >= 2^32, alpha <= 1/2 or not finite, C not finite, R <= 0, a NULL
 * pointer; ERANGE if cosh(alpha R) overflows.
 */
int girg_hrg_points(uint64_t n, double alpha, double C, uint64_t seed, double *r_dev, double *x_dev,
                    double *w_dev, void *stream);

typedef struct {
    uint64_t super_edges; /* edges of the dominating GIRG                                  */
    uint64_t neartie;     /* thinning decisions within 1e-12 of their threshold (must be 0) */
    uint64_t violations;  /* pairs with p_HRG > p_GIRG' (must be 0)                         */
} girg_hrg_stats;

/*
 * girg_hrg_edges -- the HRG edge set of points (r_dev, x_dev) with dominating weights w_dev
 * (girg_hrg_points), R = 2 ln(n) + C, temperature T in [0, 1): T = 0 threshold model, edge iff
 * the hyperbolic distance d < R; T > 0 binomial model, p_T(d) = 1/(exp((d-R)/(2T))+1)
 * (P:316-318); cosh d = cosh r_u cosh r_v - sinh r_u sinh r_v cos(2 pi dx).
 * Sampled exactly as girg_edges of the dominating GIRG (w', x, d = 1, T, s = e^(-R/2)/sqrt(2)
 * (1 + 2^-30) instead of kappa/W, merged scheme, `seed`) thinned by p_HRG / p_GIRG' (uniform of
 * Philox counter (u, v, 0, 6), u < v; T = 0: the exact test cosh d < cosh R).  Output as
 * girg_edges: edges_dev[cap][2] uint32 (u < v), *m_out, ECAPACITY when m > cap (then re-run with
 * cap >= m: identical set).  stats_out may be NULL.  Synchronises `stream`.
 * Errors: EINVAL (NULL pointer, n < 2, T not in [0,1), C not finite, R <= 0), ECAPACITY, ENOMEM,
 * ECUDA, and the errors of girg_edges for the dominating GIRG (e.g. ERANGE for > 64 layers).
 */
int girg_hrg_edges(const double *r_dev, const double *x_dev, const double *w_dev, uint64_t n,
                   double C, double T, uint64_t seed, uint32_t *edges_dev, uint64_t cap,
                   uint64_t *m_out, girg_hrg_stats *stats_out, void *stream);

/* Phase timings of the last successful girg_edges / girg_edges_shard / girg_edges_host call on
 * the calling host thread, measured with CUDA events recorded on the call's stream around each
 * phase (the events cost ~1 us; they are always recorded). */
typedef struct {
    double ms_total;   /* whole call: first launch .. edge count read back (device clock)       */
    double ms_wstats;  /* K0 weight statistics + host plan (includes the one mid-call sync)      */
    double ms_index;   /* K1-K4 keys, scan, scatter, in-cell order / gather (Lemma-1 index)      */
    double ms_sample;  /* K5 sampling kernel (type-I tests, type-II jumps, edge output)          */
    uint64_t launches; /* kernels launched by the call                                          */
    uint64_t n, m, key_space;
    int d;
    int pad;
} girg_timings;
int girg_last_timings(girg_timings *out);

/* Human-readable text of a status code (static storage). */
const char *girg_strerror(int status);

/* The CUDA runtime error string of the last GIRG_ECUDA on this host thread ("" if none). */
const char *girg_last_cuda_error(void);

/* Library ABI version (major*100 + minor). */
int girg_version(void);

/* TEST HOOK (not part of the product API): threshold of GIRG_SCHEME_REFINED's level rule, in
 * points of layer i per level-l cell: 0 = the default (4096), k > 0 = k points, -1 = every level
 * l < CL(i,j), so that small parity cases exercise refined sequences.  Process-wide.  Returns 0. */
int girg_debug_set_ref_x(int x);

/* TEST HOOK (not part of the product API): the Lemma-1 index that girg_edges builds for these
 * inputs (App. A; H5), for a direct comparison with the oracle's:
 * sid_dev[n] (device) = vertex ids in sorted order (by layer, then Morton cell on level I(layer),
 * then id); P_dev[min(K+1, P_cap)] (device) = first sorted position of every cell of the
 * concatenated cell space (layer i's 2^(d I(i)) cells start at base[i]; P[K] = n).  Host outputs:
 * *K_out, *L_out (layers), base_out[L+1], lstart_out[L+1], I_out[L] (arrays of 65 / 65 / 64).
 * Either device pointer may be NULL.  Runs the whole pipeline with edge capacity 0.  Synchronises. */
int girg_debug_index(const double *w_dev, const double *x_dev, uint64_t n, int d, double T, double kappa,
                     uint32_t *sid_dev, uint32_t *P_dev, uint64_t P_cap, uint64_t *K_out, int *L_out,
                     uint32_t *base_out, uint32_t *lstart_out, uint8_t *I_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GIRG_H */
