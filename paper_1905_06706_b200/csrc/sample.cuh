// sample.cuh -- K5: the GIRG sampling kernels (v4), included by girg.cu inside namespace girg.
//
// Events (Algorithm 1; R2, R16): for a layer pair i <= j, a neighbouring cell pair
// (A, B) on level CL(i,j) is a type-I event (every candidate tested, Alg. 1 line 3), a distant
// cell pair with neighbouring parents on a level 2 <= l <= CL(i,j) is a type-II event (geometric
// jumps under the bound pbar, Alg. 1 lines 5-6).  Every event of a level-l cell A
// lies inside the "region" of A's parent: the 2^d children of the 3^d neighbours of parent(A)
// (all cells of level l when l <= 2).
//
// Work decomposition:
//   * task = (layer i, partner j, level l, parent cell Cpar of layer i on level l-1).  It is
//     owned by the first sorted point of Cpar, so every nonempty parent is visited exactly once
//     per (j, l); host tables list the tasks of a point by (layer, first level lf).
//   * one warp per task: lanes load the region's Lemma-1 ranges (P entries) once for the up to
//     2^d children A of Cpar, classify the region's cells per child (kind 0: neighbour / type-I,
//     kind 1: distant with delta_max = 2, kind 2: delta_max = 3) as bit masks, and prefix-sum
//     the per-parent counts in Morton order.
//   * units: a type-I candidate pair, or one chunk (jump chain) of a type-II sequence.  A
//     sequence is one distant cell pair (scheme EVENT, Alg. 1 as written) or the concatenation of
//     all distant cells of A with the same bound class (scheme MERGED, R22).  Lanes pull units
//     dynamically and advance one Philox draw / one candidate per step, so jump chains of
//     different lengths do not serialise the warp.
//   * tasks with too much work are split into unit-range items of a global queue (k_big).
//   * edges are staged per warp in shared memory and written with one atomic per flush.
#pragma once

// GIRG_DEBUG builds (libgirg_debug.so) bounds-check the indexed accesses of the sampler
#ifdef GIRG_DEBUG
#define GCHK(cond)                                                                                   \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("GIRG_DEBUG check failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   blockIdx.x, threadIdx.x);                                                         \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define GCHK(cond) \
    do {           \
    } while (0)
#endif

constexpr int SCHEME_EVENT = 0, SCHEME_MERGED = 1;
constexpr int EB = 256;                          // staged edges per warp
constexpr unsigned long long BIG_WORK = 24576;   // weighted units above which a batch is queued
constexpr unsigned long long ITEM_WORK = 6144;   // weighted units per queued item
constexpr int ERR_ITEMS = 16;

template <int D>
struct Geo {
    static constexpr int G = D == 1 ? 3 : 1;                 // levels between a task cell and its children
    static constexpr int NCH = 1 << (D * G);                 // children (= sub-cells per region parent)
    static constexpr int NPAR = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : 243;  // 3^d
    static constexpr int MAXPAR = NPAR > (1 << D) ? NPAR : (1 << D);  // level-1 tasks: all 2^d level-1 cells
    static constexpr int CB = D <= 3 ? NCH : (D == 4 ? 4 : 2);        // children per batch
    static constexpr int WPB = D <= 3 ? 8 : (D == 4 ? 4 : 2);         // warps per block
    static constexpr int MINB = D <= 2 ? 4 : (D == 3 ? 3 : 1);        // resident blocks per SM (register cap)
    static constexpr int RECW = D == 1 ? 2 : (D <= 3 ? 4 : 6);       // doubles per point record
};

struct Counters {
    unsigned long long cand1, ev2, chunks, draws, landings, edges1, edges2, nt1, nt2;
};

// one (child, kind) sequence of a batch
struct Seq {
    unsigned long long units;  // candidates (kind 0) or chunks (kinds 1, 2)
    unsigned long long N;      // merged: nA * M
    uint32_t A, a0, nA, M;     // child cell, its sorted range, candidates per row (kind 0 / merged)
    int cl2;                   // log2 chunk length (merged)
    int pad;
};

struct BigItem {
    uint32_t Cpar;
    uint16_t task;     // j | l<<6 | t1<<12 | t2<<13
    uint8_t i, batch;
    unsigned long long lo, hi;  // unit range of the batch
};

struct SampleArgs {
    const Plan* pl;
    const TabEntry* tab;
    const uint16_t* tasks;
    const uint32_t* skey;
    const double* rec;  // sorted point records [n][RECW]: x_0..x_{d-1}, w
    const uint32_t* sid;
    const uint32_t* P;
    uint32_t n, ntiles;
    uint32_t k0, k1;
    uint2* edges;
    unsigned long long cap;
    unsigned long long* m;
    unsigned int* tile_ctr;
    BigItem* items;
    unsigned int* nitems;
    unsigned int items_cap;
    Counters* stats;
    int* err;
    unsigned long long nP;
    unsigned int ntab, ntasks;
};

template <int D>
struct WarpSmem {
    static constexpr int NPAR = Geo<D>::MAXPAR, NCH = Geo<D>::NCH, CB = Geo<D>::CB;
    uint32_t par[NPAR];                   // region parent codes on level l-1, Morton order
    uint32_t rstart[NPAR][NCH + 1];       // sorted positions of the region sub-cells (layer j)
    uint32_t achild[NCH + 1];             // sorted positions of Cpar's children (layer i)
    uint32_t pre[CB][3][NPAR + 1];        // per (child, kind): prefix over parents (candidates / chunks)
    uint32_t mask[CB][3][NPAR];           // per (child, kind, parent): sub-cells of that kind
    Seq seq[CB][3];
    unsigned long long uoff[CB * 3 + 1];  // unit offsets of the (child, kind) sequences
    uint8_t child[NCH];                   // nonempty owned children of Cpar
    uint2 ebuf[EB];
};

// ---------------------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total)
{
    const unsigned lane = lane_id();
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__device__ __forceinline__ void warp_flush(const SampleArgs& a, uint2* buf, unsigned& fill)
{
    __syncwarp();
    unsigned long long base = 0;
    if (lane_id() == 0 && fill) base = atomicAdd(a.m, (unsigned long long)fill);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (unsigned k = lane_id(); k < fill; k += 32) {
        const unsigned long long slot = base + k;
        if (slot < a.cap) a.edges[slot] = buf[k];
    }
    __syncwarp();
    fill = 0;
}

// append this lane's edge (if any); `fill` is warp-uniform
__device__ __forceinline__ void warp_emit(const SampleArgs& a, uint2* buf, unsigned& fill, bool edge, uint32_t u,
                                          uint32_t v)
{
    const unsigned em = __ballot_sync(0xffffffffu, edge);
    if (!em) return;
    const unsigned cnt = __popc(em);
    if (fill + cnt > (unsigned)EB) warp_flush(a, buf, fill);
    if (edge) buf[fill + __popc(em & ((1u << lane_id()) - 1u))] = make_uint2(min(u, v), max(u, v));
    fill += cnt;
}

template <int D>
__device__ __forceinline__ void load_rec(const SampleArgs& a, uint32_t p, double (&xp)[D], double& w)
{
    GCHK(p < a.n);
    const double2* r = reinterpret_cast<const double2*>(a.rec + (size_t)p * Geo<D>::RECW);
    double v[Geo<D>::RECW];
#pragma unroll
    for (int k = 0; k < Geo<D>::RECW / 2; ++k) {
        const double2 t = __ldg(r + k);
        v[2 * k] = t.x;
        v[2 * k + 1] = t.y;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) xp[k] = v[k];
    w = v[D];
}

// torus cell gap on level l per dimension, max over dimensions (R8): delta_max(A, B)
template <int D>
__device__ __forceinline__ int delta_max_cells(const uint32_t (&ac)[D], uint32_t B, int l)
{
    if (l == 0) return 0;
    uint32_t bc[D];
    morton_decode<D>(B, bc);
    const uint32_t side = 1u << l;
    int dm = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const uint32_t g = ac[k] > bc[k] ? ac[k] - bc[k] : bc[k] - ac[k];
        dm = max(dm, (int)min(g, side - g));
    }
    return dm;
}

// ---------------------------------------------------------------------------------------
// task setup: region parents, their sub-cell ranges in layer j, Cpar's children in layer i
// ---------------------------------------------------------------------------------------
struct TaskDesc {
    int i, j, l, t1, t2;
    uint32_t Cpar;  // the task cell, on level lg = max(0, l - G)
    int lg, npar, cs;  // task level, region parents, child shift d (l - lg)
};

template <int D>
__device__ __forceinline__ void setup_task(const SampleArgs& a, WarpSmem<D>& W, const TaskDesc& t, int& nchild)
{
    constexpr int NCH = Geo<D>::NCH;
    const Plan* pl = a.pl;
    const unsigned lane = lane_id();
    const int nsub = 1 << t.cs;
    // region parents in Morton order
    if (t.lg >= 2) {
        const int lam = t.lg;
        uint32_t pc[D];
        morton_decode<D>(t.Cpar, pc);
        const uint32_t mask = (1u << lam) - 1u;
        for (int q = lane; q < t.npar; q += 32) {
            uint32_t c[D];
            int r = q;
#pragma unroll
            for (int k = D - 1; k >= 0; --k) {  // offsets in {-1,0,1}^d (any fixed order; sorted below)
                c[k] = (pc[k] + (uint32_t)(r % 3) - 1u) & mask;
                r /= 3;
            }
            W.par[q] = morton_encode<D>(c);
        }
        __syncwarp();
        // rank sort (codes are distinct on levels >= 2)
        uint32_t mine[(Geo<D>::MAXPAR + 31) / 32];
        int rk[(Geo<D>::MAXPAR + 31) / 32];
#pragma unroll
        for (int s = 0; s < (Geo<D>::MAXPAR + 31) / 32; ++s) {
            const int q = lane + 32 * s;
            rk[s] = 0;
            mine[s] = q < t.npar ? W.par[q] : 0u;
            if (q < t.npar)
                for (int o = 0; o < t.npar; ++o) rk[s] += W.par[o] < mine[s];
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < (Geo<D>::MAXPAR + 31) / 32; ++s) {
            const int q = lane + 32 * s;
            if (q < t.npar) W.par[rk[s]] = mine[s];
        }
    } else {
        for (int q = lane; q < t.npar; q += 32) W.par[q] = (uint32_t)q;  // lg = 1: all level-1 cells; lg = 0: root
    }
    __syncwarp();
    // Lemma-1 ranges of the region sub-cells in layer j and of Cpar's children in layer i
    const int shj = D * ((int)pl->I[t.j] - t.l), shi = D * ((int)pl->I[t.i] - t.l);
    const uint32_t bj = pl->base[t.j], bi = pl->base[t.i];
    const int per = nsub + 1;
    for (int e = lane; e < t.npar * per; e += 32) {
        const int q = e / per, k = e - q * per;
        const unsigned long long cell = ((unsigned long long)W.par[q] << t.cs) + (unsigned)k;
        GCHK(bj + (cell << shj) < a.nP);
        W.rstart[q][k] = __ldg(&a.P[bj + (cell << shj)]);
    }
    for (int k = lane; k <= nsub; k += 32) {
        const unsigned long long cell = ((unsigned long long)t.Cpar << t.cs) + (unsigned)k;
        GCHK(bi + (cell << shi) < a.nP);
        W.achild[k] = __ldg(&a.P[bi + (cell << shi)]);
    }
    __syncwarp();
    // nonempty children owned by this shard (ownership by the A cell's block)
    bool ok = false;
    if ((int)lane < nsub) {
        ok = W.achild[lane + 1] > W.achild[lane];
        const uint32_t A = (t.Cpar << t.cs) + lane;
        const unsigned long long b = t.l >= pl->sl ? ((unsigned long long)A >> (D * (t.l - pl->sl)))
                                                   : ((unsigned long long)A << (D * (pl->sl - t.l)));
        ok = ok && b >= pl->blo && b < pl->bhi;
    }
    const unsigned bm = __ballot_sync(0xffffffffu, ok);
    if (ok) W.child[__popc(bm & ((1u << lane) - 1u))] = (uint8_t)lane;
    nchild = __popc(bm);
    (void)NCH;
    __syncwarp();
}

// chunk length (log2) of a type-II sequence of N candidates with table log2 length c0 and a
// cap of 2^capbits chunks (R10 / R22)
__device__ __forceinline__ int chunk_log2(unsigned long long N, int c0, int capbits)
{
    int c = c0;
    while (((N - 1) >> c) >= (1ull << capbits)) ++c;
    return c;
}

// kind of region sub-cell B relative to child A (-1: none): 0 neighbours (type-I), 1 / 2 distant
// with neighbouring parents and delta_max = 2 / 3 (type-II)
template <int D>
__device__ __forceinline__ int kind_of(const TaskDesc& t, const uint32_t (&ac)[D], uint32_t A, uint32_t B)
{
    const int dm = delta_max_cells<D>(ac, B, t.l);
    if (dm <= 1) return (t.t1 && (t.i < t.j || B >= A)) ? 0 : -1;
    if (!t.t2 || (t.i == t.j && B <= A)) return -1;
    if (Geo<D>::G > 1 && t.l >= 3) {  // the region spans more than parent(A)'s neighbours
        uint32_t pa[D];
#pragma unroll
        for (int k = 0; k < D; ++k) pa[k] = ac[k] >> 1;
        if (delta_max_cells<D>(pa, B >> D, t.l - 1) > 1) return -1;
    }
    return dm - 1;  // 1: delta_max = 2, 2: delta_max = 3
}

// per-batch setup: masks, per-parent prefix counts, sequences and unit offsets
template <int D, int SCHEME>
__device__ __forceinline__ unsigned long long setup_batch(const SampleArgs& a, WarpSmem<D>& W, const TaskDesc& t,
                                                          int c0, int nc, unsigned long long& work)
{
    const unsigned lane = lane_id();
    const int nsub = 1 << t.cs;
    const TabEntry* te = t.t2 ? a.tab + (a.pl->tab_off[t.i * MAXL + t.j] + 2u * (uint32_t)(t.l - 2)) : nullptr;
    unsigned long long wk = 0;
    for (int cc = 0; cc < nc; ++cc) {
        const int e = W.child[c0 + cc];
        const uint32_t A = (t.Cpar << t.cs) + (uint32_t)e;
        uint32_t ac[D];
        morton_decode<D>(A, ac);
        const uint32_t a0 = W.achild[e], nA = W.achild[e + 1] - a0;
        uint32_t base[3] = {0u, 0u, 0u};
        for (int q0 = 0; q0 < t.npar; q0 += 32) {
            const int q = q0 + (int)lane;
            uint32_t cnt[3] = {0u, 0u, 0u}, m[3] = {0u, 0u, 0u};
            if (q < t.npar) {
                for (int s = 0; s < nsub; ++s) {
                    const uint32_t B = (W.par[q] << t.cs) + (uint32_t)s;
                    const int k = kind_of<D>(t, ac, A, B);
                    if (k < 0) continue;
                    const uint32_t nB = W.rstart[q][s + 1] - W.rstart[q][s];
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk) {
                        if (kk != k) continue;
                        m[kk] |= 1u << s;
                        if (kk == 0 || SCHEME == SCHEME_MERGED) {
                            cnt[kk] += nB;
                        } else if (nB) {  // EVENT: chunks of the event (A, B)
                            const unsigned long long N = (unsigned long long)nA * nB;
                            const TabEntry& tk = te[kk - 1];
                            if (tk.pbar > 0.0) cnt[kk] += (uint32_t)(((N - 1) >> chunk_log2(N, tk.clog2, 15)) + 1);
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) W.mask[cc][kk][q] = m[kk];
            }
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                uint32_t tot;
                const uint32_t ex = warp_excl_scan(cnt[kk], tot);
                if (q < t.npar) W.pre[cc][kk][q] = base[kk] + ex;
                base[kk] += tot;
            }
        }
        if (lane < 3) {
            const int k = (int)lane;
            const uint32_t M = k == 0 ? base[0] : (k == 1 ? base[1] : base[2]);
            W.pre[cc][k][t.npar] = M;
            Seq& S = W.seq[cc][k];
            S.A = A;
            S.a0 = a0;
            S.nA = nA;
            S.M = M;
            S.cl2 = 0;
            S.N = 0;
            unsigned long long units = 0;
            if (k == 0) {
                units = (unsigned long long)nA * M;
            } else if (SCHEME == SCHEME_EVENT) {
                units = M;
            } else if (M) {
                const TabEntry& tk = te[k - 1];
                if (tk.pbar > 0.0) {
                    S.N = (unsigned long long)nA * M;
                    S.cl2 = chunk_log2(S.N, tk.clog2m, 32);
                    units = ((S.N - 1) >> S.cl2) + 1;
                }
            }
            S.units = units;
            wk += units * (k == 0 ? 1ull : 8ull);
        }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) wk += __shfl_xor_sync(0xffffffffu, wk, o);
    __syncwarp();
    if (lane == 0) {
        unsigned long long acc = 0;
        for (int s = 0; s < nc * 3; ++s) {
            W.uoff[s] = acc;
            acc += W.seq[s / 3][s % 3].units;
        }
        W.uoff[nc * 3] = acc;
    }
    __syncwarp();
    work = __shfl_sync(0xffffffffu, wk, 0);
    return W.uoff[nc * 3];
}

// concatenated index t (< M) of sequence (cc, k) -> sorted position in layer j and the cell
template <int D>
__device__ __forceinline__ uint32_t locate(const WarpSmem<D>& W, int npar, int cs, int cc, int k, uint32_t t,
                                           uint32_t& B)
{
    int lo = 0, hi = npar - 1;  // last parent with pre <= t
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (W.pre[cc][k][mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    uint32_t r = t - W.pre[cc][k][lo];
    uint32_t m = W.mask[cc][k][lo];
    for (;;) {
        GCHK(m != 0);
        const int s = __ffs(m) - 1;
        const uint32_t nB = W.rstart[lo][s + 1] - W.rstart[lo][s];
        if (r < nB) {
            B = (W.par[lo] << cs) + (uint32_t)s;
            return W.rstart[lo][s] + r;
        }
        r -= nB;
        m &= m - 1u;
    }
}

// EVENT scheme: chunk index u of sequence (cc, k) -> event (B, its range) and chunk within it
template <int D>
__device__ __forceinline__ void locate_event(const WarpSmem<D>& W, const TabEntry& tk, int npar, int cs, int cc,
                                             int k, uint32_t nA, uint32_t u, uint32_t& B, uint32_t& b0,
                                             uint32_t& nB, uint32_t& ch, int& cl2)
{
    int lo = 0, hi = npar - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (W.pre[cc][k][mid] <= u) lo = mid;
        else hi = mid - 1;
    }
    uint32_t r = u - W.pre[cc][k][lo];
    uint32_t m = W.mask[cc][k][lo];
    for (;;) {
        GCHK(m != 0);
        const int s = __ffs(m) - 1;
        m &= m - 1u;
        const uint32_t nb = W.rstart[lo][s + 1] - W.rstart[lo][s];
        if (!nb) continue;
        const unsigned long long N = (unsigned long long)nA * nb;
        const int c = chunk_log2(N, tk.clog2, 15);
        const uint32_t nch = (uint32_t)(((N - 1) >> c) + 1);
        if (r < nch) {
            B = (W.par[lo] << cs) + (uint32_t)s;
            b0 = W.rstart[lo][s];
            nB = nb;
            ch = r;
            cl2 = c;
            return;
        }
        r -= nch;
    }
}

// ---------------------------------------------------------------------------------------
// unit processing: lanes pull units of the batch's range [lo, hi) and advance one step each
// ---------------------------------------------------------------------------------------
template <int D, int SCHEME, bool STATS>
__device__ __forceinline__ void run_units(const SampleArgs& a, WarpSmem<D>& W, const TaskDesc& t, int nc,
                                          unsigned long long lo, unsigned long long hi, unsigned& fill,
                                          Counters& C)
{
    const Plan* pl = a.pl;
    const unsigned lane = lane_id();
    const bool T0 = pl->T == 0.0;
    const TabEntry* te = t.t2 ? a.tab + (pl->tab_off[t.i * MAXL + t.j] + 2u * (uint32_t)(t.l - 2)) : nullptr;
    const uint32_t tag_base = (uint32_t)t.l | ((uint32_t)t.i << 5) | ((uint32_t)t.j << 11);
    const bool same_layer = t.i == t.j;
    unsigned long long next = lo;
    bool busy = false;
    int cc = 0, kind = 0;
    // type-I unit state
    uint32_t pa = 0, pb = 0, ua = 0, ub = 0;
    // type-II chain state
    long long pos = 0, end = 0;
    uint32_t r = 0, ch = 0, Bev = 0, eb0 = 0, enB = 0;
    for (;;) {
        const unsigned idle = __ballot_sync(0xffffffffu, !busy);
        if (next >= hi && idle == 0xffffffffu) break;
        if (!busy && next < hi) {
            const unsigned long long u = next + __popc(idle & ((1u << lane) - 1u));
            if (u < hi) {
                int s = 0;  // sequence holding unit u
                while (W.uoff[s + 1] <= u) ++s;
                cc = s / 3;
                kind = s - 3 * cc;
                const Seq& S = W.seq[cc][kind];
                const unsigned long long x = u - W.uoff[s];
                if (kind == 0) {
                    const uint32_t si = (uint32_t)(x / S.M), ti = (uint32_t)(x - (unsigned long long)si * S.M);
                    uint32_t B;
                    pa = S.a0 + si;
                    pb = locate<D>(W, t.npar, t.cs, cc, 0, ti, B);
                    busy = !(same_layer && B == S.A && pb <= pa);  // same cell: only s < t (R16)
                    if (busy && !T0) {
                        ua = __ldg(&a.sid[pa]);
                        ub = __ldg(&a.sid[pb]);
                    }
                } else {
                    busy = true;
                    r = 0;
                    if (SCHEME == SCHEME_MERGED) {
                        ch = (uint32_t)x;
                        const unsigned long long st = x << S.cl2;
                        pos = (long long)st - 1;
                        end = (long long)min(S.N, st + (1ull << S.cl2));
                    } else {
                        int c2;
                        locate_event<D>(W, te[kind - 1], t.npar, t.cs, cc, kind, S.nA, (uint32_t)x, Bev, eb0, enB,
                                        ch, c2);
                        const unsigned long long N = (unsigned long long)S.nA * enB;
                        const unsigned long long st = (unsigned long long)ch << c2;
                        pos = (long long)st - 1;
                        end = (long long)min(N, st + (1ull << c2));
                    }
                    if (STATS) ++C.chunks;
                }
            }
        }
        next += __popc(idle);
        // ---- one step ----
        bool have = false, edge = false;
        double ra = 0.0, pbar = 1.0;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (busy && !T0) {
            const Seq& S = W.seq[cc][kind];
            uint4 ctr;
            if (kind == 0) ctr = make_uint4(min(ua, ub), max(ua, ub), 0u, 3u);
            else if (SCHEME == SCHEME_MERGED) ctr = make_uint4(S.A, ch, tag_base | ((uint32_t)(kind - 1) << 17) | (1u << 18), r);
            else ctr = make_uint4(S.A, Bev, tag_base | (ch << 17), r);
            o = philox4x32_10(ctr, a.k0, a.k1);
        }
        if (busy) {
            if (kind == 0) {
                have = true;
            } else {
                const Seq& S = W.seq[cc][kind];
                const TabEntry& tk = te[kind - 1];
                pbar = tk.pbar;
                ++r;
                if (STATS) ++C.draws;
                const double rj = u53(o.x, o.y);
                ra = u53(o.z, o.w);
                const double z = pbar == 1.0 ? 0.0 : __ddiv_rn(log(__dsub_rn(1.0, rj)), tk.Lbar);
                const long long remaining = end - pos - 1;
                if (z >= (double)remaining) {
                    busy = false;
                } else {
                    pos += 1 + (long long)z;
                    have = true;
                    if (STATS) ++C.landings;
                    if (SCHEME == SCHEME_MERGED) {
                        const unsigned long long g = (unsigned long long)pos;
                        uint32_t si, ti;
                        if (S.N <= 0xFFFFFFFFull) {
                            si = (uint32_t)g / S.M;
                            ti = (uint32_t)g - si * S.M;
                        } else {
                            si = (uint32_t)(g / S.M);
                            ti = (uint32_t)(g - (unsigned long long)si * S.M);
                        }
                        uint32_t B;
                        pa = S.a0 + si;
                        pb = locate<D>(W, t.npar, t.cs, cc, kind, ti, B);
                    } else {
                        const unsigned long long g = (unsigned long long)pos;
                        const uint32_t si = (uint32_t)(g / enB), ti = (uint32_t)(g - (unsigned long long)si * enB);
                        pa = S.a0 + si;
                        pb = eb0 + ti;
                    }
                }
            }
        }
        if (have) {
            double xu[D], xv[D], wu, wv;
            load_rec<D>(a, pa, xu, wu);
            load_rec<D>(a, pb, xv, wv);
            const double Dp = dist_pow<D>(xu, xv);
            if (T0) {
                edge = Dp <= __dmul_rn(__dmul_rn(wu, wv), pl->s);
            } else {
                const double p = prob_uv(wu, wv, pl->s, Dp, pl->invT);
                if (kind == 0) {
                    const double r1 = u53(o.x, o.y);
                    if (STATS && p < 1.0) C.nt1 += fabs(r1 - p) < 1e-12;
                    edge = p >= 1.0 || r1 < p;
                } else {
                    const double rp = __dmul_rn(ra, pbar);
                    if (STATS) C.nt2 += fabs(rp - p) < 1e-12 * pbar;
                    edge = rp < p;
                }
            }
            if (kind == 0) {
                busy = false;
                if (STATS) ++C.cand1;
            }
            if (edge) {
                if (STATS) {
                    if (kind == 0) ++C.edges1;
                    else ++C.edges2;
                }
                if (kind != 0 || T0) {
                    ua = __ldg(&a.sid[pa]);
                    ub = __ldg(&a.sid[pb]);
                }
            }
        }
        warp_emit(a, W.ebuf, fill, edge, ua, ub);
    }
}

template <bool STATS>
__device__ __forceinline__ void flush_counters(const SampleArgs& a, const Counters& c)
{
    if (!STATS) return;
    atomicAdd(&a.stats->cand1, c.cand1);
    atomicAdd(&a.stats->ev2, c.ev2);
    atomicAdd(&a.stats->chunks, c.chunks);
    atomicAdd(&a.stats->draws, c.draws);
    atomicAdd(&a.stats->landings, c.landings);
    atomicAdd(&a.stats->edges1, c.edges1);
    atomicAdd(&a.stats->edges2, c.edges2);
    atomicAdd(&a.stats->nt1, c.nt1);
    atomicAdd(&a.stats->nt2, c.nt2);
}

template <int D>
__device__ __forceinline__ TaskDesc make_task(const Plan* pl, int i, uint16_t task, uint32_t Cpar)
{
    TaskDesc t;
    t.i = i;
    t.j = task & 63;
    t.l = (task >> 6) & 63;
    t.t1 = (task >> 12) & 1;
    t.t2 = (task >> 13) & 1;
    t.Cpar = Cpar;
    t.lg = max(0, t.l - Geo<D>::G);
    t.cs = D * (t.l - t.lg);
    t.npar = t.lg >= 2 ? Geo<D>::NPAR : (t.lg == 1 ? (1 << D) : 1);
    return t;
}

// process (or queue) every batch of a task
template <int D, int SCHEME, bool STATS>
__device__ __forceinline__ void do_task(const SampleArgs& a, WarpSmem<D>& W, const TaskDesc& t, uint16_t task,
                                        unsigned& fill, Counters& C)
{
    int nchild;
    setup_task<D>(a, W, t, nchild);
    for (int c0 = 0, b = 0; c0 < nchild; c0 += Geo<D>::CB, ++b) {
        const int nc = min(Geo<D>::CB, nchild - c0);
        unsigned long long work;
        const unsigned long long U = setup_batch<D, SCHEME>(a, W, t, c0, nc, work);
        if (STATS && lane_id() == 0)
            for (int s = 0; s < nc * 3; ++s)
                if (s % 3 && W.seq[s / 3][s % 3].units) ++C.ev2;
        if (U == 0) continue;
        if (work > BIG_WORK) {  // too much for one warp: queue unit ranges for k_big
            if (lane_id() == 0) {
                const unsigned long long per = max(1ull, U * ITEM_WORK / work);
                const unsigned long long nit = (U + per - 1) / per;
                const unsigned base = atomicAdd(a.nitems, (unsigned)min(nit, 0xFFFFFFFFull));
                if ((unsigned long long)base + nit > a.items_cap) {
                    atomicOr(a.err, ERR_ITEMS);
                } else {
                    for (unsigned long long k = 0; k < nit; ++k) {
                        BigItem it;
                        it.Cpar = t.Cpar;
                        it.task = task;
                        it.i = (uint8_t)t.i;
                        it.batch = (uint8_t)b;
                        it.lo = k * per;
                        it.hi = min(U, (k + 1) * per);
                        a.items[base + k] = it;
                    }
                }
            }
            __syncwarp();
            continue;
        }
        run_units<D, SCHEME, STATS>(a, W, t, nc, 0, U, fill, C);
    }
}

// persistent warps pull tiles of 32 sorted points; each point's owned tasks are processed by
// the whole warp, one task at a time
template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB) k_sample(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    const Plan* pl = a.pl;
    const unsigned lane = lane_id();
    unsigned fill = 0;
    Counters C = {};
    for (;;) {
        unsigned tile = 0;
        if (lane == 0) tile = atomicAdd(a.tile_ctr, 1u);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= a.ntiles) break;
        const uint32_t p = tile * 32 + lane;
        int i = 0, lf = 255;
        uint32_t code = 0;
        if (p < a.n) {
            int lo = 0, hi = pl->L - 1;  // layer: last with lstart <= p
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (pl->lstart[mid] <= p) lo = mid;
                else hi = mid - 1;
            }
            i = lo;
            code = __ldg(&a.skey[p]) - pl->base[i];
            lf = 0;  // coarsest level on which p is the first point of its cell
            if (p != pl->lstart[i]) {
                const uint32_t xr = code ^ (__ldg(&a.skey[p - 1]) - pl->base[i]);
                lf = xr == 0 ? 255 : (int)pl->I[i] - (31 - __clz(xr)) / D;
            }
        }
        const uint32_t cnt = lf == 255 ? 0u : pl->tcnt[i * 33 + lf];
        uint32_t total;
        const uint32_t start = warp_excl_scan(cnt, total);
        for (uint32_t tk = 0; tk < total; ++tk) {
            const unsigned own = __ballot_sync(0xffffffffu, cnt > 0 && start <= tk);
            const int ol = 31 - __clz(own);
            const int oi = __shfl_sync(0xffffffffu, i, ol);
            const int olf = __shfl_sync(0xffffffffu, lf, ol);
            const uint32_t ocode = __shfl_sync(0xffffffffu, code, ol);
            const uint32_t ostart = __shfl_sync(0xffffffffu, start, ol);
            GCHK(pl->toff[oi * 33 + olf] + (tk - ostart) < a.ntasks);
            const uint16_t task = __ldg(&a.tasks[pl->toff[oi * 33 + olf] + (tk - ostart)]);
            const int lg = max(0, ((task >> 6) & 63) - Geo<D>::G);
            const uint32_t Cpar = ocode >> (D * ((int)pl->I[oi] - lg));
            const TaskDesc t = make_task<D>(pl, oi, task, Cpar);
            do_task<D, SCHEME, STATS>(a, W, t, task, fill, C);
        }
    }
    warp_flush(a, W.ebuf, fill);
    flush_counters<STATS>(a, C);
}

// big items: one warp per item (rebuilds the task's batch and runs its unit range)
template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB) k_big(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    unsigned fill = 0;
    Counters C = {};
    const unsigned nit = min(*a.nitems, a.items_cap);
    const unsigned nw = gridDim.x * Geo<D>::WPB;
    for (unsigned k = blockIdx.x * Geo<D>::WPB + (threadIdx.x >> 5); k < nit; k += nw) {
        const BigItem it = a.items[k];
        const TaskDesc t = make_task<D>(a.pl, it.i, it.task, it.Cpar);
        int nchild;
        setup_task<D>(a, W, t, nchild);
        const int c0 = it.batch * Geo<D>::CB;
        const int nc = min(Geo<D>::CB, nchild - c0);
        unsigned long long work;
        setup_batch<D, SCHEME>(a, W, t, c0, nc, work);
        run_units<D, SCHEME, STATS>(a, W, t, nc, it.lo, it.hi, fill, C);
    }
    warp_flush(a, W.ebuf, fill);
    flush_counters<STATS>(a, C);
}
