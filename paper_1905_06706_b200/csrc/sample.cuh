// sample.cuh -- K5: the GIRG sampling kernels (v2), included by girg.cu.
//
// Work decomposition:
//   * An event is (layer pair i <= j, level l, A cell of layer i, B cell of layer j, type):
//     type-I = neighbouring cells at l = CL(i,j) (Alg. 1 line 3), type-II = distant
//     cells with neighbouring parents at 2 <= l <= CL(i,j) (Alg. 1 lines 5-6, R2).
//     The sorted point p that is first in its A cell at level l owns the event (R16: i == j
//     -> A <= B, A < B for distant pairs), so every event is enumerated exactly once.
//   * k_sample: persistent blocks pull tiles of 256 sorted points.  Each thread enumerates the
//     events of its point with a resumable enumerator and pushes the nonempty ones into a
//     shared-memory queue; the block then processes the queued events as a flat list of units
//     (type-I: one candidate pair; type-II: one jump chain of <= C candidates) spread over all
//     threads, so hub cells and empty cells do not serialise a warp.  Events with more than
//     BIG1 candidates / BIG2 chains are split into items of a global queue for k_big.
//   * Edges are staged in shared memory and written with one global atomic per flush (>= 1536
//     edges), as coalesced 8-byte stores.
#pragma once
// (included by girg.cu inside namespace girg)

// GIRG_DEBUG builds (libgirg_debug.so) bounds-check every indexed access of the sampler
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

constexpr int SB = 256;                 // threads per block
constexpr int QCAP = 512;               // events per round
constexpr int STAGE_CAP = 3072;         // staged edges per block
constexpr int FLUSH_AT = 1536;          // flush threshold (headroom 1536 for one sub-round)
constexpr unsigned long long BIG1 = 4096;   // type-I: more candidates -> item queue
constexpr unsigned long long BIG2 = 64;     // type-II: more chains -> item queue
constexpr unsigned long long ITEM1 = 4096;  // candidates per item
constexpr unsigned long long ITEM2 = 256;   // chains per item
constexpr int ERR_ITEMS = 16;

struct Counters {
    unsigned long long cand1, ev2, chunks, draws, landings, edges1, edges2, nt1, nt2;
};

struct Event {
    uint32_t a0, nA, b0, nB;  // sorted-position ranges of V_i^A and V_j^B
    uint32_t A, B;            // cell codes at level l (type-II Philox key)
    uint32_t tag;             // type-I: 1 if (i == j && A == B); type-II: l | i<<5 | j<<11
    uint32_t meta;            // bit 31: type-II; bits 24-29: log2 chunk length; bits 0-23: table index
};

struct BigItem {
    Event ev;
    unsigned long long lo, hi;  // unit range
};

struct SampleArgs {
    const Plan* pl;
    const TabEntry* tab;
    const uint16_t* tasks;
    const uint32_t* skey;
    const double* sx;
    const double* sw;
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
    unsigned long long nP;     // entries of P (K+1)
    unsigned int ntab, ntasks;
};

struct Stage {
    uint2 buf[STAGE_CAP];
    unsigned int fill;
    unsigned long long base;
};

__device__ __forceinline__ void stage_emit(const SampleArgs& a, Stage& S, uint32_t u, uint32_t v)
{
    const uint2 e = make_uint2(min(u, v), max(u, v));
    const unsigned idx = atomicAdd(&S.fill, 1u);
    if (idx < (unsigned)STAGE_CAP) {
        S.buf[idx] = e;
    } else {  // rare: the stage overflowed within one sub-round
        const unsigned long long slot = atomicAdd(a.m, 1ull);
        if (slot < a.cap) a.edges[slot] = e;
    }
}

// Block-wide flush of the staged edges if at least `threshold` are staged.  Call after a
// __syncthreads() (all emits done).  Every thread reads S.fill before thread 0 resets it (a
// barrier separates the two), so the decision -- and the barrier count -- is block-uniform.
__device__ __forceinline__ void stage_flush(const SampleArgs& a, Stage& S, unsigned threshold = 1)
{
    const unsigned f = S.fill;
    if (f < threshold) return;
    const unsigned c = min(f, (unsigned)STAGE_CAP);
    __syncthreads();
    if (threadIdx.x == 0) {
        S.base = atomicAdd(a.m, (unsigned long long)c);
        S.fill = 0;
    }
    __syncthreads();
    const unsigned long long b = S.base;
    for (unsigned k = threadIdx.x; k < c; k += blockDim.x) {
        const unsigned long long slot = b + k;
        if (slot < a.cap) a.edges[slot] = S.buf[k];
    }
    __syncthreads();
}

template <int D>
__device__ __forceinline__ void load_point(const SampleArgs& a, uint32_t p, double (&xp)[D])
{
    GCHK(p < a.n);
#pragma unroll
    for (int k = 0; k < D; ++k) xp[k] = __ldg(&a.sx[(size_t)k * a.n + p]);
}

// ---------------------------------------------------------------------------------------
// units
// ---------------------------------------------------------------------------------------
// type-I unit k of event e: candidate (s, t) = (k / nB, k % nB); same cell -> only s < t
template <int D, bool STATS>
__device__ __forceinline__ void type1_unit(const SampleArgs& a, Stage& S, const Event& e, unsigned long long k,
                                           Counters& c)
{
    const uint32_t s = (uint32_t)(k / e.nB);
    const uint32_t t = (uint32_t)(k - (unsigned long long)s * e.nB);
    if (e.tag && t <= s) return;
    const uint32_t pa = e.a0 + s, pb = e.b0 + t;
    GCHK(s < e.nA && t < e.nB);
    double xu[D], xv[D];
    load_point<D>(a, pa, xu);
    load_point<D>(a, pb, xv);
    const double wu = __ldg(&a.sw[pa]), wv = __ldg(&a.sw[pb]);
    const double Dp = dist_pow<D>(xu, xv);
    const Plan* pl = a.pl;
    if (STATS) ++c.cand1;
    bool edge;
    uint32_t u = 0, v = 0;
    if (pl->T == 0.0) {
        edge = Dp <= __dmul_rn(__dmul_rn(wu, wv), pl->s);
        if (edge) { u = __ldg(&a.sid[pa]); v = __ldg(&a.sid[pb]); }
    } else {
        const double p = prob_uv(wu, wv, pl->s, Dp, pl->invT);
        u = __ldg(&a.sid[pa]);
        v = __ldg(&a.sid[pb]);
        if (p >= 1.0) {
            edge = true;
        } else {
            const uint4 o = philox4x32_10(make_uint4(min(u, v), max(u, v), 0u, 3u), a.k0, a.k1);
            const double r = u53(o.x, o.y);
            if (STATS) c.nt1 += fabs(r - p) < 1e-12;
            edge = r < p;
        }
    }
    if (edge) {
        if (STATS) ++c.edges1;
        stage_emit(a, S, u, v);
    }
}

// type-II unit = jump chain `ch` of event e (R10, R14)
template <int D, bool STATS>
__device__ __forceinline__ void type2_unit(const SampleArgs& a, Stage& S, const Event& e, unsigned long long ch,
                                           Counters& c)
{
    GCHK((e.meta & 0xFFFFFFu) < a.ntab);
    const TabEntry te = a.tab[e.meta & 0xFFFFFFu];
    const int cl2 = (int)((e.meta >> 24) & 63u);
    const unsigned long long N = (unsigned long long)e.nA * e.nB;
    const unsigned long long start = ch << cl2;
    const long long end = (long long)min(N, start + (1ull << cl2));
    long long pos = (long long)start - 1;
    const Plan* pl = a.pl;
    const uint32_t c2 = e.tag | ((uint32_t)ch << 17);
    if (STATS) ++c.chunks;
    for (uint32_t k = 0;; ++k) {
        const uint4 o = philox4x32_10(make_uint4(e.A, e.B, c2, k), a.k0, a.k1);
        if (STATS) ++c.draws;
        const double rj = u53(o.x, o.y), ra = u53(o.z, o.w);
        const double z = te.pbar == 1.0 ? 0.0 : __ddiv_rn(log(__dsub_rn(1.0, rj)), te.Lbar);
        const long long remaining = end - pos - 1;
        if (z >= (double)remaining) break;
        pos += 1 + (long long)z;
        if (STATS) ++c.landings;
        uint32_t s, t;
        if (e.nB == 1) {
            s = (uint32_t)pos;
            t = 0;
        } else if (N <= 0xFFFFFFFFull) {
            s = (uint32_t)pos / e.nB;
            t = (uint32_t)pos - s * e.nB;
        } else {
            s = (uint32_t)((unsigned long long)pos / e.nB);
            t = (uint32_t)((unsigned long long)pos - (unsigned long long)s * e.nB);
        }
        const uint32_t pa = e.a0 + s, pb = e.b0 + t;
        GCHK(s < e.nA && t < e.nB);
        double xu[D], xv[D];
        load_point<D>(a, pa, xu);
        load_point<D>(a, pb, xv);
        const double p = prob_uv(__ldg(&a.sw[pa]), __ldg(&a.sw[pb]), pl->s, dist_pow<D>(xu, xv), pl->invT);
        const double rp = __dmul_rn(ra, te.pbar);
        if (STATS) c.nt2 += fabs(rp - p) < 1e-12 * te.pbar;
        if (rp < p) {
            if (STATS) ++c.edges2;
            stage_emit(a, S, __ldg(&a.sid[pa]), __ldg(&a.sid[pb]));
        }
    }
}

template <int D, bool STATS>
__device__ __forceinline__ void run_unit(const SampleArgs& a, Stage& S, const Event& e, unsigned long long k,
                                         Counters& c)
{
    if (e.meta >> 31) type2_unit<D, STATS>(a, S, e, k, c);
    else type1_unit<D, STATS>(a, S, e, k, c);
}

__device__ __forceinline__ unsigned long long event_units(const Event& e)
{
    if (e.meta >> 31) {
        const unsigned long long N = (unsigned long long)e.nA * e.nB;
        return ((N - 1) >> ((e.meta >> 24) & 63u)) + 1;
    }
    return (unsigned long long)e.nA * e.nB;
}

// ---------------------------------------------------------------------------------------
// flattened enumeration: probe units
// ---------------------------------------------------------------------------------------
// A sorted point p that is the first point of its cell from level lf on owns the events of
// its A cells (R16).  Its tasks are host-listed per (layer, lf): type-I tasks (j, CL(i,j)),
// type-II tasks (j, l).  A task has PAD probe slots (one candidate B cell each); probe unit
// u = task * PAD + slot is one thread's work, so all threads of a warp share a task (d = 3)
// or a few neighbouring tasks (d = 1) and enumeration runs at full SIMT width.
template <int D>
struct Pads {
    static constexpr uint32_t P3 = D == 1 ? 3u : D == 2 ? 9u : D == 3 ? 27u : D == 4 ? 81u : 243u;
    static constexpr uint32_t P6 = D == 1 ? 6u : D == 2 ? 36u : D == 3 ? 216u : D == 4 ? 1296u : 7776u;
};

struct TileShared {
    uint32_t code[SB];     // Morton code of the point at I(layer)
    uint8_t layer[SB];
    uint8_t lf[SB];        // 255: the point owns no event
    uint32_t tstart[SB + 1];
};

__device__ __forceinline__ void vrange_l(const SampleArgs& a, int jj, uint32_t B, int lv, int D, uint32_t& lo,
                                         uint32_t& hi)
{
    const Plan* pl = a.pl;
    const int sh = D * ((int)pl->I[jj] - lv);
    const uint32_t b = pl->base[jj];
    GCHK(sh >= 0 && (unsigned long long)b + ((unsigned long long)(B + 1u) << sh) < a.nP);
    lo = __ldg(&a.P[b + (B << sh)]);
    hi = __ldg(&a.P[b + ((B + 1u) << sh)]);
    GCHK(lo <= hi && hi <= a.n);
}

// one probe unit of pass K (0: type-I, 1: type-II); returns true and fills ev for a nonempty event
template <int D, int K>
__device__ __forceinline__ bool probe(const SampleArgs& a, const TileShared& T, uint32_t tile, uint32_t u, Event& ev)
{
    constexpr uint32_t PAD = K == 0 ? Pads<D>::P3 : Pads<D>::P6;
    const Plan* pl = a.pl;
    const uint32_t t = u / PAD, o = u - t * PAD;
    unsigned lo = 0, hi = SB - 1;  // owner: last point with tstart <= t
    while (lo < hi) {
        const unsigned mid = (lo + hi + 1) >> 1;
        if (T.tstart[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    const int i = T.layer[lo], lf = T.lf[lo];
    GCHK(lf < 32 && t - T.tstart[lo] < pl->tcnt[K][i * 32 + lf]);
    GCHK(pl->toff[K][i * 32 + lf] + (t - T.tstart[lo]) < a.ntasks);
    const uint16_t task = __ldg(&a.tasks[pl->toff[K][i * 32 + lf] + (t - T.tstart[lo])]);
    const int j = task & 63, l = task >> 6;
    const int Ii = pl->I[i];
    const uint32_t A = T.code[lo] >> (D * (Ii - l));
    {   // shard ownership
        const unsigned long long b = l >= pl->sl ? ((unsigned long long)A >> (D * (l - pl->sl)))
                                                 : ((unsigned long long)A << (D * (pl->sl - l)));
        if (b < pl->blo || b >= pl->bhi) return false;
    }
    uint32_t ac[D];
    morton_decode<D>(A, ac);
    uint32_t B;
    int dm = 0;
    if (K == 0) {  // neighbours at CL(i,j); levels 0, 1: every cell (R8)
        if (l <= 1) {
            if (o >= (1u << (D * l))) return false;
            B = o;
        } else {
            const uint32_t mask = (1u << l) - 1u;
            uint32_t bc[D], r = o;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const uint32_t dk = r % 3u;
                r /= 3u;
                bc[k] = (ac[k] + dk - 1u) & mask;
            }
            B = morton_encode<D>(bc);
        }
        if (i == j && B < A) return false;
    } else {  // distant cells with neighbouring parents at level l (R2, R9)
        if (l == 2) {
            if (o >= (1u << (2 * D))) return false;
            B = o;
            uint32_t bc[D];
            morton_decode<D>(B, bc);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int g = abs((int)bc[k] - (int)ac[k]);
                dm = max(dm, min(g, 4 - g));
            }
        } else {
            const uint32_t mask = (1u << l) - 1u;
            uint32_t bc[D], r = o;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int off = (int)(r % 6u) - 2 - (int)(ac[k] & 1u);
                r /= 6u;
                dm = max(dm, abs(off));
                bc[k] = (ac[k] + (uint32_t)off) & mask;
            }
            B = morton_encode<D>(bc);
        }
        if (dm <= 1) return false;
        if (i == j && B <= A) return false;
    }
    uint32_t b0, b1;
    vrange_l(a, j, B, l, D, b0, b1);
    if (b1 == b0) return false;
    const uint32_t p = tile * SB + lo;
    const int sh = D * (Ii - l);
    GCHK(sh >= 0 && (unsigned long long)pl->base[i] + ((unsigned long long)(A + 1u) << sh) < a.nP);
    const uint32_t a1 = __ldg(&a.P[pl->base[i] + ((A + 1u) << sh)]);
    GCHK(__ldg(&a.P[pl->base[i] + (A << sh)]) == p && a1 > p && a1 <= a.n);
    ev.a0 = p;
    ev.nA = a1 - p;
    ev.b0 = b0;
    ev.nB = b1 - b0;
    ev.A = A;
    ev.B = B;
    if (K == 0) {
        ev.tag = (i == j && A == B) ? 1u : 0u;
        ev.meta = 0u;
        return true;
    }
    const uint32_t ti = pl->tab_off[i * MAXL + j] + 2u * (uint32_t)(l - 2) + (uint32_t)(dm - 2);
    GCHK(ti < a.ntab && dm <= 3);
    const TabEntry te = a.tab[ti];
    if (te.pbar == 0.0) return false;
    const unsigned long long N = (unsigned long long)ev.nA * ev.nB;
    int cl2 = te.clog2;
    while (((N - 1) >> cl2) >= (1ull << 15)) ++cl2;
    ev.tag = (uint32_t)l | ((uint32_t)i << 5) | ((uint32_t)j << 11);
    ev.meta = (1u << 31) | ((uint32_t)cl2 << 24) | ti;
    return true;
}

// push a big event as items of <= ITEM units; false if the item queue is full
__device__ __forceinline__ void push_items(const SampleArgs& a, const Event& e, unsigned long long units)
{
    const unsigned long long per = (e.meta >> 31) ? ITEM2 : ITEM1;
    const unsigned long long nit = (units + per - 1) / per;
    const unsigned int base = atomicAdd(a.nitems, (unsigned int)min(nit, 0xFFFFFFFFull));
    if ((unsigned long long)base + nit > a.items_cap) {
        atomicOr(a.err, ERR_ITEMS);
        return;
    }
    for (unsigned long long k = 0; k < nit; ++k) {
        BigItem it;
        it.ev = e;
        it.lo = k * per;
        it.hi = min(units, (k + 1) * per);
        a.items[base + k] = it;
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

template <int D, bool STATS>
__device__ __forceinline__ void process_queue(const SampleArgs& a, Stage& S, Event* q, uint32_t* uoff,
                                              uint32_t* sh_scan, unsigned nq, Counters& c)
{
    // exclusive scan of the units of the queued events (2 per thread)
    {
        const unsigned e0 = 2 * threadIdx.x, e1 = e0 + 1;
        const uint32_t u0 = e0 < nq ? (uint32_t)event_units(q[e0]) : 0u;
        const uint32_t u1 = e1 < nq ? (uint32_t)event_units(q[e1]) : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(u0 + u1, sh_scan, tot);
        if (e0 <= nq) uoff[e0] = ex;
        if (e1 <= nq) uoff[e1] = ex + u0;
        if (threadIdx.x == 0) uoff[nq] = tot;  // nq == QCAP is not covered by e0/e1
    }
    __syncthreads();
    const uint32_t total = uoff[nq];
    for (uint32_t base = 0; base < total; base += SB) {
        const uint32_t u = base + threadIdx.x;
        if (u < total) {
            unsigned lo = 0, hi = nq - 1;  // last event with uoff <= u
            while (lo < hi) {
                const unsigned mid = (lo + hi + 1) >> 1;
                if (uoff[mid] <= u) lo = mid;
                else hi = mid - 1;
            }
#ifdef GIRG_DEBUG
            if (!(lo < nq && u - uoff[lo] < event_units(q[lo]))) {
                if (atomicExch(a.err, 1 << 20) == 0)
                    printf("bad unit: nq=%u lo=%u u=%u total=%u uoff[lo]=%u uoff[lo+1]=%u units=%llu uoff[nq]=%u\n", nq, lo, u,
                           total, uoff[lo], uoff[lo + 1], event_units(q[lo]), uoff[nq]);
                return;
            }
#endif
            run_unit<D, STATS>(a, S, q[lo], u - uoff[lo], c);
        }
        __syncthreads();
        stage_flush(a, S, FLUSH_AT);
    }
}

#ifndef GIRG_SAMPLE_MINB
#define GIRG_SAMPLE_MINB 1
#endif
template <int D, bool STATS>
__global__ void __launch_bounds__(SB, GIRG_SAMPLE_MINB) k_sample(SampleArgs a)
{
    __shared__ Event q[QCAP];
    __shared__ uint32_t uoff[QCAP + 1];
    __shared__ uint32_t sh_scan[SB / 32];
    __shared__ Stage S;
    __shared__ TileShared T;
    __shared__ unsigned int qn, tile;
    if (threadIdx.x == 0) { S.fill = 0; qn = 0; }
    Counters c = {};
    const Plan* pl = a.pl;
    const int npass = pl->T > 0.0 ? 2 : 1;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) tile = atomicAdd(a.tile_ctr, 1u);
        __syncthreads();
        if (tile >= a.ntiles) break;
        // ---- point info of the tile ----
        {
            const uint32_t p = tile * SB + threadIdx.x;
            uint8_t lf8 = 255;
            int i = 0;
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
                int lf = 0;  // coarsest level at which p is the first point of its cell
                bool owner = true;
                if (p != pl->lstart[i]) {
                    const uint32_t xr = code ^ (__ldg(&a.skey[p - 1]) - pl->base[i]);
                    if (xr == 0) owner = false;
                    else lf = (int)pl->I[i] - (31 - __clz(xr)) / D;
                }
                if (owner) lf8 = (uint8_t)lf;
            }
            T.code[threadIdx.x] = code;
            T.layer[threadIdx.x] = (uint8_t)i;
            T.lf[threadIdx.x] = lf8;
        }
        for (int pass = 0; pass < npass; ++pass) {
            __syncthreads();
            {
                const int lf = T.lf[threadIdx.x];
                const uint32_t cnt = lf == 255 ? 0u : pl->tcnt[pass][T.layer[threadIdx.x] * 32 + lf];
                uint32_t tot;
                const uint32_t ex = block_exclusive_scan(cnt, sh_scan, tot);
                T.tstart[threadIdx.x] = ex;
                if (threadIdx.x == 0) T.tstart[SB] = tot;
            }
            __syncthreads();
            const uint32_t PU = T.tstart[SB] * (pass == 0 ? Pads<D>::P3 : Pads<D>::P6);
            uint32_t cursor = 0;
            while (cursor < PU) {
                // probe phase: QCAP/SB sub-steps of SB probe units, each pushing at most SB events.
                // The sub-step count depends only on the (uniform) cursor, never on qn, which
                // other warps may already be incrementing.
                for (int sub = 0; sub < QCAP / SB && cursor < PU; ++sub) {
                    const uint32_t u = cursor + threadIdx.x;
                    Event ev;
                    if (u < PU && (pass == 0 ? probe<D, 0>(a, T, tile, u, ev) : probe<D, 1>(a, T, tile, u, ev))) {
                        if (STATS && pass == 1) ++c.ev2;
                        const unsigned long long units = event_units(ev);
                        if (units > (pass ? BIG2 : BIG1)) push_items(a, ev, units);
                        else {
                            const unsigned slot = atomicAdd(&qn, 1u);
                            GCHK(slot < (unsigned)QCAP);
                            q[slot] = ev;
                        }
                    }
                    cursor += SB;
                    __syncthreads();
                }
                const unsigned nq = qn;
                if (nq) process_queue<D, STATS>(a, S, q, uoff, sh_scan, nq, c);
                __syncthreads();
                if (threadIdx.x == 0) qn = 0;
                __syncthreads();
            }
        }
    }
    __syncthreads();
    stage_flush(a, S);
    flush_counters<STATS>(a, c);
}

// big items: one block per item, units spread over the threads
template <int D, bool STATS>
__global__ void __launch_bounds__(SB) k_big(SampleArgs a)
{
    __shared__ Stage S;
    __shared__ BigItem it;
    if (threadIdx.x == 0) S.fill = 0;
    Counters c = {};
    const unsigned nit = min(*a.nitems, a.items_cap);
    for (unsigned k = blockIdx.x; k < nit; k += gridDim.x) {
        __syncthreads();
        if (threadIdx.x == 0) it = a.items[k];
        __syncthreads();
        const Event e = it.ev;
        for (unsigned long long base = it.lo; base < it.hi; base += SB) {
            const unsigned long long u = base + threadIdx.x;
            if (u < it.hi) run_unit<D, STATS>(a, S, e, u, c);
            __syncthreads();
            stage_flush(a, S, FLUSH_AT);
        }
    }
    __syncthreads();
    stage_flush(a, S);
    flush_counters<STATS>(a, c);
}
