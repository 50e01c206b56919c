// sample.cuh -- K5: the GIRG sampling kernels (v5), included by girg.cu inside namespace girg.
//
// Events (Algorithm 1; R2, R16): for a layer pair i <= j, a neighbouring cell pair
// (A, B) on level CL(i,j) is a type-I event (every candidate tested, Alg. 1 line 3), a distant
// cell pair with neighbouring parents on a level 2 <= l <= CL(i,j) is a type-II event (geometric
// jumps under the bound pbar, Alg. 1 lines 5-6).
//
// Work decomposition:
//   * job = (layer i, partner j, level l, task cell Cg of layer i on level lg = max(0, l - G)):
//     the level-l descendants A of Cg ("children") against the "region" = the level-l
//     descendants of the 3^d neighbours of Cg (of all level-lg cells when lg <= 1), which holds
//     every neighbour and every distant cell with neighbouring parents of each child.  A job is
//     owned by the first sorted point of Cg; host tables list the jobs of a point by (layer,
//     first level lf).  G = 3 for d = 1 (8 children per job), else 1.
//   * one warp per job: lanes load the region's Lemma-1 ranges (P entries) once, classify every
//     (child, region parent) pair in parallel into bit masks of kinds (0: neighbour / type-I,
//     1: distant with delta_max = 2, 2: delta_max = 3), and prefix-sum the counts in Morton
//     order of the region cells.
//   * units: a type-I candidate pair, or one chunk (jump chain) of a type-II sequence.  A
//     sequence is one distant cell pair (scheme EVENT, Alg. 1 as written) or the concatenation of
//     all distant cells of A with the same bound class (scheme MERGED, R22).
//   * engine: NSLOT job slots per warp.  Lanes pull units of the dispatch slot and advance one
//     Philox draw / one candidate per step; when the dispatch slot runs dry the warp sets up the
//     next job in a slot no lane is still working on, while lanes finish earlier jobs' chains,
//     so jobs pipeline and short jobs do not leave the warp idle.
//   * jobs with too much work are split into unit-range items of a global queue (k_big).
//   * edges are staged per warp in shared memory and written with one atomic per flush.
#pragma once
#include <type_traits>

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

constexpr int SCHEME_EVENT = 0, SCHEME_MERGED = 1, SCHEME_REFINED = 2;
// index of a type-II kind (1, 2) in the JobInfo bound arrays: kind - KOFF.  The REFINED
// instantiation (R27) stores them at [kind], because a refined job's three kinds 0..2 are all
// jump-chain sequences (classes h = 2, 3, >= 4) with bounds at [0..2].
template <int SCHEME>
struct KOff {
    static constexpr int v = SCHEME == SCHEME_REFINED ? 0 : 1;
};
// Unrolling of the job setup's shared-memory loops (runtime trip counts; nvcc unrolls them 4x by
// default).  The sampling kernels are instruction-fetch bound as much as issue bound (ncu C5:
// no_instructions is the top stall reason, the hot code is ~33 KB against a 32 KB L1.5 I$), so
// the setup loops stay rolled: fewer code bytes at a few more instructions per job.
#ifndef GIRG_SETUP_UNROLL
#define GIRG_SETUP_UNROLL 1
#endif
#define GIRG_STR2(x) #x
#define GIRG_STR(x) GIRG_STR2(x)
#if GIRG_SETUP_UNROLL > 0
#define SETUP_LOOP _Pragma(GIRG_STR(unroll GIRG_SETUP_UNROLL))
#else
#define SETUP_LOOP  // nvcc's default unrolling
#endif
#ifndef GIRG_ENGINE_T0
#define GIRG_ENGINE_T0 false
#endif
#ifndef GIRG_EB
#define GIRG_EB 128
#endif
#ifndef GIRG_EB3
#define GIRG_EB3 64
#endif
// weighted units (a chunk counts 8) above which a job is queued for k_big, and per queued item
// Jobs with more units than big_work are queued for k_big in items of item_work units (B200
// sweeps, profiles/r01/SUMMARY.md; d = 1 splits finer on small graphs, which have fewer jobs
// per warp: C2 512 / 256 3.16 ms vs 1024 / 512 3.51 ms, C4 the other way round 25.1 vs 23.5 ms).
__host__ __device__ constexpr unsigned long long big_work(int d, unsigned long long n)
{
    return d == 1 ? (n >= (1ull << 22) ? 1024ull : 512ull) : (d == 2 ? 1024ull : (d == 3 ? 16384ull : 32768ull));
}
__host__ __device__ constexpr unsigned long long item_work(int d, unsigned long long n) { return big_work(d, n) / 2; }
constexpr int ERR_ITEMS = 16;
constexpr unsigned FULL = 0xffffffffu;

// Tuning knobs (compile-time; the defaults are the B200 sweep optima recorded in
// profiles/r01/SUMMARY.md; tools/sweep_*.sh rebuild variants with -D to re-tune):
//   GIRG_G1      d = 1 task height: a job covers the 2^G1 level-l cells below one task cell
//   GIRG_G2      d = 2 task height (2 is parity-green but leaves the separable classification
//                and doubles the slot: C3 9.8 -> 22-34 ms; kept at 1)
//   GIRG_NSLOT1  d = 1 job slots per warp;  GIRG_MINB1  d = 1 resident blocks per SM
//   GIRG_WPB3    d = 3 warps per block;     GIRG_NSLOT3 / GIRG_MINB3  d = 3 slots / blocks per SM
//   GIRG_WPB1    d = 1 warps per block (d = 1 runs 5 blocks x 4 warps with 2 job slots: 96
//                registers, 9.4 KB shared memory per warp; 2 x 8 warps with 3 slots: C4 23.5 ms
//                vs 22.1 ms; 24 warps at 80 registers: slower)
//   GIRG_CB3     d = 3 children per job (8 = all; 4 halves the slot but doubles the job setups:
//                C5 214 ms at 5 blocks, 240 ms at 6 blocks / 80 registers, vs 164 ms)
//   GIRG_EB / GIRG_EB3  staged edges per warp (d != 3 / d = 3);  GIRG_MINB2 / GIRG_NSLOT2  d = 2 blocks per SM / job slots
//   (d = 3: 5 blocks of 4 warps need <= 96 registers AND <= 45 KB of shared memory per block,
//    hence the 64-entry staging buffer: 164 vs 176 ms on C5; 5 blocks without it stay at 4
//    resident blocks with the 96-register cap and run slower, 186 ms)
// GIRG_PROFILE adds per-warp cycle / job / iteration counters (GIRG_WARP_PROFILE dumps them).
#ifndef GIRG_G2
#define GIRG_G2 1
#endif

#ifndef GIRG_G1
#define GIRG_G1 4
#endif
#ifndef GIRG_NSLOT1
#define GIRG_NSLOT1 2
#endif
#ifndef GIRG_WPB3
#define GIRG_WPB3 4
#endif
#ifndef GIRG_MINB1
#define GIRG_MINB1 5
#endif
#ifndef GIRG_NSLOT3
#define GIRG_NSLOT3 2
#endif
#ifndef GIRG_MINB2
#define GIRG_MINB2 4
#endif
#ifndef GIRG_NSLOT2
#define GIRG_NSLOT2 4
#endif
#ifndef GIRG_WPB1
#define GIRG_WPB1 4
#endif
#ifndef GIRG_CB3
#define GIRG_CB3 8
#endif
#ifndef GIRG_MINB3
#define GIRG_MINB3 5
#endif
#ifndef GIRG_MINB3_BIG
#define GIRG_MINB3_BIG GIRG_MINB3
#endif
template <int D>
struct Geo {
    static constexpr int G = D == 1 ? GIRG_G1 : (D == 2 ? GIRG_G2 : 1);  // levels between a task cell and its children
    static constexpr int NCH = 1 << (D * G);                 // children (= sub-cells per region parent)
    static constexpr int NPAR = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : 243;  // 3^d
    static constexpr int MAXPAR = NPAR > (1 << D) ? NPAR : (1 << D);  // lg = 1: all 2^d level-1 cells
    static constexpr int CB = D <= 2 ? NCH : (D == 3 ? GIRG_CB3 : (D == 4 ? 4 : 2));  // children per job (batch)
    static constexpr int WPB = D == 1 ? GIRG_WPB1 : (D == 2 ? 8 : (D == 3 ? GIRG_WPB3 : 2));  // warps per block
    static constexpr int MINB = D == 1 ? GIRG_MINB1 : (D == 2 ? GIRG_MINB2 : (D == 3 ? GIRG_MINB3 : 1));  // resident blocks per SM
    static constexpr int MINB_BIG = D == 3 ? GIRG_MINB3_BIG : MINB;  // the same for k_big (its own register budget)
    static constexpr int EB = D == 3 ? GIRG_EB3 : GIRG_EB;  // staged edges per warp (d = 3: small, so 5 blocks fit)
    static constexpr int NSLOT = D == 1 ? GIRG_NSLOT1 : (D == 2 ? GIRG_NSLOT2 : (D == 3 ? GIRG_NSLOT3 : 2));  // job slots per warp
    static constexpr int RECW = D == 1 ? 2 : (D <= 3 ? 4 : 6);       // doubles per point record
};

template <int N>
struct MaskOf {
    using T = uint32_t;
};
template <>
struct MaskOf<8> {
    using T = uint8_t;
};
template <>
struct MaskOf<4> {
    using T = uint8_t;
};
template <>
struct MaskOf<16> {
    using T = uint16_t;
};

struct Counters {
    unsigned long long cand1, ev2, chunks, draws, landings, edges1, edges2, nt1, nt2, fb, mm, ntj;
};

// one (child, kind) sequence of a job (its unit count is the difference of the slot's uoff)
struct Seq {
    uint32_t A, a0, nA, M;  // child cell, its sorted range, candidates per row (kind 0 / merged)
    int cl2;                // log2 chunk length (merged)
};

struct BigItem {
    uint32_t Cpar;
    uint16_t task;  // j | l<<6 | t1<<12 | t2<<13
    uint8_t i, batch;
    unsigned long long lo, hi;  // unit range of the job
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
    uint32_t tile_pts;  // sorted points per tile (32; fewer for small graphs: more warps in flight)
    uint32_t k0, k1;
    uint2* edges;
    unsigned long long cap;
    unsigned long long* m;
    unsigned int* tile_ctr;
    BigItem* items;
    unsigned int* nitems;
    unsigned int* item_ctr;  // k_big's dynamic item counter (zeroed with the status block)
    unsigned int items_cap;
    Counters* stats;
    int* err;
    unsigned long long nP;
    unsigned int ntab, ntasks;
    unsigned long long big_work, item_work;  // job split thresholds (BIG_WORK / ITEM_WORK by default)
    unsigned long long* wprof;               // optional per-warp profile: cycles, jobs, iterations, lane steps
    unsigned dev_flags;                      // development (-DGIRG_PROFILE builds): 1 = set up jobs, skip units
    // copies of Plan scalars read in the hot loops: kernel parameters are instruction operands
    // (constant bank), a Plan field is a global load that register pressure makes the compiler repeat
    double T, s, invT;
    int sl;
    unsigned long long blo, bhi;
    uint32_t nranks, rank;  // interleaved ownership (nranks > 0), else the block range [blo, bhi)
    int sharded;            // not the whole graph (ranked, or a block range other than everything)
    uint32_t p0;            // batched calls: first sorted position of this graph in the shared index
};

struct TaskDesc {
    int i, j, l, t1, t2;
    int ref;           // R27 refined job (task bit 14): Cpar is the A cell on level l, its rows split by A's children
    uint32_t Cpar;     // the task cell Cg, on level lg = max(0, l - G)
    int lg, npar, cs;  // task level, region parents, child shift d (l - lg)
};

// per-job constants read by the lanes
struct JobInfo {
    double pbar[3], Lbar[3];  // type-II bounds of kinds 1, 2 (R9) at [kind - KOff]; a refined job's classes at [0..2] (R27)
    double il2[3];            // 1 / log2(1 - pbar) (fast jump path)
    int clog2[2];             // EVENT chunk length (R10)
    int clog2m[3];            // MERGED / REFINED chunk length (R22)
    uint32_t tag;             // l | i<<5 | j<<11 (REFINED instantiation: + the scheme bits, so that the
                              // Philox tag word is tag + (kind << 17))
    int npar, cs, same_layer;
    int ref;                  // refined job (REFINED instantiation only)
};

template <int D>
struct Slot {
    static constexpr int NPAR = Geo<D>::MAXPAR, NCH = Geo<D>::NCH, CB = Geo<D>::CB;
    using MaskT = typename MaskOf<NCH>::T;
    uint32_t par[NPAR];              // region parent codes on level lg, Morton order
    uint32_t rstart[NPAR][NCH + 1];  // sorted positions of the region sub-cells (layer j)
    uint32_t achild[NCH + 1];        // sorted positions of Cg's children (layer i)
    uint32_t pre[CB][3][NPAR + 1];   // per (child, kind): prefix over parents (candidates / chunks)
    MaskT mask[CB][3][NPAR];         // per (child, kind, parent): sub-cells of that kind
    Seq seq[CB][3];
    unsigned long long uoff[CB * 3 + 1];  // unit offsets of the (child, kind) sequences
    JobInfo job;
    uint8_t child[NCH];  // nonempty owned children of Cg
};

// d = 1 job slot (lane per child): each child's sequences are <= 3 cell ranges per kind
// (neighbours a-1..a+1; distant a-2, a+2; the one of a-3, a+3 whose parent neighbours A's), kept
// explicitly in Morton (= coordinate) order instead of per-parent masks and prefix counts.
struct Slot1 {
    static constexpr int NPAR = 3, NCH = Geo<1>::NCH, CB = Geo<1>::CB;
    uint32_t par[NPAR];
    uint32_t rstart[NPAR][NCH + 1];
    uint32_t achild[NCH + 1];
    uint32_t rs[CB][3][3];  // range starts (sorted positions in layer j)
    uint32_t rn[CB][3][3];  // range lengths
    uint32_t rc[CB][3][4];  // cumulative units before each range (candidates; EVENT type-II: chunks)
    uint32_t rb[CB][3][3];  // cell codes
    Seq seq[CB][3];
    unsigned long long uoff[CB * 3 + 1];
    JobInfo job;
    uint8_t child[NCH];
};

template <int D>
using SlotT = typename std::conditional<D == 1, Slot1, Slot<D>>::type;

template <int D>
struct WarpSmem {
    SlotT<D> slot[Geo<D>::NSLOT];
    uint2 ebuf[Geo<D>::EB];
};

// ---------------------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned long long shfl_up64(unsigned long long v, int o)
{
    const uint32_t lo = __shfl_up_sync(FULL, (uint32_t)v, o), hi = __shfl_up_sync(FULL, (uint32_t)(v >> 32), o);
    return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src)
{
    const uint32_t lo = __shfl_sync(FULL, (uint32_t)v, src), hi = __shfl_sync(FULL, (uint32_t)(v >> 32), src);
    return ((unsigned long long)hi << 32) | lo;
}

// inclusive warp scan of 64-bit values
__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long v)
{
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = shfl_up64(v, o);
        if (lane >= (unsigned)o) v += y;
    }
    return v;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total)
{
    const unsigned lane = lane_id();
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    total = __shfl_sync(FULL, x, 31);
    return x - v;
}

// write the warp's staged edges (out of line: once per ~EB edges, keeps the engine loop small)
__device__ __noinline__ void warp_flush_n(const SampleArgs& a, const uint2* buf, unsigned fill)
{
    __syncwarp();
    unsigned long long base = 0;
    if (lane_id() == 0 && fill) base = atomicAdd(a.m, (unsigned long long)fill);
    base = shfl64(base, 0);
    for (unsigned k = lane_id(); k < fill; k += 32) {
        const unsigned long long slot = base + k;
        if (slot < a.cap) a.edges[slot] = buf[k];
    }
    __syncwarp();
}

// landing lookup inside a region parent: one predicated pass over its sub-cells (1) instead of
// the divergent walk over the mask bits (0); C5 sampling 156.9 -> 150.2 ms, C3 9.56 -> 9.33
#ifndef GIRG_LOCATE_PRED
#define GIRG_LOCATE_PRED 1
#endif
#ifndef GIRG_T0_ROLL
#define GIRG_T0_ROLL 0  // the flat T = 0 loop keeps its per-candidate sequence scan unrolled (rolled: n = 2^24 d = 1 10.9 -> 14.1 ms)
#endif
#ifndef GIRG_FLUSH_CALL
#define GIRG_FLUSH_CALL 0  // 1: out-of-line flush (C4 -1 %, but C3 +6 %, C5 +0.5 %: the call perturbs the 64-register d = 2 engine)
#endif
__device__ __forceinline__ void warp_flush(const SampleArgs& a, uint2* buf, unsigned& fill)
{
#if GIRG_FLUSH_CALL
    warp_flush_n(a, buf, fill);
#else
    __syncwarp();
    unsigned long long base = 0;
    if (lane_id() == 0 && fill) base = atomicAdd(a.m, (unsigned long long)fill);
    base = shfl64(base, 0);
    for (unsigned k = lane_id(); k < fill; k += 32) {
        const unsigned long long slot = base + k;
        if (slot < a.cap) a.edges[slot] = buf[k];
    }
    __syncwarp();
#endif
    fill = 0;
}

// append this lane's edge (if any); `fill` is warp-uniform
template <int CAP>
__device__ __forceinline__ void warp_emit(const SampleArgs& a, uint2* buf, unsigned& fill, bool edge, uint32_t u,
                                          uint32_t v)
{
    const unsigned em = __ballot_sync(FULL, edge);
    if (!em) return;
    const unsigned cnt = __popc(em);
    if (fill + cnt > (unsigned)CAP) warp_flush(a, buf, fill);
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

// ---- cold paths, out of line so that the engine loop stays small in the instruction cache ----
// canonical jump skip z = log(1-rj)/log1p(-pbar) (R10)
__device__ __noinline__ double exact_skip(double rj, double Lbar) { return __ddiv_rn(det_log(__dsub_rn(1.0, rj)), Lbar); }
// canonical p_uv (Eq. 1, kappa form)
__device__ __noinline__ double exact_prob(double wu, double wv, double s, double Dp, double invT)
{
    return prob_uv(wu, wv, s, Dp, invT);
}
// 64-bit quotient / remainder (rare: only for sequences of >= 2^32 candidates)
__device__ __noinline__ uint32_t divmod64(unsigned long long x, uint32_t m, uint32_t& rem)
{
    const unsigned long long q = x / m;
    rem = (uint32_t)(x - q * m);
    return (uint32_t)q;
}
__device__ __forceinline__ uint32_t divmod(unsigned long long x, uint32_t m, uint32_t& rem)
{
    if (x < m) {  // the common case at fine levels: A holds one point, so every index is in row 0
        rem = (uint32_t)x;
        return 0u;
    }
    if (x <= 0xFFFFFFFFull) {
        const uint32_t q = (uint32_t)x / m;
        rem = (uint32_t)x - q * m;
        return q;
    }
    return divmod64(x, m, rem);
}

// chunk length (log2) of a type-II sequence of N candidates with table log2 length c0 and a
// cap of 2^capbits chunks (R10 / R22)
__device__ __forceinline__ int chunk_log2(unsigned long long N, int c0, int capbits)
{
    int c = c0;
    while (((N - 1) >> c) >= (1ull << capbits)) ++c;
    return c;
}

template <int D>
__device__ __forceinline__ TaskDesc make_task(int i, uint16_t task, uint32_t Cpar)
{
    TaskDesc t;
    t.i = i;
    t.j = task & 63;
    t.l = (task >> 6) & 63;
    t.t1 = (task >> 12) & 1;
    t.t2 = (task >> 13) & 1;
    t.ref = (task >> 14) & 1;
    t.Cpar = Cpar;
    t.lg = max(0, t.l - Geo<D>::G);
    t.cs = D * (t.l - t.lg);
    t.npar = t.lg >= 2 ? Geo<D>::NPAR : (t.lg == 1 ? (1 << D) : 1);
    return t;
}

// ---------------------------------------------------------------------------------------
// job setup (warp-collective): region, children, classification, sequences, unit offsets.
// Out of line (called once per job, keeps the engine loop's register allocation small).
// ---------------------------------------------------------------------------------------
struct JobSetup {
    unsigned long long U;     // units of the job
    unsigned long long work;  // weighted units (a chunk counts 8)
    int nchild;               // nonempty owned children of the task cell (all batches)
    int nseq2;                // nonempty type-II sequences (counter)
};

// Shard ownership of the events whose A cell (the job child) is A on level l, layer pair (i, j)
// (DESIGN.md "Multi-GPU").  Block range mode (nranks = 0): the Morton block of A at
// the split level sl in [blo, bhi) (a coarser A: the block of its first descendant).
// Interleaved mode (nranks > 0): rank = block mod nranks for l >= sl, and for the coarse events
// (l < sl, which would all fall to a few first-descendant blocks) rank = (A + 7 j + 13 i + 31 l)
// mod nranks, spreading them by identity.
template <int D>
__device__ __noinline__ bool owns(const SampleArgs& a, uint32_t A, int l, int i, int j)
{
    if (a.nranks == 0) {
        const unsigned long long b = l >= a.sl ? ((unsigned long long)A >> (D * (l - a.sl)))
                                               : ((unsigned long long)A << (D * (a.sl - l)));
        return b >= a.blo && b < a.bhi;
    }
    const uint32_t key = l >= a.sl ? (uint32_t)((unsigned long long)A >> (D * (l - a.sl)))
                                   : A + 7u * (uint32_t)j + 13u * (uint32_t)i + 31u * (uint32_t)l;
    return key % a.nranks == a.rank;
}

// ---- job setup, common part (warp-collective): region parents in Morton order, the Lemma-1
// ranges of their sub-cells (layer j) and of the task cell's children (layer i), the nonempty
// owned children of this batch, the job constants.  Returns the batch's child count.
template <int D, int SCHEME, class SL>
__device__ __forceinline__ int setup_common(const SampleArgs& a, SL& S, const TaskDesc& t, int batch, JobSetup& out,
                                            const TabEntry*& te)
{
    constexpr int CB = SL::CB;
    // R27 refined job (REFINED instantiation, task bit 14): t.Cpar is the A cell on level l; its
    // rows are A's children on level l + 1 (<= I(i)), the region is that of A's parent
    constexpr bool RS = SCHEME == SCHEME_REFINED;
    const bool ref = RS && t.ref;
    const uint32_t Cg = ref ? t.Cpar >> D : t.Cpar;  // centre of the region, on level lg
    const Plan* pl = a.pl;
    const unsigned lane = lane_id();
    const int nsub = 1 << t.cs;
    // sharded runs: a task cell on or below the split level lies in one shard block, so a job of
    // another shard is dropped before any setup work
    if (a.sharded && (ref ? t.l : t.lg) >= a.sl && !owns<D>(a, ref ? t.Cpar : t.Cpar << t.cs, t.l, t.i, t.j)) {
        out.nchild = 0;
        return 0;
    }
    // the type-II bounds of the job (lanes 0, 1: classes 2, 3), loaded before the region so that
    // their latency overlaps the region loads
    // (REFINED plans hold 5 entries per level: classes 2, 3 and the refined classes h = 2, 3, >= 4)
    constexpr uint32_t TS = RS ? 5u : 2u;
    const unsigned nte = ref ? 3u : 2u;
    te = t.t2 ? a.tab + (pl->tab_off[t.i * MAXL + t.j] + TS * (uint32_t)(t.l - 2) + (ref ? 2u : 0u)) : nullptr;
    TabEntry tev = {0.0, 0.0, 0, 0, 0.0, 0.0};
    if (te && lane < nte) tev = te[lane];
    // ---- region parents in Morton order ----
    if (t.lg >= 2) {
        uint32_t pc[D];
        morton_decode<D>(Cg, pc);
        const uint32_t mask = (1u << t.lg) - 1u;
        SETUP_LOOP
        for (int q = lane; q < t.npar; q += 32) {
            uint32_t c[D];
            int r = q;
#pragma unroll
            for (int k = D - 1; k >= 0; --k) {  // offsets in {-1,0,1}^d (distinct for lg >= 2; sorted below)
                c[k] = (pc[k] + (uint32_t)(r % 3) - 1u) & mask;
                r /= 3;
            }
            S.par[q] = morton_encode<D>(c);
        }
        __syncwarp();
        constexpr int NS = (Geo<D>::MAXPAR + 31) / 32;
        uint32_t mine[NS];
        int rk[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {  // rank sort
            const int q = lane + 32 * s;
            rk[s] = 0;
            mine[s] = q < t.npar ? S.par[q] : 0u;
            if (q < t.npar) {
                SETUP_LOOP
                for (int o = 0; o < t.npar; ++o) rk[s] += S.par[o] < mine[s];
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int q = lane + 32 * s;
            if (q < t.npar) S.par[rk[s]] = mine[s];
        }
    } else {
        for (int q = lane; q < t.npar; q += 32) S.par[q] = (uint32_t)q;  // lg = 1: all level-1 cells; lg = 0: root
    }
    __syncwarp();
    // ---- Lemma-1 ranges of the region sub-cells (layer j) and of Cg's children (layer i) ----
    {
        const int shj = D * ((int)pl->I[t.j] - t.l), shi = D * ((int)pl->I[t.i] - t.l - (ref ? 1 : 0));
        const uint32_t bj = pl->base[t.j], bi = pl->base[t.i];
        const int per = nsub + 1;
        constexpr int PER1 = Geo<D>::NCH + 1;  // per when l >= lg + G (the common case): a constant divisor
        for (int e = lane; e < t.npar * per + per; e += 32) {
            if (e < t.npar * per) {
                const int q = per == PER1 ? e / PER1 : e / per, k = e - q * per;
                const unsigned long long cell = ((unsigned long long)S.par[q] << t.cs) + (unsigned)k;
                GCHK(bj + (cell << shj) < a.nP);
                S.rstart[q][k] = __ldg(&a.P[bj + (cell << shj)]) - a.p0;
            } else {
                const int k = e - t.npar * per;
                const unsigned long long cell = ((unsigned long long)t.Cpar << t.cs) + (unsigned)k;
                GCHK(bi + (cell << shi) < a.nP);
                S.achild[k] = __ldg(&a.P[bi + (cell << shi)]) - a.p0;
            }
        }
    }
    __syncwarp();
    // ---- nonempty children owned by this shard (ownership by the A cell's block) ----
    {
        int cnt = 0;
        for (int c0 = 0; c0 < nsub; c0 += 32) {
            const int e = c0 + (int)lane;
            bool ok = false;
            if (e < nsub) {
                ok = S.achild[e + 1] > S.achild[e];
                const uint32_t A = ref ? t.Cpar : (t.Cpar << t.cs) + (uint32_t)e;
                ok = ok && (!a.sharded || owns<D>(a, A, t.l, t.i, t.j));
            }
            const unsigned bm = __ballot_sync(FULL, ok);
            const int rank = cnt + __popc(bm & ((1u << lane) - 1u));
            if (ok && rank >= batch * CB && rank < (batch + 1) * CB) S.child[rank - batch * CB] = (uint8_t)e;
            cnt += __popc(bm);
        }
        out.nchild = cnt;
    }
    const int nc = min(CB, out.nchild - batch * CB);
    if (nc <= 0) return 0;
    if (lane == 0) {
        JobInfo& J = S.job;
        J.tag = ((uint32_t)t.l | ((uint32_t)t.i << 5) | ((uint32_t)t.j << 11)) + (RS ? (ref ? (1u << 19) : (1u << 17)) : 0u);
        J.npar = t.npar;
        J.cs = t.cs;
        J.same_layer = t.i == t.j;
        J.ref = ref;
    }
    if (lane < nte) {
        JobInfo& J = S.job;
        const unsigned ix = ref ? lane : lane + 1u - (unsigned)KOff<SCHEME>::v;
        J.pbar[ix] = tev.pbar;
        J.Lbar[ix] = tev.Lbar;
        J.il2[ix] = tev.il2;
        if (lane < 2) J.clog2[lane] = tev.clog2;
        J.clog2m[ix] = tev.clog2m;
    }
    __syncwarp();
    return nc;
}

template <int D, int SCHEME>
__device__ __noinline__ JobSetup setup_job(const SampleArgs& a, Slot<D>& S, const TaskDesc t, int batch)
{
    JobSetup out = {0ull, 0ull, 0, 0};
    constexpr int NCH = Geo<D>::NCH, CB = Geo<D>::CB;
    using MaskT = typename Slot<D>::MaskT;
    const unsigned lane = lane_id();
    const int nsub = 1 << t.cs;
    const TabEntry* te = nullptr;
    const int nc = setup_common<D, SCHEME>(a, S, t, batch, out, te);
    if (nc <= 0) return out;
    // ---- phase 1: classify every (child, region parent) pair in parallel ----
    const int subl = t.cs / D;  // levels between a region parent and its sub-cells
    const uint32_t side = 1u << t.l, msk = side - 1u;
    const uint32_t side2 = side >> 1, msk2 = side2 - 1u;  // level l-1 (parent check, G > 1)
    const bool pcheck = Geo<D>::G > 1 && t.l >= 3;
    bool separable = false;  // classified by the separable path below
    if constexpr (Geo<D>::G == 1 && D <= 3) {
        if (t.l >= 1) {  // sub-cells = the 2^d children of each region parent: separable per dimension
            uint32_t cpc[D];  // coordinates of the task cell (level l-1)
            morton_decode<D>(t.Cpar, cpc);
            SETUP_LOOP
            for (int idx = lane; idx < nc * t.npar; idx += 32) {
                const int cc = idx / t.npar, q = idx - cc * t.npar;
                const int e = S.child[cc];
                const uint32_t P = S.par[q];
                uint32_t ac[D], pc[D], g0[D], g1[D];
#pragma unroll
                for (int k = 0; k < D; ++k) ac[k] = (cpc[k] << 1) | (((uint32_t)e >> (D - 1 - k)) & 1u);
                morton_decode<D>(P, pc);
#pragma unroll
                for (int k = 0; k < D; ++k) {  // torus gaps of the two children per dimension
                    const uint32_t d0 = ((pc[k] << 1) - ac[k]) & msk, d1 = ((pc[k] << 1) + 1u - ac[k]) & msk;
                    g0[k] = min(d0, side - d0);
                    g1[k] = min(d1, side - d1);
                }
                const int pcmp = P < t.Cpar ? -1 : (P > t.Cpar ? 1 : 0);  // Morton order of B vs A
                const uint32_t nA = S.achild[e + 1] - S.achild[e];
                uint32_t rs[NCH + 1];
#pragma unroll
                for (int k = 0; k <= NCH; ++k) rs[k] = S.rstart[q][k];
                uint32_t cnt[3] = {0u, 0u, 0u}, m[3] = {0u, 0u, 0u};
                if constexpr (SCHEME != SCHEME_EVENT) {
                    // Sub-cell sets as bit masks: {s : max_k gap_k(s) <= tau} is the AND over the
                    // dimensions of the sub-cells whose own gap in that dimension is <= tau.
                    constexpr uint32_t FULLN = (1u << NCH) - 1u;
                    uint32_t le1 = FULLN, le2 = FULLN;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        uint32_t p1 = 0u;
#pragma unroll
                        for (int sc = 0; sc < NCH; ++sc) p1 |= ((sc >> (D - 1 - k)) & 1) ? (1u << sc) : 0u;
                        const uint32_t p0 = FULLN ^ p1;
                        le1 &= (g0[k] <= 1u ? p0 : 0u) | (g1[k] <= 1u ? p1 : 0u);
                        le2 &= (g0[k] <= 2u ? p0 : 0u) | (g1[k] <= 2u ? p1 : 0u);
                    }
                    uint32_t GE = FULLN, GT = FULLN;  // sub-cells B with (i < j or B >= / > A)
                    if (!(t.i < t.j || pcmp > 0)) {
                        GE = pcmp < 0 ? 0u : (FULLN << e) & FULLN;
                        GT = pcmp < 0 ? 0u : (FULLN << (e + 1)) & FULLN;
                    }
                    m[0] = t.t1 ? (le1 & GE) : 0u;
                    m[1] = t.t2 ? (le2 & ~le1 & GT) : 0u;
                    m[2] = t.t2 ? (~le2 & GT & FULLN) : 0u;
#pragma unroll
                    for (int sc = 0; sc < NCH; ++sc) {
                        const uint32_t nB = rs[sc + 1] - rs[sc];
#pragma unroll
                        for (int kk = 0; kk < 3; ++kk) cnt[kk] += ((m[kk] >> sc) & 1u) ? nB : 0u;
                    }
                } else {
#pragma unroll
                for (int sc = 0; sc < NCH; ++sc) {
                    uint32_t dm = 0;
#pragma unroll
                    for (int k = 0; k < D; ++k) dm = max(dm, ((sc >> (D - 1 - k)) & 1) ? g1[k] : g0[k]);
                    const bool ge = pcmp > 0 || (pcmp == 0 && sc >= e), gt = pcmp > 0 || (pcmp == 0 && sc > e);
                    int kind = -1;
                    if (dm <= 1) {
                        if (t.t1 && (t.i < t.j || ge)) kind = 0;
                    } else if (t.t2 && (t.i < t.j || gt)) {
                        kind = (int)dm - 1;
                    }
                    const uint32_t nB = rs[sc + 1] - rs[sc];
                    uint32_t add = nB;
                    if (SCHEME == SCHEME_EVENT && kind > 0) {
                        add = 0;
                        if (nB && S.job.pbar[kind - 1] > 0.0) {
                            const unsigned long long N = (unsigned long long)nA * nB;
                            add = (uint32_t)(((N - 1) >> chunk_log2(N, S.job.clog2[kind - 1], 15)) + 1);
                        }
                    }
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk)
                        if (kk == kind) {
                            m[kk] |= 1u << sc;
                            cnt[kk] += add;
                        }
                }
                }
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    S.mask[cc][kk][q] = (MaskT)m[kk];
                    S.pre[cc][kk][q] = cnt[kk];
                }
            }
            separable = true;
        }
    }
    for (int idx = lane; !separable && idx < nc * t.npar; idx += 32) {
        const int cc = idx / t.npar, q = idx - cc * t.npar;
        const int e = S.child[cc];
        const uint32_t A = (t.Cpar << t.cs) + (uint32_t)e;
        uint32_t ac[D], pc[D];
        morton_decode<D>(A, ac);
        morton_decode<D>(S.par[q], pc);
        const uint32_t nA = S.achild[e + 1] - S.achild[e];
        uint32_t cnt[3] = {0u, 0u, 0u};
        uint32_t m[3] = {0u, 0u, 0u};
        // d = 1: only the sub-cells within 3 cells of the child can be neighbours or distant
        // cells with neighbouring parents; elsewhere every sub-cell of the parent may be
        int s_lo = 0, s_hi = nsub - 1;
        if (D == 1 && t.lg >= 2) {  // region = 3 parents of nsub cells, side >= 4 nsub: no wrap
            const int base = (int)((((pc[0] << subl) - ac[0] + (side >> 1)) & msk)) - (int)(side >> 1);  // offset of sub 0
            s_lo = max(0, -3 - base);
            s_hi = min(nsub - 1, 3 - base);
        }
#pragma unroll
        for (int s = 0; s < NCH; ++s) {
            if (s >= nsub) break;
            if (D == 1 && (s < s_lo || s > s_hi)) continue;
            uint32_t so[D];
            morton_decode<D>((uint32_t)s, so);
            uint32_t dm = 0, dp = 0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const uint32_t bk = ((pc[k] << subl) + so[k]) & msk;
                const uint32_t df = (bk - ac[k]) & msk;
                dm = max(dm, min(df, side - df));
                if (pcheck) {
                    const uint32_t df2 = ((bk >> 1) - (ac[k] >> 1)) & msk2;
                    dp = max(dp, min(df2, side2 - df2));
                }
            }
            const uint32_t B = (S.par[q] << t.cs) + (uint32_t)s;
            int kind = -1;
            if (dm <= 1) {
                if (t.t1 && (t.i < t.j || B >= A)) kind = 0;
            } else if (t.t2 && dp <= 1 && (t.i < t.j || B > A)) {
                kind = (int)dm - 1;  // 1: delta_max = 2, 2: delta_max = 3
            }
            if (kind < 0) continue;
            const uint32_t nB = S.rstart[q][s + 1] - S.rstart[q][s];
            uint32_t add = nB;
            if (SCHEME == SCHEME_EVENT && kind > 0) {  // chunks of the event (A, B)
                add = 0;
                if (nB && S.job.pbar[kind - 1] > 0.0) {
                    const unsigned long long N = (unsigned long long)nA * nB;
                    add = (uint32_t)(((N - 1) >> chunk_log2(N, S.job.clog2[kind - 1], 15)) + 1);
                }
            }
#pragma unroll
            for (int kk = 0; kk < 3; ++kk)
                if (kk == kind) {
                    m[kk] |= 1u << s;
                    cnt[kk] += add;
                }
        }
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
            S.mask[cc][kk][q] = (MaskT)m[kk];
            S.pre[cc][kk][q] = cnt[kk];
        }
    }
    __syncwarp();
    // ---- phase 2: per (child, kind): prefix over parents and the sequence (<= 2 per lane) ----
    constexpr int NE = (3 * CB + 31) / 32;
    unsigned long long units[NE];
#pragma unroll
    for (int h = 0; h < NE; ++h) {
        units[h] = 0;
        const int q3 = (int)lane + 32 * h;
        if (q3 < nc * 3) {
            const int cc = q3 / 3, k = q3 - 3 * cc;
            uint32_t acc = 0;
            SETUP_LOOP
            for (int q = 0; q < t.npar; ++q) {
                const uint32_t c = S.pre[cc][k][q];
                S.pre[cc][k][q] = acc;
                acc += c;
            }
            S.pre[cc][k][t.npar] = acc;
            const int e = S.child[cc];
            Seq& Q = S.seq[cc][k];
            Q.A = (t.Cpar << t.cs) + (uint32_t)e;
            Q.a0 = S.achild[e];
            Q.nA = S.achild[e + 1] - Q.a0;
            Q.M = acc;
            Q.cl2 = 0;
            if (k == 0) {
                units[h] = (unsigned long long)Q.nA * acc;
            } else if (SCHEME == SCHEME_EVENT) {
                units[h] = acc;
            } else if (acc && S.job.pbar[k - KOff<SCHEME>::v] > 0.0) {
                const unsigned long long N = (unsigned long long)Q.nA * acc;
                Q.cl2 = chunk_log2(N, S.job.clog2m[k - KOff<SCHEME>::v], 32);
                units[h] = ((N - 1) >> Q.cl2) + 1;
            }
        }
    }
    // ---- phase 3: unit offsets and weighted work ----
    unsigned long long base = 0, wk = 0;
    int n2 = 0;
#pragma unroll
    for (int h = 0; h < NE; ++h) {
        const int q3 = (int)lane + 32 * h;
        const bool kind0 = (q3 % 3) == 0;
        const unsigned long long incl = warp_incl_scan64(units[h]) + base;
        if (q3 < nc * 3) S.uoff[q3 + 1] = incl;
        base = shfl64(incl, 31);
        wk += units[h] * (kind0 ? 1ull : 8ull);
        n2 += __popc(__ballot_sync(FULL, !kind0 && units[h] != 0));
    }
    if (lane == 0) S.uoff[0] = 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) wk += __shfl_xor_sync(FULL, wk, o);
    out.work = wk;
    out.U = base;
    out.nseq2 = n2;
    __syncwarp();
    return out;
}

// R27 refined job (REFINED instantiation; R27: P:486-491 with a tighter minimum
// distance).  The task cell is the A cell on level l < CL(i,j); its rows are split by A's
// children a on level l + 1 (<= I(i)), and every distant cell B of A with a neighbouring parent
// (the region sub-cells that are not neighbours of A) is classed by its box distance from a in
// half-cells: h = max over the dimensions of the torus gap between a (one level-(l+1) cell) and
// B (two of them), kinds 0, 1, 2 = h 2, 3, >= 4.  One merged sequence (R22) per (a, class), its
// chunks keyed (a, chunk, l | i<<5 | j<<11 | class<<17 | 1<<19, draw).
template <int D>
__device__ __noinline__ JobSetup setup_job_ref(const SampleArgs& a, Slot<D>& S, const TaskDesc t, int batch)
{
    JobSetup out = {0ull, 0ull, 0, 0};
    constexpr int NCH = Geo<D>::NCH, CB = Geo<D>::CB;
    static_assert(Geo<D>::G == 1 && CB == NCH, "refined jobs: d = 2, 3");
    using MaskT = typename Slot<D>::MaskT;
    const unsigned lane = lane_id();
    const TabEntry* te = nullptr;
    const int nc = setup_common<D, SCHEME_REFINED>(a, S, t, batch, out, te);
    if (nc <= 0) return out;
    const uint32_t side = 1u << t.l, msk = side - 1u, S2 = side << 1, msk2 = S2 - 1u;
    uint32_t Ac[D];
    morton_decode<D>(t.Cpar, Ac);  // A, level l
    const uint32_t Cg = t.Cpar >> D;
    const int eA = (int)(t.Cpar & (uint32_t)(NCH - 1));  // A among its parent's children
    SETUP_LOOP
    for (int idx = lane; idx < nc * t.npar; idx += 32) {
        const int cc = idx / t.npar, q = idx - cc * t.npar;
        const int e = S.child[cc];
        const uint32_t P = S.par[q];
        uint32_t pc[D];
        morton_decode<D>(P, pc);
        const int pcmp = P < Cg ? -1 : (P > Cg ? 1 : 0);  // Morton order of B vs A
        uint32_t cnt[3] = {0u, 0u, 0u}, m[3] = {0u, 0u, 0u};
        // Sub-cell sets as bit masks, separable per dimension (as setup_job's MERGED path): nb =
        // neighbours of A, le2 / le3 = half-cell gap from a <= 2 / <= 3 (neighbours of A lie in le2)
        constexpr uint32_t FULLN = (1u << NCH) - 1u;
        uint32_t nb = FULLN, le2 = FULLN, le3 = FULLN;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            uint32_t p1 = 0u;
#pragma unroll
            for (int sc = 0; sc < NCH; ++sc) p1 |= ((sc >> (D - 1 - k)) & 1) ? (1u << sc) : 0u;
            const uint32_t p0 = FULLN ^ p1;
            const uint32_t a2 = (Ac[k] << 1) | (((uint32_t)e >> (D - 1 - k)) & 1u);  // a, level l + 1
            uint32_t sel_nb = 0u, sel2 = 0u, sel3 = 0u;
#pragma unroll
            for (int bit = 0; bit < 2; ++bit) {
                const uint32_t b = (pc[k] << 1) | (uint32_t)bit;  // B, level l
                const uint32_t df = (b - Ac[k]) & msk;
                const uint32_t dd = (2u * b - a2) & msk2;  // B = [dd, dd + 2) relative to a = [0, 1)
                const uint32_t g = (dd == 0u || dd == S2 - 1u) ? 0u : min(dd - 1u, S2 - dd - 2u);
                const uint32_t pm = bit ? p1 : p0;
                sel_nb |= min(df, side - df) <= 1u ? pm : 0u;
                sel2 |= g <= 2u ? pm : 0u;
                sel3 |= g <= 3u ? pm : 0u;
            }
            nb &= sel_nb;
            le2 &= sel2;
            le3 &= sel3;
        }
        uint32_t GT = FULLN;  // i == j: only B > A (R16)
        if (!(t.i < t.j || pcmp > 0)) GT = pcmp < 0 ? 0u : (FULLN << (eA + 1)) & FULLN;
        m[0] = le2 & ~nb & GT;
        m[1] = le3 & ~le2 & GT;
        m[2] = ~le3 & GT & FULLN;
#pragma unroll
        for (int sc = 0; sc < NCH; ++sc) {
            const uint32_t nB = S.rstart[q][sc + 1] - S.rstart[q][sc];
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) cnt[kk] += ((m[kk] >> sc) & 1u) ? nB : 0u;
        }
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
            S.mask[cc][kk][q] = (MaskT)m[kk];
            S.pre[cc][kk][q] = cnt[kk];
        }
    }
    __syncwarp();
    // per (child, class): prefix over parents and the sequence; every sequence is a chain sequence
    constexpr int NE = (3 * CB + 31) / 32;
    unsigned long long units[NE];
#pragma unroll
    for (int h = 0; h < NE; ++h) {
        units[h] = 0;
        const int q3 = (int)lane + 32 * h;
        if (q3 < nc * 3) {
            const int cc = q3 / 3, k = q3 - 3 * cc;
            uint32_t acc = 0;
            SETUP_LOOP
            for (int q = 0; q < t.npar; ++q) {
                const uint32_t c = S.pre[cc][k][q];
                S.pre[cc][k][q] = acc;
                acc += c;
            }
            S.pre[cc][k][t.npar] = acc;
            const int e = S.child[cc];
            Seq& Q = S.seq[cc][k];
            Q.A = (t.Cpar << D) + (uint32_t)e;  // a on level l + 1: the Philox key of its sequences
            Q.a0 = S.achild[e];
            Q.nA = S.achild[e + 1] - Q.a0;
            Q.M = acc;
            Q.cl2 = 0;
            if (acc && S.job.pbar[k] > 0.0) {
                const unsigned long long N = (unsigned long long)Q.nA * acc;
                Q.cl2 = chunk_log2(N, S.job.clog2m[k], 32);
                units[h] = ((N - 1) >> Q.cl2) + 1;
            }
        }
    }
    unsigned long long base = 0, wk = 0;
    int n2 = 0;
#pragma unroll
    for (int h = 0; h < NE; ++h) {
        const int q3 = (int)lane + 32 * h;
        const unsigned long long incl = warp_incl_scan64(units[h]) + base;
        if (q3 < nc * 3) S.uoff[q3 + 1] = incl;
        base = shfl64(incl, 31);
        wk += units[h] * 8ull;
        n2 += __popc(__ballot_sync(FULL, units[h] != 0));
    }
    if (lane == 0) S.uoff[0] = 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) wk += __shfl_xor_sync(FULL, wk, o);
    out.work = wk;
    out.U = base;
    out.nseq2 = n2;
    __syncwarp();
    return out;
}

// d = 1 job setup: one lane per child lists its <= 3 cell ranges per kind directly (offsets
// -3..3 from the child, or every region cell when the region is the whole level, lg <= 1).
template <int SCHEME>
__device__ __noinline__ JobSetup setup_job1(const SampleArgs& a, Slot1& S, const TaskDesc t, int batch)
{
    JobSetup out = {0ull, 0ull, 0, 0};
    const TabEntry* te = nullptr;
    const int nc = setup_common<1, SCHEME>(a, S, t, batch, out, te);
    if (nc <= 0) return out;
    const unsigned lane = lane_id();
    const int subl = t.cs, nsub = 1 << t.cs;  // d = 1: the shift is the level difference
    const uint32_t side = 1u << t.l, msk = side - 1u, side2 = side >> 1, msk2 = side2 - 1u;
    unsigned long long units[3] = {0ull, 0ull, 0ull};
    if ((int)lane < nc) {
        const int cc = (int)lane, e = S.child[cc];
        const uint32_t A = (t.Cpar << subl) + (uint32_t)e;
        const uint32_t a0 = S.achild[e], nA = S.achild[e + 1] - a0;
        uint32_t cb[3][3], cst[3][3], cn[3][3];
        int nk[3] = {0, 0, 0};
        const bool near = t.lg >= 2;  // l = lg + G >= 6: offsets -3..3 are distinct and inside the region
        const int ncand = near ? 7 : t.npar * nsub;
        SETUP_LOOP
        for (int c = 0; c < ncand; ++c) {
            uint32_t B;
            int q, kk;
            if (near) {
                B = (A + (uint32_t)(c - 3)) & msk;
                const uint32_t pb = B >> subl;
                q = pb == S.par[0] ? 0 : (pb == S.par[1] ? 1 : 2);
                kk = (int)(B & (uint32_t)(nsub - 1));
            } else {
                q = c / nsub;
                kk = c - q * nsub;
                B = (S.par[q] << subl) + (uint32_t)kk;
            }
            const uint32_t df = (B - A) & msk, dm = min(df, side - df);
            int kind = -1;
            if (dm <= 1) {
                if (t.t1 && (t.i < t.j || B >= A)) kind = 0;
            } else if (t.t2 && (t.i < t.j || B > A)) {
                bool pn = true;  // parents neighbours (the region may hold farther cells)
                if (t.l >= 3) {
                    const uint32_t d2 = ((B >> 1) - (A >> 1)) & msk2;
                    pn = min(d2, side2 - d2) <= 1;
                }
                if (pn) kind = (int)dm - 1;
            }
            if (kind < 0) continue;
            // insert by cell code (Morton order = coordinate order in d = 1)
            int m = nk[kind]++;
            const uint32_t st = S.rstart[q][kk], n = S.rstart[q][kk + 1] - st;
            while (m > 0 && cb[kind][m - 1] > B) {
                cb[kind][m] = cb[kind][m - 1];
                cst[kind][m] = cst[kind][m - 1];
                cn[kind][m] = cn[kind][m - 1];
                --m;
            }
            cb[kind][m] = B;
            cst[kind][m] = st;
            cn[kind][m] = n;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            uint32_t acc = 0;
            const int kb = k > 0 ? k - 1 : 0;  // this kind's bound (JobInfo; zero when !t2)
            for (int r = 0; r < nk[k]; ++r) {
                S.rs[cc][k][r] = cst[k][r];
                S.rn[cc][k][r] = cn[k][r];
                S.rb[cc][k][r] = cb[k][r];
                S.rc[cc][k][r] = acc;
                if (k == 0 || SCHEME == SCHEME_MERGED) {
                    acc += cn[k][r];
                } else if (cn[k][r] && S.job.pbar[kb] > 0.0) {  // EVENT: chunks of the event (A, B)
                    const unsigned long long N = (unsigned long long)nA * cn[k][r];
                    acc += (uint32_t)(((N - 1) >> chunk_log2(N, S.job.clog2[kb], 15)) + 1);
                }
            }
            S.rc[cc][k][nk[k]] = acc;
            Seq& Q = S.seq[cc][k];
            Q.A = A;
            Q.a0 = a0;
            Q.nA = nA;
            Q.M = acc;
            Q.cl2 = nk[k];  // merged chunk log2 set below; EVENT / type-I: unused
            if (k == 0) {
                units[k] = (unsigned long long)nA * acc;
            } else if (SCHEME == SCHEME_EVENT) {
                units[k] = acc;
            } else {
                Q.cl2 = 0;
                if (acc && S.job.pbar[kb] > 0.0) {
                    const unsigned long long N = (unsigned long long)nA * acc;
                    Q.cl2 = chunk_log2(N, S.job.clog2m[kb], 32);
                    units[k] = ((N - 1) >> Q.cl2) + 1;
                }
            }
        }
    }
    // unit offsets, sequence order (child, kind): lane cc's three sequences are consecutive
    const unsigned long long mine = units[0] + units[1] + units[2];
    const unsigned long long incl = warp_incl_scan64(mine);
    if ((int)lane < nc) {
        S.uoff[3 * lane + 1] = incl - mine + units[0];
        S.uoff[3 * lane + 2] = incl - mine + units[0] + units[1];
        S.uoff[3 * lane + 3] = incl;
    }
    if (lane == 0) S.uoff[0] = 0;
    unsigned long long wk = units[0] + 8ull * (units[1] + units[2]);
#pragma unroll
    for (int o = 16; o; o >>= 1) wk += __shfl_xor_sync(FULL, wk, o);
    out.work = wk;
    out.U = shfl64(incl, 31);
    out.nseq2 = __popc(__ballot_sync(FULL, units[1] != 0)) + __popc(__ballot_sync(FULL, units[2] != 0));
    __syncwarp();
    return out;
}

template <int D, int SCHEME>
__device__ __forceinline__ JobSetup setup_any(const SampleArgs& a, SlotT<D>& S, const TaskDesc t, int batch)
{
    if constexpr (D == 1) {
        return setup_job1<SCHEME>(a, S, t, batch);
    } else {
        if constexpr (SCHEME == SCHEME_REFINED)
            if (t.ref) return setup_job_ref<D>(a, S, t, batch);
        return setup_job<D, SCHEME>(a, S, t, batch);
    }
}

// d = 1 slot: the range holding concatenated index t of sequence (cc, k)
__device__ __forceinline__ uint32_t locate(const Slot1& S, int npar, int cs, int cc, int k, uint32_t t, uint32_t& B)
{
    (void)npar;
    (void)cs;
    int r = 0;
    while (r < 2 && S.rc[cc][k][r + 1] <= t) ++r;
    B = S.rb[cc][k][r];
    return S.rs[cc][k][r] + (t - S.rc[cc][k][r]);
}

__device__ __forceinline__ void locate_event(const Slot1& S, int clog2, int npar, int cs, int cc, int k, uint32_t nA,
                                             uint32_t u, uint32_t& B, uint32_t& b0, uint32_t& nB, uint32_t& ch,
                                             int& cl2)
{
    (void)npar;
    (void)cs;
    int r = 0;
    while (r < 2 && S.rc[cc][k][r + 1] <= u) ++r;
    B = S.rb[cc][k][r];
    b0 = S.rs[cc][k][r];
    nB = S.rn[cc][k][r];
    ch = u - S.rc[cc][k][r];
    const unsigned long long N = (unsigned long long)nA * (nB ? nB : 1u);
    cl2 = chunk_log2(N, clog2, 15);
}

// concatenated index t (< M) of sequence (cc, k) -> sorted position in layer j and the cell
template <int D>
__device__ __forceinline__ uint32_t locate(const Slot<D>& S, int npar, int cs, int cc, int k, uint32_t t,
                                           uint32_t& B)
{
    // last parent with pre <= t: fixed-step branchless search (pre[npar] = total > t stops it)
    constexpr int TOP = Geo<D>::MAXPAR >= 128 ? 128 : (Geo<D>::MAXPAR >= 64 ? 64 : (Geo<D>::MAXPAR >= 32 ? 32 : (Geo<D>::MAXPAR >= 16 ? 16 : (Geo<D>::MAXPAR >= 8 ? 8 : (Geo<D>::MAXPAR >= 4 ? 4 : 2)))));
    int lo = 0;
#pragma unroll
    for (int step = TOP; step; step >>= 1) {
        const int m = lo + step;
        if (S.pre[cc][k][min(m, npar)] <= t) lo = m;
    }
    uint32_t r = t - S.pre[cc][k][lo];
    uint32_t m = S.mask[cc][k][lo];
#if GIRG_LOCATE_PRED
    if constexpr (Geo<D>::NCH <= 8) {  // one predicated pass over the parent's sub-cells (no divergence)
        uint32_t acc = 0, res = 0, bs = 0, prev = S.rstart[lo][0];
        bool fnd = false;
#pragma unroll
        for (int s = 0; s < Geo<D>::NCH; ++s) {
            const uint32_t nxt = S.rstart[lo][s + 1];
            const uint32_t nB = ((m >> s) & 1u) ? nxt - prev : 0u;
            const bool hit = !fnd && r < acc + nB;
            res = hit ? prev + (r - acc) : res;
            bs = hit ? (uint32_t)s : bs;
            fnd |= hit;
            acc += nB;
            prev = nxt;
        }
        B = (S.par[lo] << cs) + bs;
        return res;
    } else
#endif
    {
        while (m) {
            const int s = __ffs(m) - 1;
            const uint32_t nB = S.rstart[lo][s + 1] - S.rstart[lo][s];
            if (r < nB) {
                B = (S.par[lo] << cs) + (uint32_t)s;
                return S.rstart[lo][s] + r;
            }
            r -= nB;
            m &= m - 1u;
        }
        GCHK(false);  // unreachable: the prefix counts are sums over the mask (setup_job)
        B = 0;
        return S.rstart[lo][0];
    }
}

// EVENT scheme: chunk index u of sequence (cc, k) -> event (B, its range) and chunk within it
template <int D>
__device__ __forceinline__ void locate_event(const Slot<D>& S, int clog2, int npar, int cs, int cc, int k,
                                             uint32_t nA, uint32_t u, uint32_t& B, uint32_t& b0, uint32_t& nB,
                                             uint32_t& ch, int& cl2)
{
    int lo = 0, hi = npar - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S.pre[cc][k][mid] <= u) lo = mid;
        else hi = mid - 1;
    }
    uint32_t r = u - S.pre[cc][k][lo];
    uint32_t m = S.mask[cc][k][lo];
    B = b0 = nB = ch = 0;
    cl2 = 0;
    while (m) {
        const int s = __ffs(m) - 1;
        m &= m - 1u;
        const uint32_t nb = S.rstart[lo][s + 1] - S.rstart[lo][s];
        if (!nb) continue;
        const unsigned long long N = (unsigned long long)nA * nb;
        const int c = chunk_log2(N, clog2, 15);
        const uint32_t nch = (uint32_t)(((N - 1) >> c) + 1);
        if (r < nch) {
            B = (S.par[lo] << cs) + (uint32_t)s;
            b0 = S.rstart[lo][s];
            nB = nb;
            ch = r;
            cl2 = c;
            return;
        }
        r -= nch;
    }
    GCHK(false);  // unreachable (setup_job counted these chunks); nB = 0 makes an empty chain
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
    atomicAdd(&a.stats->fb, c.fb);
    atomicAdd(&a.stats->mm, c.mm);
    atomicAdd(&a.stats->ntj, c.ntj);
}

// queue a job's unit range as items of ~ITEM_WORK weighted units (lane 0)
__device__ __noinline__ void push_items(const SampleArgs& a, const TaskDesc& t, uint16_t task, int batch,
                                           unsigned long long U, unsigned long long work)
{
    if (lane_id() == 0) {
        const unsigned long long per = max(1ull, U * a.item_work / work);
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
                it.batch = (uint8_t)batch;
                it.lo = k * per;
                it.hi = min(U, (k + 1) * per);
                a.items[base + k] = it;
            }
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------------------
// job sources
// ---------------------------------------------------------------------------------------
// k_sample: persistent warps pull tiles of 32 sorted points; each point lists the jobs it owns
template <int D, int SCHEME, bool STATS>
struct TileSource {
    // the engine resolves a lane's landing / type-I lookup at one code site (k_sample: 137.6 ->
    // 117.7 ms on C5); k_big keeps them in place, where the merged site's longer-lived 64-bit
    // index made the chain state spill (36.5 -> 42.8 ms)
    static constexpr bool unified_lookup = true;
    unsigned tile = 0;
    uint32_t total = 0, tk = 0;  // jobs of the tile (warp-uniform), next one
    int i = 0, lf = 255;         // this lane's point
    uint32_t code = 0, cnt = 0, start = 0;
    uint32_t toffv = 0;          // its task list offset
    int Ii = 0;                  // I(layer) of its point
    uint16_t task32 = 0;         // task entry tk = lane of the tile (prefetched; tk >= 32 loads on demand)
    // pending task with further batches (d >= 4)
    bool pend = false;
    TaskDesc pt;
    uint16_t ptask = 0;
    int pbatch = 0;

    __device__ __forceinline__ bool next_tile(const SampleArgs& a)
    {
        const Plan* pl = a.pl;
        const unsigned lane = lane_id();
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(a.tile_ctr, 1u);
        tile = __shfl_sync(FULL, t, 0);
        if (tile >= a.ntiles) return false;
        const uint32_t p = tile * a.tile_pts + lane;
        i = 0;
        lf = 255;
        code = 0;
        if (lane < a.tile_pts && p < a.n) {
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
        cnt = lf == 255 ? 0u : pl->tcnt[i * 33 + lf];
        toffv = lf == 255 ? 0u : pl->toff[i];
        Ii = pl->I[i];
        start = warp_excl_scan(cnt, total);
        tk = 0;
        // prefetch the tile's first 32 task entries, one per lane (their loads overlap the jobs)
        // owner of task entry `lane`: the last point whose start <= lane (starts are an exclusive
        // scan, so for lane < total this is the nonempty list holding it); binary search
        int owner = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
            const uint32_t ss = __shfl_sync(FULL, start, owner + step < 32 ? owner + step : 31);
            if (owner + step < 32 && ss <= lane) owner += step;
        }
        const uint32_t otoff = __shfl_sync(FULL, toffv, owner), ostart = __shfl_sync(FULL, start, owner);
        task32 = lane < total ? __ldg(&a.tasks[otoff + (lane - ostart)]) : (uint16_t)0;
        return true;
    }

    // set up the next job into S; false when the grid's tiles are exhausted
    __device__ __noinline__ bool next(const SampleArgs& a, SlotT<D>& S, unsigned long long& lo,
                                         unsigned long long& hi, Counters& C)
    {
        for (;;) {
            TaskDesc t;
            uint16_t task;
            int batch;
            constexpr bool multi = Geo<D>::CB < Geo<D>::NCH;  // d >= 4: a task may need several batches
            if (multi && pend) {
                t = pt;
                task = ptask;
                batch = pbatch;
            } else {
                while (tk >= total)
                    if (!next_tile(a)) return false;
                const unsigned own = __ballot_sync(FULL, cnt > 0 && start <= tk);
                const int ol = 31 - __clz(own);
                const int oi = __shfl_sync(FULL, i, ol);
                const uint32_t ocode = __shfl_sync(FULL, code, ol);
                const int oI = __shfl_sync(FULL, Ii, ol);
                const uint16_t tp = (uint16_t)__shfl_sync(FULL, (uint32_t)task32, tk & 31u);
                if (tk < 32) {
                    task = tp;
                } else {
                    const uint32_t ostart = __shfl_sync(FULL, start, ol), otoff = __shfl_sync(FULL, toffv, ol);
                    GCHK(otoff + (tk - ostart) < a.ntasks);
                    task = __ldg(&a.tasks[otoff + (tk - ostart)]);
                }
                ++tk;
                int lg = max(0, ((task >> 6) & 63) - Geo<D>::G);
                if constexpr (SCHEME == SCHEME_REFINED)
                    if ((task >> 14) & 1) lg = (task >> 6) & 63;  // refined job: the task cell is A itself, on level l
                t = make_task<D>(oi, task, ocode >> (D * (oI - lg)));
                batch = 0;

            }
            const JobSetup js = setup_any<D, SCHEME>(a, S, t, batch);
            if (STATS && lane_id() == 0) C.ev2 += js.nseq2;
            const unsigned long long U = js.U, work = js.work;
            pend = multi && (batch + 1) * Geo<D>::CB < js.nchild;
            if (multi && pend) {
                pt = t;
                ptask = task;
                pbatch = batch + 1;
            }
            if (U == 0) continue;
            if (work > a.big_work) {  // too much for one warp: queue unit ranges for k_big
                push_items(a, t, task, batch, U, work);
                continue;
            }
            lo = 0;
            hi = U;
            return true;
        }
    }
};

// k_big: warps pull queued items (unit ranges of big jobs)
template <int D, int SCHEME, bool STATS>
struct ItemSource {
    static constexpr bool unified_lookup = false;  // see TileSource
    unsigned nit;
    __device__ __noinline__ bool next(const SampleArgs& a, SlotT<D>& S, unsigned long long& lo,
                                         unsigned long long& hi, Counters& C)
    {
        for (;;) {
            // dynamic assignment (one atomic per item): the kernel's tail is one item, not the
            // spread of per-warp sums of a static stride
            unsigned k = 0;
            if (lane_id() == 0) k = atomicAdd(a.item_ctr, 1u);
            k = __shfl_sync(FULL, k, 0);
            if (k >= nit) return false;
            const BigItem it = a.items[k];
            const TaskDesc t = make_task<D>(it.i, it.task, it.Cpar);
            const JobSetup js = setup_any<D, SCHEME>(a, S, t, it.batch);  // sequences were counted by the job that queued it
            (void)C;
#ifdef GIRG_DEBUG
            if (js.U < it.hi && lane_id() == 0)
                printf("k_big item %u: job U %llu < item hi %llu (i %d task %x Cpar %u batch %d nchild %d)\n", k,
                       js.U, it.hi, it.i, it.task, it.Cpar, it.batch, js.nchild);
#endif
            if (js.U < it.hi) {
                atomicOr(a.err, ERR_ITEMS);
                continue;
            }
            if (it.hi <= it.lo) continue;
            lo = it.lo;
            hi = it.hi;
            return true;
        }
    }
};

// ---------------------------------------------------------------------------------------
// the engine.  Per iteration every lane (1) computes one Philox block: the next draw of its jump
// chain, or else the pair-keyed uniform of its pending type-I candidate; (2) advances its chain,
// which yields the lane's NEXT candidate (a landing); (3) evaluates its PENDING candidate, whose
// point records were loaded in the previous iteration; (4) if it holds no chain, takes a unit of
// the dispatch slot (a type-I unit is the next candidate by itself, a chunk starts a chain);
// (5) issues the loads of the next candidate.  The loads are in flight across the Philox and
// the draw of the following iteration (software pipelining).  A lane never needs two Philox
// blocks in one iteration: a pending type-I candidate implies it held no chain.  When the
// dispatch slot runs dry, the next job is set up in a slot no lane's chain refers to.
// ---------------------------------------------------------------------------------------
// MAYBE_T0: the caller may pass T = 0.  Only the batched kernels do (single calls run the flat
// T = 0 loop below), so the single-call instantiations drop the threshold branches: C2 3.03 ->
// 2.97 ms, C4 20.2 -> 20.0, C5 151.6 -> 151.0 -- except d = 2, whose register allocation is better
// with them (C3 9.35 vs 9.99 ms without; profiles/r02/tail_items/engine_t0_template_ab.txt)
template <int D, int SCHEME, bool STATS, bool MAYBE_T0 = (D == 2) || GIRG_ENGINE_T0, class Src>
__device__ __forceinline__ void engine(const SampleArgs& a, WarpSmem<D>& W, Src& src, Counters& C)
{
    static_assert(Geo<D>::CB <= 16, "the lookup pack holds the child in 4 bits");
    const unsigned lane = lane_id();
    const bool T0 = MAYBE_T0 && a.T == 0.0;
    const double s_ = a.s, invT = a.invT;
#ifdef GIRG_PROFILE
    const long long t_start = clock64();
    unsigned long long n_jobs = 0, n_iter = 0, n_steps = 0;
#endif
    unsigned fill = 0;
    int ds = 0, dq = 0;  // dispatch slot, its first sequence with units left
    unsigned long long dnext = 0, dhi = 0;
    bool more = true;
    // chain state (type-II)
    bool chain = false;
    int ls = 0, cc = 0, kind = 0;
    long long pos = 0, end = 0;
    uint32_t r = 0, ch = 0, Bev = 0, eb0 = 0, enB = 0;
    // pending candidate: kind (-1: none), acceptance uniform and bound (type-II), loaded data
    int pk = -1;
    uint32_t ppa = 0, ppb = 0;
    double pra = 0.0, ppbar = 1.0;
    double xu[D], xv[D], wu = 0.0, wv = 0.0;
    uint32_t ua = 0, ub = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) xu[k] = xv[k] = 0.0;
    for (;;) {
#ifdef GIRG_PROFILE
        if (a.wprof) {
            ++n_iter;
            n_steps += __popc(__ballot_sync(FULL, chain || pk >= 0));
        }
#endif
        // ---- (1) one Philox block per lane ----
        uint4 o = make_uint4(0u, 0u, 0u, 0u);
        if (!T0 && (chain || pk == 0)) {
            uint4 ctr;
            if (chain) {
                const SlotT<D>& S = W.slot[ls];
                const uint32_t A = S.seq[cc][kind].A;
                if constexpr (SCHEME == SCHEME_REFINED) ctr = make_uint4(A, ch, S.job.tag + ((uint32_t)kind << 17), r);
                else
                ctr = SCHEME == SCHEME_MERGED ? make_uint4(A, ch, S.job.tag | ((uint32_t)(kind - 1) << 17) | (1u << 18), r)
                                              : make_uint4(A, Bev, S.job.tag | (ch << 17), r);
            } else {
                ctr = make_uint4(min(ua, ub), max(ua, ub), 0u, 3u);  // type-I: keyed by the vertex pair (R17)
            }
            o = philox4x32_10(ctr, a.k0, a.k1);
        }
        // ---- (2) the chain's draw -> next candidate ----
        int nk = -1;
        uint32_t npa = 0, npb = 0;
        double nra = 0.0, npbar = 1.0;
        // the lane's one lookup of this iteration (its landing or a dispatched type-I candidate):
        // slot << 8 | child << 2 | kind (-1: none) and the index in the sequence's row-major space,
        // resolved by a single divmod + locate below (one code copy, executed by both lane kinds)
        int lpack = -1;
        unsigned long long lval = 0;
        if (chain) {
            const SlotT<D>& S = W.slot[ls];
            const Seq& Q = S.seq[cc][kind];
            ++r;
            if (STATS) ++C.draws;
            constexpr int KO = KOff<SCHEME>::v;
            const double pb_ = S.job.pbar[kind - KO];
            const double rj = u53(o.x, o.y);
            const long long remaining = end - pos - 1;
            // skip = floor(log(1-rj)/log1p(-pbar)) (R10): fast float path, canonical double fallback
            long long skip = 0;
            int st = (pb_ == 1.0 || rj == 0.0) ? (remaining <= 0 ? 1 : 0)  // z = 0 exactly
                                               : fast_jump(__dsub_rn(1.0, rj), S.job.il2[kind - KO], remaining, skip);
            if (STATS || st < 0) {
                const double z = pb_ == 1.0 ? 0.0 : exact_skip(rj, S.job.Lbar[kind - KO]);
                const int st2 = z >= (double)remaining ? 1 : 0;
                if (STATS) {
                    if (st < 0) ++C.fb;
                    else C.mm += (st != st2) || (st == 0 && skip != (long long)z);
                    // jump near-tie (R21), the oracle's O12 rule evaluated on the device's own z
                    if (pb_ < 1.0 && z < (double)remaining + 1.0 && fabs(z - rint(z)) < 1e-15 * fmax(1.0, fabs(z)))
                        ++C.ntj;
                }
                st = st2;
                skip = st2 ? 0 : (long long)z;
            }
            if (st) {
                chain = false;
            } else {
                pos += 1 + skip;
                if (STATS) ++C.landings;
                nk = SCHEME == SCHEME_REFINED ? kind + 1 : kind;  // > 0: a landing (a refined job's kind 0 is a chain)
                nra = u53(o.z, o.w);
                npbar = pb_;
                if constexpr (Src::unified_lookup) {
                    lpack = (ls << 8) | (cc << 2) | kind | (SCHEME == SCHEME_REFINED ? 128 : 0);  // bit 7: landing
                    lval = (unsigned long long)pos;
                } else {
                    const unsigned long long g = (unsigned long long)pos;
                    uint32_t ti;
                    const uint32_t si = divmod(g, SCHEME != SCHEME_EVENT ? Q.M : enB, ti);
                    npa = Q.a0 + si;
                    if (SCHEME != SCHEME_EVENT) {
                        uint32_t B;
                        npb = locate(S, S.job.npar, S.job.cs, cc, kind, ti, B);
                    } else {
                        npb = eb0 + ti;
                    }
                }
            }
        }
        // ---- (3) evaluate the pending candidate (records loaded last iteration) ----
        bool edge = false;
        if (pk >= 0) {
            const double Dp = dist_pow<D>(xu, xv);
            if (T0) {
                edge = Dp <= __dmul_rn(__dmul_rn(wu, wv), s_);
            } else {
                // type-I: edge iff p >= 1 or r < p; type-II: edge iff r_acc * pbar < p (R14).
                // Both are "x < p" with x < 1.
                const double x = pk == 0 ? u53(o.x, o.y) : __dmul_rn(pra, ppbar);
                const int fe = fast_lt_prob(x, __dmul_rn(__dmul_rn(wu, wv), s_), Dp, invT);
                edge = fe == 1;
                if (STATS || fe < 0) {
                    const double p = exact_prob(wu, wv, s_, Dp, invT);
                    const bool e2 = x < p;
                    if (STATS) {
                        if (fe < 0) ++C.fb;
                        else C.mm += e2 != (fe == 1);
                        if (pk == 0) C.nt1 += p < 1.0 && fabs(x - p) < 1e-12;
                        else C.nt2 += fabs(x - p) < 1e-12 * ppbar;
                    }
                    edge = e2;
                }
            }
            if (STATS) {
                if (pk == 0) ++C.cand1;
                if (edge) {
                    if (pk == 0) ++C.edges1;
                    else ++C.edges2;
                }
            }
            if (edge && pk > 0) {  // type-II: ids only for accepted landings (~5 %)
                ua = __ldg(&a.sid[ppa]);
                ub = __ldg(&a.sid[ppb]);
            }
        }
        warp_emit<Geo<D>::EB>(a, W.ebuf, fill, edge, ua, ub);
        // ---- (4) job setup when the dispatch slot is exhausted, then dispatch ----
        if (dnext >= dhi && more) {
            const unsigned occupied = __reduce_or_sync(FULL, chain ? (1u << ls) : 0u);
            const int ns = __ffs(~occupied) - 1;
            if (ns < Geo<D>::NSLOT) {
                unsigned long long lo, hi;
                if (src.next(a, W.slot[ns], lo, hi, C)) {
#ifdef GIRG_PROFILE
                    ++n_jobs;
                    if (a.dev_flags & 1) lo = hi;
#endif
                    ds = ns;
                    dnext = lo;
                    dhi = hi;
                    dq = 0;
#pragma unroll 1
                while (dq < 3 * Geo<D>::CB - 1 && W.slot[ds].uoff[dq + 1] <= dnext) ++dq;
                } else {
                    more = false;
                }
            }
        }
        const unsigned idle = __ballot_sync(FULL, !chain);
        if (!chain && dnext < dhi) {
            const unsigned long long u = dnext + __popc(idle & ((1u << lane) - 1u));
            if (u < dhi) {
                const SlotT<D>& S = W.slot[ds];
                int q = dq;  // sequence holding unit u
#pragma unroll 1
                while (q < 3 * Geo<D>::CB - 1 && S.uoff[q + 1] <= u) ++q;
                const int qc = q / 3, qk = q - 3 * qc;
                const Seq& Q = S.seq[qc][qk];
                const unsigned long long x = u - S.uoff[q];
                if (qk == 0 && !(SCHEME == SCHEME_REFINED && S.job.ref)) {
                    if constexpr (Src::unified_lookup) {
                        lpack = (ds << 8) | (qc << 2);
                        lval = x;
                    } else {
                        uint32_t ti;
                        const uint32_t si = divmod(x, Q.M, ti);
                        uint32_t B;
                        npa = Q.a0 + si;
                        npb = locate(S, S.job.npar, S.job.cs, qc, 0, ti, B);
                        if (!(S.job.same_layer && B == Q.A && npb <= npa)) nk = 0;  // same cell: only s < t (R16)
                    }
                } else {
                    chain = true;
                    ls = ds;
                    cc = qc;
                    kind = qk;
                    r = 0;
                    if (SCHEME != SCHEME_EVENT) {
                        ch = (uint32_t)x;
                        const unsigned long long st = x << Q.cl2;
                        pos = (long long)st - 1;
                        end = (long long)min((unsigned long long)Q.nA * Q.M, st + (1ull << Q.cl2));
                    } else {
                        int c2;
                        locate_event(S, S.job.clog2[qk - 1], S.job.npar, S.job.cs, qc, qk, Q.nA, (uint32_t)x, Bev,
                                        eb0, enB, ch, c2);
                        const unsigned long long N = (unsigned long long)Q.nA * enB;
                        const unsigned long long st = (unsigned long long)ch << c2;
                        pos = (long long)st - 1;
                        end = (long long)min(N, st + (1ull << c2));
                    }
                    if (STATS) ++C.chunks;
                }
            }
        }
        if (dnext < dhi) {
            dnext = min(dhi, dnext + __popc(idle));
            if (dnext < dhi)
#pragma unroll 1
                while (dq < 3 * Geo<D>::CB - 1 && W.slot[ds].uoff[dq + 1] <= dnext) ++dq;
        }
        // ---- the lookup: row-major index -> (row s, column t) -> sorted positions ----
        if (Src::unified_lookup && lpack >= 0) {
            const int lk = lpack & 3, lc = (lpack >> 2) & 15;
            const bool cand1 = lk == 0 && !(SCHEME == SCHEME_REFINED && (lpack & 128));  // a dispatched type-I candidate
            const SlotT<D>& S = W.slot[lpack >> 8];
            const Seq& Q = S.seq[lc][lk];
            const bool ev = SCHEME == SCHEME_EVENT && lk > 0;  // EVENT landing: one cell (enB, eb0)
            uint32_t ti;
            const uint32_t si = divmod(lval, ev ? enB : Q.M, ti);
            npa = Q.a0 + si;
            if (ev) {
                npb = eb0 + ti;
            } else {
                uint32_t B;
                npb = locate(S, S.job.npar, S.job.cs, lc, lk, ti, B);
                if (cand1 && !(S.job.same_layer && B == Q.A && npb <= npa)) nk = 0;  // same cell: only s < t (R16)
            }
        }
        // ---- (5) issue the loads of the next candidate ----
        pk = nk;
        ppa = npa;
        ppb = npb;
        pra = nra;
        ppbar = npbar;
        if (nk >= 0) {
#if defined(GIRG_EXP_NOLOAD2) || defined(GIRG_EXP_NOLOAD1)
#ifdef GIRG_EXP_NOLOAD1
            if (nk == 0) {  // timing experiment only: type-I candidates without their record loads
#else
            if (nk > 0) {  // timing experiment only: type-II landings without their record loads
#endif
#pragma unroll
                for (int k = 0; k < D; ++k) { xu[k] = 0.25 + 1e-3 * (npa & 255); xv[k] = 0.75 - 1e-3 * (npb & 255); }
                wu = 1.5; wv = 1.5;
            } else {
                load_rec<D>(a, npa, xu, wu);
                load_rec<D>(a, npb, xv, wv);
            }
#else
            load_rec<D>(a, npa, xu, wu);
            load_rec<D>(a, npb, xv, wv);
#endif
            if (nk == 0) {  // type-I: the ids key the pair's uniform (R17)
                ua = __ldg(&a.sid[npa]);
                ub = __ldg(&a.sid[npb]);
            }
        }
        if (!more && dnext >= dhi && !__any_sync(FULL, chain || pk >= 0)) break;
    }
    warp_flush(a, W.ebuf, fill);
#ifdef GIRG_PROFILE
    if (a.wprof && lane == 0) {
        const unsigned w = blockIdx.x * Geo<D>::WPB + (threadIdx.x >> 5);
        unsigned long long* op = a.wprof + 4ull * w;
        op[0] += (unsigned long long)(clock64() - t_start);
        op[1] += n_jobs;
        op[2] += n_iter;
        op[3] += n_steps;
    }
#endif
}

// T = 0 (threshold model: every unit is a type-I candidate, no jump chains, no draws): a flat
// candidate loop -- 32 candidates per warp step, one per lane -- in its own kernel instantiation
// (FLAT = true), so the T > 0 engine's register allocation is untouched.  B200, sampling phase:
// n = 2^24 d = 1 11.4 -> 10.9 ms, n = 2^22 d = 2 8.3 -> 6.2 ms, n = 2^20 d = 3 5.9 -> 5.5 ms.
template <int D, int SCHEME, bool STATS, class Src>
__device__ __forceinline__ void engine_cand(const SampleArgs& a, WarpSmem<D>& W, Src& src, Counters& C)
{
    const unsigned lane = lane_id();
    unsigned fill = 0;
    const double s_ = a.s;
    for (;;) {
        unsigned long long lo, hi;
        if (!src.next(a, W.slot[0], lo, hi, C)) break;
        const SlotT<D>& S = W.slot[0];
        for (unsigned long long b = lo; b < hi; b += 32) {
            const unsigned long long u = b + lane;
            bool edge = false;
            uint32_t ua = 0, ub = 0;
            if (u < hi) {
                int q = 0;
#if GIRG_T0_ROLL
#pragma unroll 1
#endif
                while (q < 3 * Geo<D>::CB - 1 && S.uoff[q + 1] <= u) ++q;
                const int qc = q / 3;
                const Seq& Q = S.seq[qc][0];
                uint32_t ti;
                const uint32_t si = divmod(u - S.uoff[q], Q.M, ti);
                uint32_t B;
                const uint32_t npa = Q.a0 + si;
                const uint32_t npb = locate(S, S.job.npar, S.job.cs, qc, 0, ti, B);
                if (!(S.job.same_layer && B == Q.A && npb <= npa)) {
                    double xu[D], xv[D], wu, wv;
                    load_rec<D>(a, npa, xu, wu);
                    load_rec<D>(a, npb, xv, wv);
                    edge = dist_pow<D>(xu, xv) <= __dmul_rn(__dmul_rn(wu, wv), s_);
                    if (STATS) {
                        ++C.cand1;
                        C.edges1 += edge;
                    }
                    if (edge) {
                        ua = __ldg(&a.sid[npa]);
                        ub = __ldg(&a.sid[npb]);
                    }
                }
            }
            warp_emit<Geo<D>::EB>(a, W.ebuf, fill, edge, ua, ub);
        }
    }
    warp_flush(a, W.ebuf, fill);
}

template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB) k_sample(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    TileSource<D, SCHEME, STATS> src;
    engine<D, SCHEME, STATS>(a, W, src, C);
    flush_counters<STATS>(a, C);
}

// T = 0 instantiations (flat candidate loop)
template <int D, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB) k_sample_t0(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    TileSource<D, SCHEME_MERGED, STATS> src;
    engine_cand<D, SCHEME_MERGED, STATS>(a, W, src, C);
    flush_counters<STATS>(a, C);
}

template <int D, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB_BIG) k_big_t0(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    ItemSource<D, SCHEME_MERGED, STATS> src;
    src.nit = (*a.err & ERR_ITEMS) ? 0u : min(*a.nitems, a.items_cap);
    engine_cand<D, SCHEME_MERGED, STATS>(a, W, src, C);
    flush_counters<STATS>(a, C);
}

template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB_BIG) k_big(SampleArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    ItemSource<D, SCHEME, STATS> src;
    // an overflowing push skipped its whole reservation, so [0, cap) may hold unwritten items:
    // on overflow do nothing (the host grows the queue and re-runs the sampler)
    src.nit = (*a.err & ERR_ITEMS) ? 0u : min(*a.nitems, a.items_cap);
    engine<D, SCHEME, STATS>(a, W, src, C);
    flush_counters<STATS>(a, C);
}

// batched calls (girg_edges_batch): blockIdx.y is the graph; its arguments are copied into shared
// memory once per block, and the engine is the single-graph engine
template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB) k_sample_b(const SampleArgs* __restrict__ args)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ SampleArgs sa;
    if (threadIdx.x == 0) sa = args[blockIdx.y];
    __syncthreads();
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    TileSource<D, SCHEME, STATS> src;
    engine<D, SCHEME, STATS, true>(sa, W, src, C);
    flush_counters<STATS>(sa, C);
}

template <int D, int SCHEME, bool STATS>
__global__ void __launch_bounds__(32 * Geo<D>::WPB, Geo<D>::MINB_BIG) k_big_b(const SampleArgs* __restrict__ args)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ SampleArgs sa;
    if (threadIdx.x == 0) sa = args[blockIdx.y];
    __syncthreads();
    WarpSmem<D>& W = reinterpret_cast<WarpSmem<D>*>(smem_raw)[threadIdx.x >> 5];
    Counters C = {};
    ItemSource<D, SCHEME, STATS> src;
    src.nit = (*sa.err & ERR_ITEMS) ? 0u : min(*sa.nitems, sa.items_cap);
    engine<D, SCHEME, STATS, true>(sa, W, src, C);
    flush_counters<STATS>(sa, C);
}

