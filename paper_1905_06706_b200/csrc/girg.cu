// girg.cu -- B200 (sm_100a) GIRG edge generator: kernels, host orchestration and the C ABI.
//
// Pipeline of girg_edges:
//   K0 k_wstats     exact W (per-block 128-bit fixed point), weight-exponent histogram -> host plan
//   H6 host plan    layers, CL / I levels, pbar tables
//   K1 k_keys       layer + Morton cell at the insertion level, histogram over the cell space
//   K2 k_scan_*     exclusive scan of the cell histogram = the prefix arrays P_C of Lemma 1
//   K3 k_scatter    slot of every vertex in its cell
//   K4 k_order      in-cell order by vertex id (R11); k_place: sorted AoS point records
//   K5 k_sample     jobs (layer pair, level, task cell): type-I pair tests and type-II geometric
//                   jumps (Algorithm 1 events), warp-staged edge output; k_big runs
//                   the unit ranges of queued big jobs (csrc/sample.cuh)
// Citations "P:NNN" are lines of PAPER.md (arXiv:1905.06706); R* are DESIGN.md readings.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstddef>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <memory>
#include <thread>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/girg.h"
#include "girg_device.cuh"

#ifndef GIRG_SMALL_TILE_N
#define GIRG_SMALL_TILE_N (1u << 17)  // graphs below this many points sample with 8-point tiles
#endif
#ifndef GIRG_CHUNK_SHIFT
#define GIRG_CHUNK_SHIFT 1  // merged chunks of 2^(SHIFT - ilogb(pbar)) candidates (R22; the oracle's value)
#endif

namespace girg {

constexpr int MAXL = 64;
constexpr int EXP_BIAS = 1023;
constexpr int HIST_BINS = 2048;
constexpr int WS_THREADS = 256, WS_PER_THREAD = 8, WS_TILE = WS_THREADS * WS_PER_THREAD;

// device error bits
constexpr int ERR_WEIGHT = 1, ERR_WRANGE = 2, ERR_POS = 4;

struct TabEntry {
    double pbar;  // type-II bound for (i, j, level, class)
    double Lbar;  // log1p(-pbar)
    int clog2;    // EVENT scheme: chunk length C = 2^clog2 candidates (2..4 expected landings, R10)
    int clog2m;   // MERGED scheme: 2^clog2m candidates (2..4 expected landings, R22)
    double il2;   // 1 / log2(1 - pbar) = ln 2 / Lbar (fast jump path; unused when pbar = 1)
    double pad;
};

struct Plan {
    int L, d, e_min, maxCL;
    double s, T, invT;
    int sl, pad;
    unsigned long long blo, bhi;
    uint32_t base[MAXL + 1];    // offset of layer i in the concatenated cell space
    uint32_t lstart[MAXL + 1];  // first sorted position of layer i
    uint32_t cnt[MAXL];
    uint8_t I[MAXL];
    // task lists per (layer i, first level lf in 0..32): entries
    // j | l<<6 | typeI<<12 | typeII<<13; layer i's tasks are stored once by decreasing task level
    // at tasks[toff[i]], and the list of (i, lf) is their first tcnt[i*33+lf] entries
    uint32_t toff[MAXL];
    uint16_t tcnt[MAXL * 33];
    uint32_t tab_off[MAXL * MAXL];  // type-II bound table offset of the layer pair (i, j)
    // ---- host only from here on (not uploaded) ----
    uint8_t CL[MAXL * MAXL];
};
// bytes of a plan the device reads: everything up to the last used tab_off entry
static inline size_t plan_upload_bytes(const Plan& p)
{
    return offsetof(Plan, tab_off) + (size_t)((p.L > 0 ? p.L - 1 : 0) * MAXL + p.L) * sizeof(uint32_t);
}

struct WPartial {
    unsigned long long lo, hi;  // sum of m * 2^(e - e_b) over the block
    int e_b, emax;
    unsigned long long wmax_bits;  // largest weight of the block (positive doubles order as ints)
};

// ======================================================================================
// H1, H2: generators
// ======================================================================================
__global__ void k_weights(uint32_t n, double ex, uint32_t k0, uint32_t k1, double* __restrict__ w)
{
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint4 o = philox4x32_10(make_uint4(v, 0u, 0u, 1u), k0, k1);
    const double U = u53(o.x, o.y);
    w[v] = pow(__dsub_rn(1.0, U), ex);  // (1-U)^(-1/(beta-1)), 1-U exact
}

__global__ void k_positions(uint32_t n, int d, uint32_t k0, uint32_t k1, double* __restrict__ x)
{
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    for (int k = 0; 2 * k < d; ++k) {
        const uint4 o = philox4x32_10(make_uint4(v, (uint32_t)k, 0u, 2u), k0, k1);
        x[(size_t)(2 * k) * n + v] = u53(o.x, o.y);
        if (2 * k + 1 < d) x[(size_t)(2 * k + 1) * n + v] = u53(o.z, o.w);
    }
}

// ======================================================================================
// K0: weight statistics.  W exactly rounded (R3): w = m 2^(e-52) with m the 53-bit
// significand; each block sums m * 2^(e - e_b) exactly in 128 bits (e_b = block minimum,
// e - e_b <= 63 because at most 64 layers are allowed), the host adds the block partials in
// 256 bits and rounds once.  Also the histogram of exponents (layer sizes).
// ======================================================================================
__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi,
                                       unsigned long long alo, unsigned long long ahi)
{
    const unsigned long long t = lo + alo;
    hi += ahi + (t < lo ? 1ull : 0ull);
    lo = t;
}

// Batched calls (girg_edges_batch) run B graphs in one launch: blockIdx.y is the graph, the
// per-graph inputs come from the pointer array wb (nullptr: the single graph w), and the outputs
// of graph g sit at hist + g HIST_BINS, part + g gridDim.x, err + g * err_stride.
__global__ void __launch_bounds__(WS_THREADS) k_wstats(const double* __restrict__ w0, uint32_t n,
                                                       uint32_t* __restrict__ hist,
                                                       WPartial* __restrict__ part,
                                                       int* __restrict__ err, const double* const* wb = nullptr,
                                                       int err_stride = 0)
{
    const unsigned g = blockIdx.y;
    const double* __restrict__ w = wb ? wb[g] : w0;
    hist += (size_t)g * HIST_BINS;
    part += (size_t)g * gridDim.x;
    err += (size_t)g * err_stride;
    __shared__ uint32_t sh_hist[HIST_BINS];
    __shared__ int sh_emin, sh_emax;
    __shared__ unsigned long long sh_lo[WS_THREADS / 32], sh_hi[WS_THREADS / 32], sh_wmax;
    for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) sh_hist[i] = 0;
    if (threadIdx.x == 0) { sh_emin = INT_MAX; sh_emax = INT_MIN; sh_wmax = 0; }
    __syncthreads();

    const size_t base = (size_t)blockIdx.x * WS_TILE;
    unsigned long long m[WS_PER_THREAD];
    int e[WS_PER_THREAD];
    int emin = INT_MAX, emax = INT_MIN, bad = 0;
    unsigned long long wmb = 0;
#pragma unroll
    for (int k = 0; k < WS_PER_THREAD; ++k) {
        const size_t idx = base + (size_t)k * WS_THREADS + threadIdx.x;
        e[k] = INT_MIN;
        m[k] = 0;
        if (idx < n) {
            const unsigned long long bits = __double_as_longlong(w[idx]);
            const int ef = (int)((bits >> 52) & 0x7ff);
            const bool sign = (bits >> 63) != 0;
            if (sign || ef == 0 || ef == 0x7ff) {  // <= 0, subnormal, inf, nan
                bad |= ERR_WEIGHT;
                continue;
            }
            const int ee = ef - EXP_BIAS;
            if (ee < -500 || ee > 500) { bad |= ERR_WRANGE; continue; }
            e[k] = ee;
            m[k] = (bits & ((1ull << 52) - 1)) | (1ull << 52);
            wmb = max(wmb, bits);
            emin = min(emin, ee);
            emax = max(emax, ee);
            // warp-aggregated histogram update
            const unsigned grp = __match_any_sync(__activemask(), ee);
            if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&sh_hist[ee + EXP_BIAS], __popc(grp));
        }
    }
    if (bad) atomicOr(err, bad);
    atomicMin(&sh_emin, emin);
    atomicMax(&sh_emax, emax);
    atomicMax(&sh_wmax, wmb);
    __syncthreads();
    const int eb = sh_emin;
    unsigned long long lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < WS_PER_THREAD; ++k) {
        if (e[k] == INT_MIN) continue;
        const int sh = e[k] - eb;
        if (sh > 63) { atomicOr(err, ERR_WRANGE); continue; }
        const unsigned long long alo = m[k] << sh;
        const unsigned long long ahi = sh ? (m[k] >> (64 - sh)) : 0ull;
        add128(lo, hi, alo, ahi);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const unsigned long long olo = __shfl_down_sync(0xffffffffu, lo, off);
        const unsigned long long ohi = __shfl_down_sync(0xffffffffu, hi, off);
        add128(lo, hi, olo, ohi);
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sh_lo[wid] = lo; sh_hi[wid] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tlo = 0, thi = 0;
        for (int k = 0; k < WS_THREADS / 32; ++k) add128(tlo, thi, sh_lo[k], sh_hi[k]);
        part[blockIdx.x].lo = tlo;
        part[blockIdx.x].hi = thi;
        part[blockIdx.x].e_b = eb;
        part[blockIdx.x].emax = sh_emax;
        part[blockIdx.x].wmax_bits = sh_wmax;
    }
    for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x)
        if (sh_hist[i]) atomicAdd(&hist[i], sh_hist[i]);
}

// ======================================================================================
// K1: cell keys at the insertion level (Lemma 1 proof P:994-996: coordinates by rounding,
// Morton index P:577-588) over the concatenated cell space; histogram of keys.
// ======================================================================================
template <int D>
__global__ void k_keys(const double* __restrict__ w0, const double* __restrict__ x0, uint32_t n,
                       const Plan* __restrict__ pl0, uint32_t* __restrict__ key,
                       uint32_t* __restrict__ cnt, int* __restrict__ err0, const double* const* wb = nullptr,
                       const double* const* xb = nullptr, int err_stride = 0)
{
    // batched: graph g = blockIdx.y, its points at g n .. g n + n - 1 of the concatenated arrays,
    // its plan's layer bases already offset into the concatenated cell space
    const unsigned g = blockIdx.y;
    const double* __restrict__ w = wb ? wb[g] : w0;
    const double* __restrict__ x = xb ? xb[g] : x0;
    const Plan* __restrict__ pl = pl0 + g;
    int* err = err0 + (size_t)g * err_stride;
    key += (size_t)g * n;
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const unsigned long long bits = __double_as_longlong(w[v]);
    const int layer = (int)((bits >> 52) & 0x7ff) - EXP_BIAS - pl->e_min;
    const int I = pl->I[layer];
    const double scale = __ull2double_rn(1ull << I);
    uint32_t c[D];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double xv = x[(size_t)k * n + v];
        ok = ok && (xv >= 0.0) && (xv < 1.0);
        c[k] = ok ? __double2uint_rz(__dmul_rn(xv, scale)) : 0u;
    }
    if (!ok) atomicOr(err, ERR_POS);
    const uint32_t kv = pl->base[layer] + morton_encode<D>(c);
    key[v] = kv;
    atomicAdd(&cnt[kv], 1u);
}

// ======================================================================================
// K2: exclusive scan of cnt[0..K] (K+1 entries) -> P (hand-written 3-phase scan)
// ======================================================================================
constexpr int SCAN_THREADS = 256, SCAN_PER_THREAD = 16, SCAN_TILE = SCAN_THREADS * SCAN_PER_THREAD;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* sh_warp, uint32_t& total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) sh_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t s = lane < nw ? sh_warp[lane] : 0u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += t;
        }
        if (lane < nw) sh_warp[lane] = s;
    }
    __syncthreads();
    total = sh_warp[(blockDim.x >> 5) - 1];
    const uint32_t wofs = wid ? sh_warp[wid - 1] : 0u;
    __syncthreads();
    return wofs + incl - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const uint32_t* __restrict__ in, uint64_t len,
                                                              uint32_t* __restrict__ bsum)
{
    __shared__ uint32_t sh[SCAN_THREADS / 32];
    const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        const uint64_t i = base + (uint64_t)k * SCAN_THREADS + threadIdx.x;
        if (i < len) s += in[i];
    }
    uint32_t total;
    block_exclusive_scan(s, sh, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(uint32_t* __restrict__ bsum, uint32_t nb)
{
    __shared__ uint32_t sh[32];
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
    uint32_t s = 0;
    for (uint32_t b = b0; b < b1; ++b) s += bsum[b];
    uint32_t total;
    uint32_t ex = block_exclusive_scan(s, sh, total);
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t t = bsum[b];
        bsum[b] = ex;
        ex += t;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_final(uint32_t* __restrict__ in, uint64_t len,
                                                             const uint32_t* __restrict__ bsum,
                                                             uint32_t* __restrict__ out)
{
    __shared__ uint32_t sh[SCAN_THREADS / 32];
    // each thread owns SCAN_PER_THREAD consecutive elements
    const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_PER_THREAD;
    uint32_t vals[SCAN_PER_THREAD];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        const uint64_t i = base + k;
        vals[k] = i < len ? in[i] : 0u;
        s += vals[k];
    }
    uint32_t total;
    uint32_t ex = block_exclusive_scan(s, sh, total) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        const uint64_t i = base + k;
        if (i < len) {
            out[i] = ex;
            in[i] = ex + vals[k];  // the counts become scatter cursors: the cell's exclusive end
        }
        ex += vals[k];
    }
}

// K5: sampling kernels (Geo<D> is also used by the index build below)
#include "sample.cuh"

// ======================================================================================
// K3/K4: counting-sort placement; in-cell order by vertex id (R11) and payload gather
// ======================================================================================
__global__ void k_scatter(const uint32_t* __restrict__ key, uint32_t n, uint32_t* __restrict__ cnt,
                          uint2* __restrict__ tk)
{
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint32_t k = key[v];
    const uint32_t slot = atomicSub(&cnt[k], 1u) - 1u;  // cursor = P[k] + remaining count
    tk[slot] = make_uint2(v, k);  // (id, key) in one 8-byte store: one random write per point
}

// in-cell order by vertex id (R11): the slot order of k_scatter is arbitrary inside a cell, the
// rank of v among its cell's ids is its final position.  Writes the sorted id / key arrays and
// the inverse permutation used by k_place.  Cells of <= ORDER_SMALL points rank each point by
// scanning the cell (<= ORDER_SMALL^2 reads per cell); larger cells are listed for k_order_big
// (a linear-time radix sort per cell), so crowded cells cost O(c), not O(c^2).
constexpr uint32_t ORDER_SMALL = 32;
__global__ void k_order(const uint2* __restrict__ tk, uint32_t n,
                        const uint32_t* __restrict__ P, uint32_t* __restrict__ sid, uint32_t* __restrict__ skey,
                        uint32_t* __restrict__ inv, uint32_t* __restrict__ big, uint32_t* __restrict__ nbig,
                        uint32_t nper)
{
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint2 e = tk[s];
    const uint32_t v = e.x, k = e.y;
    const uint32_t lo = P[k], hi = P[k + 1];
    uint32_t pos = s;
    if (hi - lo > ORDER_SMALL) {
        if (s == lo) {
            const uint32_t q = atomicAdd(nbig, 1u);
            big[2 * q] = lo;
            big[2 * q + 1] = hi;
        }
        return;
    }
    if (hi - lo > 1) {
        uint32_t rank = 0;
        for (uint32_t t = lo; t < hi; ++t) rank += tk[t].x < v;
        pos = lo + rank;
    }
    sid[pos] = v % nper;  // the graph's own vertex id (batched calls: B graphs of nper points)
    skey[pos] = k;
    inv[v] = pos;
}

// the cells k_order listed: one block per cell (grid-stride over the list), LSD radix sort of
// the cell's vertex ids by 8-bit digits, each pass a stable scatter (per-warp match + per-digit
// prefix over the block's warps), ping-ponging between sid[lo..hi) and tmp[lo..hi) (the key
// array, free after k_scatter).  O(c) per pass per cell.
constexpr int OB_THREADS = 256, OB_WARPS = OB_THREADS / 32;
__global__ void __launch_bounds__(OB_THREADS) k_order_big(const uint2* __restrict__ tk, int passes,
                                                         const uint32_t* __restrict__ big,
                                                         const uint32_t* __restrict__ nbig,
                                                         uint32_t* __restrict__ sid, uint32_t* __restrict__ skey,
                                                         uint32_t* __restrict__ inv, uint32_t* __restrict__ tmp,
                                                         uint32_t nper)
{
    __shared__ uint32_t base[256];
    __shared__ uint32_t wcnt[OB_WARPS][256];
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t nb = *nbig;
    for (uint32_t q = blockIdx.x; q < nb; q += gridDim.x) {
        const uint32_t lo = big[2 * q], hi = big[2 * q + 1], c = hi - lo, key = tk[lo].y;
        for (int pass = 0; pass < passes; ++pass) {
            const int sh = 8 * pass;
            // source of this pass: tk ids (pass 0), then alternately sid / tmp
            const uint32_t* src = pass == 0 ? nullptr : ((pass & 1) ? sid : tmp);
            uint32_t* dst = (pass & 1) ? tmp : sid;
            for (int k = tid; k < 256; k += OB_THREADS) base[k] = 0;
            for (int k = tid; k < OB_WARPS * 256; k += OB_THREADS) (&wcnt[0][0])[k] = 0;
            __syncthreads();
            for (uint32_t t = tid; t < c; t += OB_THREADS) {
                const uint32_t id = src ? src[lo + t] : tk[lo + t].x;
                atomicAdd(&base[(id >> sh) & 255u], 1u);
            }
            __syncthreads();
            if (tid == 0) {  // exclusive scan of the digit histogram (256 entries)
                uint32_t acc = 0;
                for (int k = 0; k < 256; ++k) {
                    const uint32_t x = base[k];
                    base[k] = acc;
                    acc += x;
                }
            }
            __syncthreads();
            for (uint32_t t0 = 0; t0 < c; t0 += OB_THREADS) {
                const uint32_t t = t0 + tid;
                const bool ok = t < c;
                uint32_t id = 0, dg = 0, wr = 0;
                const unsigned act = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    id = src ? src[lo + t] : tk[lo + t].x;
                    dg = (id >> sh) & 255u;
                    const unsigned peers = __match_any_sync(act, dg);
                    wr = __popc(peers & ((1u << lane) - 1u));
                    if (wr == 0) wcnt[warp][dg] = __popc(peers);
                }
                __syncthreads();
                for (int k = tid; k < 256; k += OB_THREADS) {  // per digit: prefix over the warps
                    uint32_t run = base[k];
                    for (int w2 = 0; w2 < OB_WARPS; ++w2) {
                        const uint32_t x = wcnt[w2][k];
                        wcnt[w2][k] = run;
                        run += x;
                    }
                    base[k] = run;
                }
                __syncthreads();
                if (ok) dst[lo + wcnt[warp][dg] + wr] = id;
                __syncthreads();
                for (int k = tid; k < OB_WARPS * 256; k += OB_THREADS) (&wcnt[0][0])[k] = 0;
                __syncthreads();
            }
        }
        const uint32_t* fin = (passes & 1) ? sid : tmp;
        for (uint32_t t = tid; t < c; t += OB_THREADS) {
            const uint32_t v = fin[lo + t];
            sid[lo + t] = v % nper;
            skey[lo + t] = key;
            inv[v] = lo + t;
        }
        __syncthreads();
    }
}

// sorted point records rec[pos] = (x_0, .., x_{d-1}, w): coalesced reads in vertex order,
// one aligned 16/32/48-byte record write per vertex
template <int D>
__global__ void k_place(const uint32_t* __restrict__ inv, uint32_t n, const double* __restrict__ w0,
                        const double* __restrict__ x0, double* __restrict__ rec, const double* const* wb = nullptr,
                        const double* const* xb = nullptr)
{
    const unsigned g = blockIdx.y;  // batched: graph g's points are entries g n .. g n + n - 1 of inv
    const double* __restrict__ w = wb ? wb[g] : w0;
    const double* __restrict__ x = xb ? xb[g] : x0;
    inv += (size_t)g * n;
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    constexpr int RW = Geo<D>::RECW;
    double r[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) r[k] = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) r[k] = x[(size_t)k * n + v];
    r[D] = w[v];
    double2* dst = reinterpret_cast<double2*>(rec + (size_t)inv[v] * RW);
#pragma unroll
    for (int k = 0; k < RW / 2; ++k) dst[k] = make_double2(r[2 * k], r[2 * k + 1]);
}


// ======================================================================================
// Host side
// ======================================================================================
thread_local std::string g_last_cuda;
thread_local girg_timings g_timings;

// CUDA events around the phases of one call (recorded on the call's stream)
// Per-call host resources (timing events, a page-locked staging buffer) come from a process-wide
// pool: a call borrows one set and returns it, so repeated and concurrent calls (girg_edges_batch)
// do not create and destroy driver objects every time.
struct HostRes {
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    char* pinned = nullptr;  // page-locked staging (plan upload, status download)
    size_t cap = 0;
};

static std::mutex g_res_mu;
static std::vector<HostRes*> g_res_free;

struct PhaseEvents {
    HostRes* r = nullptr;
    cudaEvent_t* ev = nullptr;
    PhaseEvents()
    {
        {
            std::lock_guard<std::mutex> lk(g_res_mu);
            if (!g_res_free.empty()) {
                r = g_res_free.back();
                g_res_free.pop_back();
            }
        }
        if (!r) {
            r = new HostRes;
            for (auto& e : r->ev) cudaEventCreate(&e);
        }
        ev = r->ev;
    }
    ~PhaseEvents()
    {
        std::lock_guard<std::mutex> lk(g_res_mu);
        g_res_free.push_back(r);
    }
    // page-locked staging of at least `bytes` (valid until the next staging() of this call)
    char* staging(size_t bytes)
    {
        if (r->cap < bytes) {
            if (r->pinned) cudaFreeHost(r->pinned);
            r->pinned = nullptr;
            r->cap = 0;
            const size_t want = std::max<size_t>(bytes, 1 << 16);
            if (cudaHostAlloc((void**)&r->pinned, want, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            r->cap = want;
        }
        return r->pinned;
    }
    void record(int k, cudaStream_t st) { cudaEventRecord(ev[k], st); }
    double ms(int a, int b) const
    {
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[a], ev[b]);
        return (double)t;
    }
};

struct CudaFail {
    cudaError_t e;
};

#define GCHECK(x)                                  \
    do {                                           \
        cudaError_t e_ = (x);                      \
        if (e_ != cudaSuccess) throw CudaFail{e_}; \
    } while (0)

static void pool_keep(int dev)
{
    static bool done[64] = {};
    if (dev < 64 && !done[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done[dev] = true;
    }
}

// stream-ordered scratch allocations released in the destructor
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        pool_keep(dev);
    }
    char* arena = nullptr;  // one block carved by alloc() (reserve()); 256-B aligned pieces
    size_t acap = 0, aoff = 0;
    static size_t rounded(size_t bytes) { return (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255; }
    void reserve(size_t bytes)
    {
        arena = alloc<char>(bytes);
        acap = bytes;
        aoff = 0;
    }
    template <class T>
    T* alloc(size_t count)
    {
        const size_t r = rounded(count * sizeof(T));
        if (arena && aoff + r <= acap) {
            T* q = (T*)(arena + aoff);
            aoff += r;
            return q;
        }
        void* p = nullptr;
        const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
        cudaError_t e = cudaMallocAsync(&p, bytes, st);
        if (e == cudaErrorMemoryAllocation) throw CudaFail{e};
        GCHECK(e);
        ptrs.push_back(p);
        return (T*)p;
    }
    ~Scratch()
    {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

static inline unsigned grid_for(uint64_t n, unsigned threads) { return (unsigned)((n + threads - 1) / threads); }

// round a 256-bit non-negative integer (4 x u64, little endian) times 2^e2 to double (RNE)
__host__ __device__ inline int clz64(unsigned long long x)
{
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

__host__ __device__ inline double round_u256(const unsigned long long a[4], int e2)
{
    int top = -1;
    for (int k = 3; k >= 0 && top < 0; --k)
        if (a[k]) top = 64 * k + 63 - clz64(a[k]);
    if (top < 0) return 0.0;
    unsigned long long mant = 0;
    const int lo = top - 52 > 0 ? top - 52 : 0;
    for (int b = top; b >= lo; --b) mant = (mant << 1) | ((a[b / 64] >> (b % 64)) & 1ull);
    if (top <= 52) return ldexp((double)mant, e2);
    const unsigned rnd = (unsigned)((a[(top - 53) / 64] >> ((top - 53) % 64)) & 1ull);
    bool sticky = false;
    for (int b = top - 54; b >= 0 && !sticky; --b) sticky = ((a[b / 64] >> (b % 64)) & 1ull) != 0;
    int t = top;
    if (rnd && (sticky || (mant & 1ull))) {
        ++mant;
        if (mant == (1ull << 53)) { mant >>= 1; ++t; }
    }
    return ldexp((double)mant, t - 52 + e2);
}

// exact W = sum_b part_b * 2^(e_b - 52), rounded once (R3)
__host__ __device__ inline double exact_W(const WPartial* parts, size_t nparts, int emin)
{
    unsigned long long acc[4] = {0, 0, 0, 0};
    for (size_t b = 0; b < nparts; ++b) {
        const WPartial& q = parts[b];
        if (q.e_b == INT_MAX) continue;  // empty block
        const int sh = q.e_b - emin;       // 0..63
        unsigned long long v[4] = {0, 0, 0, 0};
        if (sh == 0) {
            v[0] = q.lo; v[1] = q.hi;
        } else {
            v[0] = q.lo << sh;
            v[1] = (q.hi << sh) | (q.lo >> (64 - sh));
            v[2] = q.hi >> (64 - sh);
        }
        unsigned long long carry = 0;
        for (int k = 0; k < 4; ++k) {
            const unsigned long long s1 = acc[k] + v[k];
            const unsigned long long c1 = s1 < acc[k];
            const unsigned long long s2 = s1 + carry;
            const unsigned long long c2 = s2 < s1;
            acc[k] = s2;
            carry = c1 + c2;
        }
    }
    return round_u256(acc, emin - 52);
}
static double exact_W(const std::vector<WPartial>& parts, int emin) { return exact_W(parts.data(), parts.size(), emin); }

struct HostPlan {
    Plan p;
    std::vector<TabEntry> tab;
    std::vector<uint16_t> tasks;
    uint64_t K = 0;
    double W = 0;
};

// H6: layers, levels and bound tables; R5-R7, R9, R10.
// R27 (refined type-II bound): level l of layer pair (i, j) is refined where it pays -- d = 2, 3,
// T > 0, l < CL(i,j) (no type-I events on that level, and l + 1 <= I(i)) and at least REF_X points
// of layer i per level-l cell on average (R27; the oracle's ref_level()).
constexpr long REF_X = 4096;  // B200 sweep optimum (profiles/r02/refined/): 1024..16384 within 1 %, 8 is 40 % slower
static std::atomic<int> g_ref_x{0};  // TEST HOOK (girg_debug_set_ref_x): 0 = REF_X, k > 0 = k points, -1 = every l < CL
static bool ref_level(int scheme, int d, double T, int l, int cl, uint64_t cnt_i)
{
    const long x = g_ref_x.load() == 0 ? REF_X : (long)g_ref_x.load();
    return scheme == SCHEME_REFINED && (d == 2 || d == 3) && T > 0.0 && l < cl &&
           (x < 0 || cnt_i >= ((uint64_t)x << (d * l)));
}

static int make_plan(const std::vector<uint32_t>& hist, const std::vector<WPartial>& parts, uint64_t n, int d,
                     double T, double kappa, HostPlan& hp, double s_override = 0.0, int scheme = SCHEME_MERGED)
{
    Plan& p = hp.p;
    std::memset(&p, 0, sizeof(p));
    int emin = INT_MAX, emax = INT_MIN;
    for (int b = 0; b < HIST_BINS; ++b)
        if (hist[b]) {
            emin = std::min(emin, b - EXP_BIAS);
            emax = std::max(emax, b - EXP_BIAS);
        }
    if (emin == INT_MAX) return GIRG_EINVAL;
    if (emax - emin + 1 > MAXL) return GIRG_ERANGE;
    hp.W = exact_W(parts, emin);
    p.L = emax - emin + 1;
    p.d = d;
    p.e_min = emin;
    p.T = T;
    p.invT = T > 0.0 ? 1.0 / T : 0.0;
    p.s = s_override > 0.0 ? s_override : kappa / hp.W;  // s_override: the HRG's dominating GIRG (R25)
    for (int i = 0; i < p.L; ++i) p.cnt[i] = hist[emin + i + EXP_BIAS];
    int Ln = 0;
    while (std::ldexp(1.0, d * Ln) < (double)n) ++Ln;
    const int Lmax = std::min(Ln + 1, 32 / d);
    int maxCL = 0;
    for (int i = 0; i < p.L; ++i)
        for (int j = 0; j < p.L; ++j) {
            const double qbar = std::ldexp(1.0, 2 * emin + i + j + 2) * p.s;
            int cl = 0;
            for (int l = Lmax; l >= 0; --l)
                if (std::ldexp(1.0, -d * l) >= qbar) { cl = l; break; }
            p.CL[i * MAXL + j] = (uint8_t)cl;
        }
    for (int i = 0; i < p.L; ++i) {
        int I = 0;
        if (p.cnt[i])
            for (int j = 0; j < p.L; ++j)
                if (p.cnt[j]) {
                    I = std::max(I, (int)p.CL[i * MAXL + j]);
                    maxCL = std::max(maxCL, (int)p.CL[i * MAXL + j]);
                }
        if (d * I > 31) return GIRG_ERANGE;
        p.I[i] = (uint8_t)I;
    }
    p.maxCL = maxCL;
    uint64_t K = 0, ls = 0;
    for (int i = 0; i < p.L; ++i) {
        p.base[i] = (uint32_t)K;
        p.lstart[i] = (uint32_t)ls;
        K += 1ull << (d * p.I[i]);
        ls += p.cnt[i];
        if (K >= 0xFFFFFFFFull) return GIRG_ERANGE;
    }
    p.base[p.L] = (uint32_t)K;
    p.lstart[p.L] = (uint32_t)ls;
    hp.K = K;
    hp.tab.clear();
    if (T > 0.0) {
        for (int i = 0; i < p.L; ++i)
            for (int j = i; j < p.L; ++j) {
                const int cl = p.CL[i * MAXL + j];
                p.tab_off[i * MAXL + j] = (uint32_t)hp.tab.size();
                if (!p.cnt[i] || !p.cnt[j] || cl < 2) continue;
                const double qbar = std::ldexp(1.0, 2 * emin + i + j + 2) * p.s;
                // REFINED plans: 5 entries per level -- classes 2, 3, then the refined classes
                // h = 2, 3, 4 half-cells: mind^d = h^d 2^(-d(l+1)) (exact; R27)
                const int nk = scheme == SCHEME_REFINED ? 5 : 2;
                for (int l = 2; l <= cl; ++l)
                    for (int k = 0; k < nk; ++k) {
                        double mind_d = std::ldexp(1.0, -d * l + d * k);  // ((k+1) 2^-l)^d
                        if (k >= 2) {
                            double hd = 1.0;
                            for (int q = 0; q < d; ++q) hd *= (double)k;  // h = k - 2 + 2
                            mind_d = std::ldexp(hd, -d * (l + 1));
                        }
                        const double ratio = qbar / mind_d;
                        TabEntry e;
                        e.pbar = ratio >= 1.0 ? 1.0 : std::pow(ratio, p.invT);
                        e.Lbar = std::log1p(-e.pbar);
                        int c2 = 0, c2m = 0;
                        if (e.pbar > 0.0) {
                            c2 = std::min(62, std::max(0, 1 - std::ilogb(e.pbar)));   // R10
                            c2m = std::min(62, std::max(0, GIRG_CHUNK_SHIFT - std::ilogb(e.pbar)));  // R22
                        }
                        e.clog2 = c2;
                        e.clog2m = c2m;
                        e.il2 = e.pbar < 1.0 ? M_LN2 / e.Lbar : 0.0;
                        e.pad = 0.0;
                        hp.tab.push_back(e);
                    }
            }
    }
    if (hp.tab.empty()) hp.tab.push_back(TabEntry{0, 0, 0, 0, 0, 0});
    // task lists: a task (j, l) of layer i is a cell Cg of layer i on level
    // lg = max(0, l - G) (G = Geo<D>::G) with its level-l descendants; it is owned by the first
    // point of Cg: the one point of Cg whose first level lf (the coarsest level on which it is the
    // first point of its cell; it stays first on every finer level) is <= lg.  Type-I if
    // l == CL(i,j), type-II if 2 <= l (T > 0).
    // The list of (layer i, lf) is every task of layer i with lg >= lf: layer i's tasks are stored
    // once, by decreasing lg, and each list is a prefix of them (the order of the tasks in a list
    // only schedules the work; the edge set does not depend on it).
    hp.tasks.clear();
    const int G = d == 1 ? GIRG_G1 : (d == 2 ? GIRG_G2 : 1);  // Geo<D>::G
    std::vector<std::pair<int, uint16_t>> E;                  // (lg, task) of layer i
    for (int i = 0; i < p.L; ++i) {
        E.clear();
        if (p.cnt[i])
            for (int j = i; j < p.L; ++j) {
                if (!p.cnt[j]) continue;
                const int cl = p.CL[i * MAXL + j];
                for (int l = 0; l <= cl; ++l) {
                    const int lg = std::max(0, l - G);
                    const int t1 = l == cl, t2 = T > 0.0 && l >= 2;
                    if (!t1 && !t2) continue;
                    if (t2 && ref_level(scheme, d, T, l, cl, p.cnt[i])) {  // R27: one job per A cell on level l (bit 14)
                        E.emplace_back(l, (uint16_t)(j | (l << 6) | (t2 << 13) | (1 << 14)));
                        continue;
                    }
                    E.emplace_back(lg, (uint16_t)(j | (l << 6) | (t1 << 12) | (t2 << 13)));
                }
            }
        std::stable_sort(E.begin(), E.end(), [](const std::pair<int, uint16_t>& x, const std::pair<int, uint16_t>& y) {
            return x.first > y.first;
        });
        const uint32_t off = (uint32_t)hp.tasks.size();
        p.toff[i] = off;
        for (const auto& e : E) hp.tasks.push_back(e.second);
        if (E.size() > 0xFFFF) return GIRG_ERANGE;
        size_t c = E.size();
        for (int lf = 0; lf <= 32; ++lf) {
            while (c > 0 && E[c - 1].first < lf) --c;
            p.tcnt[i * 33 + lf] = (uint16_t)((p.cnt[i] && lf <= p.I[i]) ? c : 0);
        }
    }
    if (hp.tasks.empty()) hp.tasks.push_back(0);
    return GIRG_OK;
}

static int map_cuda(cudaError_t e)
{
    g_last_cuda = cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? GIRG_ENOMEM : GIRG_ECUDA;
}

// SM count of the current device (queried once per device)
static int device_sms()
{
    static std::mutex mu;
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

template <int D>
static void launch_index(const double* w, const double* x, uint32_t n, const Plan* d_plan, uint64_t K,
                         uint32_t* key, uint32_t* cnt, uint32_t* P, uint32_t* bsum, uint2* tk,
                         uint32_t* inv, uint32_t* sid, uint32_t* skey, double* rec, uint32_t* big, uint32_t* nbig,
                         int* d_err, cudaStream_t st)
{
    const uint64_t len = K + 1;
    GCHECK(cudaMemsetAsync(cnt, 0, len * sizeof(uint32_t), st));
    k_keys<D><<<grid_for(n, 256), 256, 0, st>>>(w, x, n, d_plan, key, cnt, d_err);
    const unsigned nb = grid_for(len, SCAN_TILE);
    k_scan_reduce<<<nb, SCAN_THREADS, 0, st>>>(cnt, len, bsum);
    k_scan_top<<<1, 1024, 0, st>>>(bsum, nb);
    k_scan_final<<<nb, SCAN_THREADS, 0, st>>>(cnt, len, bsum, P);
    k_scatter<<<grid_for(n, 256), 256, 0, st>>>(key, n, cnt, tk);
    k_order<<<grid_for(n, 256), 256, 0, st>>>(tk, n, P, sid, skey, inv, big, nbig, n);
    {
        int bits = 1;
        while (bits < 32 && (1ull << bits) < (unsigned long long)n) ++bits;
        const unsigned gb = (unsigned)std::min<uint64_t>((uint64_t)device_sms() * 4u, n / (ORDER_SMALL + 1) + 1);
        k_order_big<<<gb, OB_THREADS, 0, st>>>(tk, (bits + 7) / 8, big, nbig, sid, skey, inv, key, n);
    }
    k_place<D><<<grid_for(n, 256), 256, 0, st>>>(inv, n, w, x, rec);
    GCHECK(cudaGetLastError());
}

// dynamic shared memory opt-in; the attribute is per device, so the cache is keyed by
// (device, kernel)
template <class K>
static void smem_optin(K kern, size_t bytes)
{
    static thread_local std::vector<std::pair<int, const void*>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const void* f = (const void*)kern;
    for (const auto& q : done)
        if (q.first == dev && q.second == f) return;
    GCHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    GCHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    done.emplace_back(dev, f);
}

// the sampling kernel pair of an instantiation: the engine (T > 0) or the flat T = 0 loop
template <int D, int SCHEME, bool STATS, bool T0>
struct SampleKernels {
    static constexpr auto sample()
    {
        if constexpr (T0) return k_sample_t0<D, STATS>;
        else return k_sample<D, SCHEME, STATS>;
    }
    static constexpr auto big()
    {
        if constexpr (T0) return k_big_t0<D, STATS>;
        else return k_big<D, SCHEME, STATS>;
    }
};

template <int D, int SCHEME, bool STATS, bool T0 = false>
static void launch_sample_t(const SampleArgs& a, cudaStream_t st)
{
    using SK = SampleKernels<D, SCHEME, STATS, T0>;
    constexpr int WPB = Geo<D>::WPB, TPB = 32 * WPB;
    const size_t smem = sizeof(WarpSmem<D>) * WPB;
    smem_optin(SK::sample(), smem);
    smem_optin(SK::big(), smem);
    // SM count and occupancies queried once per instantiation (one GPU type per process)
    const int nsm = device_sms();
    static const int occ = [] {
        int v = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, SK::sample(), TPB, sizeof(WarpSmem<D>) * WPB);
        return v;
    }();
    static const int occ2 = [] {
        int v = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, SK::big(), TPB, sizeof(WarpSmem<D>) * WPB);
        return v;
    }();
    const unsigned wtiles = (a.ntiles + WPB - 1) / WPB;
    unsigned grid = std::max(1u, std::min<unsigned>(wtiles, (unsigned)(nsm * std::max(occ, 1))));
    if (const char* g = getenv("GIRG_SAMPLE_GRID")) grid = std::max(1u, std::min<unsigned>(wtiles, (unsigned)atoi(g)));
    static const bool sync_debug = getenv("GIRG_SYNC_DEBUG") != nullptr;
    static const char* wprof_path = getenv("GIRG_WARP_PROFILE");  // development: per-warp profile dump
    // k_big: a full wave, but no wider than k_sample's grid (small graphs leave the rest of the
    // GPU to concurrent calls, girg_edges_batch)
    const unsigned gbig = std::min<unsigned>(grid, (unsigned)(nsm * std::max(occ2, 1)));
    const size_t nwarps = (size_t)std::max(grid, gbig) * WPB;
    SampleArgs b = a;
    if (wprof_path) {
        GCHECK(cudaMallocAsync(&b.wprof, 2 * nwarps * 4 * sizeof(unsigned long long), st));
        GCHECK(cudaMemsetAsync(b.wprof, 0, 2 * nwarps * 4 * sizeof(unsigned long long), st));
    }
    SK::sample()<<<grid, TPB, smem, st>>>(b);
    GCHECK(cudaGetLastError());
    if (sync_debug) {
        cudaError_t e = cudaStreamSynchronize(st);
        fprintf(stderr, "[girg] k_sample<%d,%d,%d> grid %u smem %zu occ %d: %s\n", D, SCHEME, (int)STATS, grid, smem,
                occ, cudaGetErrorString(e));
        GCHECK(e);
    }
    if (b.wprof) b.wprof += nwarps * 4;
    SK::big()<<<gbig, TPB, smem, st>>>(b);
    GCHECK(cudaGetLastError());
    if (wprof_path) {
        std::vector<unsigned long long> h(2 * nwarps * 4);
        b.wprof -= nwarps * 4;
        GCHECK(cudaMemcpyAsync(h.data(), b.wprof, h.size() * 8, cudaMemcpyDeviceToHost, st));
        GCHECK(cudaStreamSynchronize(st));
        if (FILE* f = fopen(wprof_path, "wb")) {
            const unsigned long long hdr[4] = {nwarps, grid, gbig, (unsigned long long)WPB};
            fwrite(hdr, 8, 4, f);
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
        cudaFreeAsync(b.wprof, st);
    }
    if (sync_debug) {
        cudaError_t e = cudaStreamSynchronize(st);
        fprintf(stderr, "[girg] k_big<%d,%d,%d>: %s\n", D, SCHEME, (int)STATS, cudaGetErrorString(e));
        GCHECK(e);
    }
}

template <int D>
static void launch_sample(const SampleArgs& a, int scheme, cudaStream_t st)
{
    if (a.T == 0.0) {  // threshold model: no type-II events in either scheme, the flat loop
        if (a.stats) launch_sample_t<D, SCHEME_MERGED, true, true>(a, st);
        else launch_sample_t<D, SCHEME_MERGED, false, true>(a, st);
    } else if (scheme == SCHEME_EVENT) {
        if (a.stats) launch_sample_t<D, SCHEME_EVENT, true>(a, st);
        else launch_sample_t<D, SCHEME_EVENT, false>(a, st);
    } else if (scheme == SCHEME_REFINED && (D == 2 || D == 3)) {
        if constexpr (D == 2 || D == 3) {
            if (a.stats) launch_sample_t<D, SCHEME_REFINED, true>(a, st);
            else launch_sample_t<D, SCHEME_REFINED, false>(a, st);
        }
    } else {
        if (a.stats) launch_sample_t<D, SCHEME_MERGED, true>(a, st);
        else launch_sample_t<D, SCHEME_MERGED, false>(a, st);
    }
}

// One girg_edges call in three host stages, so that a batch can queue stage A (resp. B) of many
// graphs on several streams before waiting once:
//   A  weight statistics (k_wstats) + their read-back into page-locked staging        (async)
//   B  [after A's data arrived] host plan, one scratch block, plan upload, index build,
//      sampler, status read-back                                                       (async)
//   C  [after B's data arrived] status, item-queue regrowth (re-runs the sampler), outputs
static_assert(32 + sizeof(Counters) <= 128, "status block layout: counters end before the item counter");

struct EdgeCall {
    const double *w, *x;
    uint64_t n;
    int d;
    double T, kappa;
    uint64_t seed;
    int sl;
    uint64_t blo, bhi;
    uint32_t nranks = 0, rank = 0;  // interleaved ownership (nranks > 0) instead of a block range
    double s_override = 0.0;        // > 0: s fixed instead of kappa / W (HRG's dominating GIRG, R25)
    int scheme;
    uint32_t* edges;
    uint64_t cap;
    uint64_t* m_out;
    girg_stats* stats_out;
    cudaStream_t st;
    PhaseEvents PE;
    Scratch S;
    HostPlan hp;
    SampleArgs a;
    char* misc = nullptr;  // device status block (err, m, counters, queue counters)
    // TEST HOOK (girg_debug_index): device buffers that receive the sorted ids and the prefix array
    uint32_t* dbg_sid = nullptr;
    uint32_t* dbg_P = nullptr;
    uint64_t dbg_Pcap = 0;
    char* hmisc = nullptr;
    char hmisc_local[256];
    unsigned nb = 0;
    char* wst_dev = nullptr;  // k_wstats outputs: histogram, error flag, block partials
    char* wst_host = nullptr;
    std::vector<char> wst_pageable;
    size_t wst_bytes = 0;
    int rc = GIRG_OK;

    EdgeCall(const double* w_, const double* x_, uint64_t n_, int d_, double T_, double kappa_, uint64_t seed_,
             int sl_, uint64_t blo_, uint64_t bhi_, int scheme_, uint32_t* edges_, uint64_t cap_, uint64_t* m_out_,
             girg_stats* stats_out_, cudaStream_t st_)
        : w(w_), x(x_), n(n_), d(d_), T(T_), kappa(kappa_), seed(seed_), sl(sl_), blo(blo_), bhi(bhi_),
          scheme(scheme_), edges(edges_), cap(cap_), m_out(m_out_), stats_out(stats_out_), st(st_), S(st_)
    {
    }

    static int validate(const double* w, const double* x, uint64_t n, int d, double T, double kappa, int sl,
                        uint64_t blo, uint64_t bhi, int scheme, uint32_t* edges, uint64_t cap, uint64_t* m_out)
    {
        if (scheme != SCHEME_EVENT && scheme != SCHEME_MERGED && scheme != SCHEME_REFINED) return GIRG_EINVAL;
        if (!w || !x || !m_out || (cap && !edges)) return GIRG_EINVAL;
        if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5) return GIRG_EINVAL;
        if (!(T >= 0.0 && T < 1.0) || !(kappa > 0.0) || !std::isfinite(kappa)) return GIRG_EINVAL;
        if (sl < 0 || sl * d > 32 || blo >= bhi) return GIRG_EINVAL;
        return GIRG_OK;
    }

    void stage_a()
    {
        PE.record(0, st);
        nb = grid_for(n, WS_TILE);
        wst_bytes = HIST_BINS * sizeof(uint32_t) + 16 + nb * sizeof(WPartial);
        wst_dev = S.alloc<char>(wst_bytes);
        GCHECK(cudaMemsetAsync(wst_dev, 0, HIST_BINS * sizeof(uint32_t) + 16, st));
        k_wstats<<<nb, WS_THREADS, 0, st>>>(w, (uint32_t)n, (uint32_t*)wst_dev,
                                            (WPartial*)(wst_dev + HIST_BINS * sizeof(uint32_t) + 16),
                                            (int*)(wst_dev + HIST_BINS * sizeof(uint32_t)));
        GCHECK(cudaGetLastError());
        // staging sized for this read-back and (typically) the later plan upload: no reallocation
        wst_host = PE.staging(std::max<size_t>(wst_bytes, 1 << 20));
        if (!wst_host) {
            wst_pageable.resize(wst_bytes);
            wst_host = wst_pageable.data();
        }
        GCHECK(cudaMemcpyAsync(wst_host, wst_dev, wst_bytes, cudaMemcpyDeviceToHost, st));
    }

    void stage_b()
    {
        std::vector<uint32_t> hist((uint32_t*)wst_host, (uint32_t*)wst_host + HIST_BINS);
        int herr = 0;
        std::memcpy(&herr, wst_host + HIST_BINS * sizeof(uint32_t), sizeof(int));
        std::vector<WPartial> parts(nb);
        std::memcpy(parts.data(), wst_host + HIST_BINS * sizeof(uint32_t) + 16, nb * sizeof(WPartial));
        if (herr & ERR_WEIGHT) { rc = GIRG_EINVAL; return; }
        if (herr & ERR_WRANGE) { rc = GIRG_ERANGE; return; }
        // the refined bound exists for d = 2, 3 and T > 0 (R27); elsewhere REFINED is MERGED
        if (scheme == SCHEME_REFINED && !((d == 2 || d == 3) && T > 0.0)) scheme = SCHEME_MERGED;
        rc = make_plan(hist, parts, n, d, T, kappa, hp, s_override, scheme);
        if (rc) return;
        hp.p.sl = sl;
        hp.p.blo = blo;
        hp.p.bhi = bhi;
        const uint32_t n32 = (uint32_t)n;
        const uint64_t K = hp.K;
        // scratch: one stream-ordered block for everything this call needs
        const int recw = d == 1 ? 2 : (d <= 3 ? 4 : 6);
        const unsigned int items_cap = std::max<unsigned int>(1u << 18, n32 / 2);
        const size_t up_plan = Scratch::rounded(sizeof(Plan)), up_tab = Scratch::rounded(hp.tab.size() * sizeof(TabEntry)),
                     up_bytes = up_plan + up_tab + hp.tasks.size() * sizeof(uint16_t);
        S.reserve(Scratch::rounded(up_bytes) + Scratch::rounded(256) + 6 * Scratch::rounded(n * 4) +
                  2 * Scratch::rounded((K + 1) * 4) + Scratch::rounded((grid_for(K + 1, SCAN_TILE) + 1) * 4) +
                  Scratch::rounded((size_t)recw * n * 8) + Scratch::rounded((size_t)items_cap * sizeof(BigItem)) +
                  Scratch::rounded((2 * (n / (ORDER_SMALL + 1) + 1)) * 4));
        char* d_up = S.alloc<char>(up_bytes);
        Plan* d_plan = (Plan*)d_up;
        TabEntry* d_tab = (TabEntry*)(d_up + up_plan);
        uint16_t* d_tasks = (uint16_t*)(d_up + up_plan + up_tab);
        misc = S.alloc<char>(256);
        int* d_err = (int*)misc;
        uint32_t* key = S.alloc<uint32_t>(n);
        uint2* tk = S.alloc<uint2>(n);  // (id, key) pairs in slot order
        uint32_t* inv = S.alloc<uint32_t>(n);
        uint32_t* cnt = S.alloc<uint32_t>(K + 1);
        uint32_t* P = S.alloc<uint32_t>(K + 1);
        uint32_t* bsum = S.alloc<uint32_t>(grid_for(K + 1, SCAN_TILE) + 1);
        uint32_t* sid = S.alloc<uint32_t>(n);
        uint32_t* skey = S.alloc<uint32_t>(n);
        double* rec = S.alloc<double>((size_t)recw * n);
        BigItem* items = S.alloc<BigItem>(items_cap);
        uint32_t* big = S.alloc<uint32_t>(2 * (n / (ORDER_SMALL + 1) + 1));  // crowded cells for k_order_big
        uint32_t* nbig = (uint32_t*)(misc + 132);
        // plan, bound table and task lists in one upload from page-locked staging (the weight
        // statistics above are consumed); the staging tail receives the status block
        char* stage = PE.staging(up_bytes + 256);
        hmisc = stage ? stage + up_bytes : hmisc_local;
        if (stage) {
            std::memcpy(stage, &hp.p, plan_upload_bytes(hp.p));
            std::memcpy(stage + up_plan, hp.tab.data(), hp.tab.size() * sizeof(TabEntry));
            std::memcpy(stage + up_plan + up_tab, hp.tasks.data(), hp.tasks.size() * sizeof(uint16_t));
            GCHECK(cudaMemcpyAsync(d_up, stage, up_bytes, cudaMemcpyHostToDevice, st));
        } else {
            GCHECK(cudaMemcpyAsync(d_plan, &hp.p, plan_upload_bytes(hp.p), cudaMemcpyHostToDevice, st));
            GCHECK(cudaMemcpyAsync(d_tab, hp.tab.data(), hp.tab.size() * sizeof(TabEntry), cudaMemcpyHostToDevice, st));
            GCHECK(cudaMemcpyAsync(d_tasks, hp.tasks.data(), hp.tasks.size() * sizeof(uint16_t),
                                   cudaMemcpyHostToDevice, st));
            GCHECK(cudaStreamSynchronize(st));  // pageable sources must outlive the copies
        }
        GCHECK(cudaMemsetAsync(misc, 0, 256, st));
        PE.record(1, st);
        switch (d) {
            case 1: launch_index<1>(w, x, n32, d_plan, K, key, cnt, P, bsum, tk, inv, sid, skey, rec, big, nbig, d_err, st); break;
            case 2: launch_index<2>(w, x, n32, d_plan, K, key, cnt, P, bsum, tk, inv, sid, skey, rec, big, nbig, d_err, st); break;
            case 3: launch_index<3>(w, x, n32, d_plan, K, key, cnt, P, bsum, tk, inv, sid, skey, rec, big, nbig, d_err, st); break;
            case 4: launch_index<4>(w, x, n32, d_plan, K, key, cnt, P, bsum, tk, inv, sid, skey, rec, big, nbig, d_err, st); break;
            default: launch_index<5>(w, x, n32, d_plan, K, key, cnt, P, bsum, tk, inv, sid, skey, rec, big, nbig, d_err, st); break;
        }
        if (dbg_sid) GCHECK(cudaMemcpyAsync(dbg_sid, sid, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        if (dbg_P)
            GCHECK(cudaMemcpyAsync(dbg_P, P, std::min<uint64_t>(K + 1, dbg_Pcap) * sizeof(uint32_t),
                                   cudaMemcpyDeviceToDevice, st));
        a.pl = d_plan;
        a.tab = d_tab;
        a.tasks = d_tasks;
        a.skey = skey;
        a.rec = rec;
        a.sid = sid;
        a.P = P;
        a.n = n32;
        // small graphs: 8-point tiles, so that 4x more warps share the jobs (C1: 313 -> 1250 tiles)
        a.tile_pts = n32 < GIRG_SMALL_TILE_N ? 8u : 32u;
        if (const char* e = getenv("GIRG_TILE_PTS")) a.tile_pts = (uint32_t)std::max(1, std::min(32, atoi(e)));
        a.ntiles = (n32 + a.tile_pts - 1) / a.tile_pts;
        a.k0 = (uint32_t)seed;
        a.k1 = (uint32_t)(seed >> 32);
        a.edges = (uint2*)edges;
        a.cap = cap;
        a.m = (unsigned long long*)(misc + 16);
        a.tile_ctr = (unsigned int*)(misc + 24);
        a.nitems = (unsigned int*)(misc + 28);
        a.item_ctr = (unsigned int*)(misc + 128);  // after the counters (32 + sizeof(Counters) <= 128)
        a.stats = stats_out ? (Counters*)(misc + 32) : nullptr;
        a.err = d_err;
        a.items = items;
        a.items_cap = items_cap;
        a.nP = K + 1;
        a.ntab = (unsigned)hp.tab.size();
        a.ntasks = (unsigned)hp.tasks.size();
        a.big_work = big_work(d, n);
        a.item_work = item_work(d, n);
        if (const char* e = getenv("GIRG_BIG_WORK")) a.big_work = strtoull(e, nullptr, 10);
        if (const char* e = getenv("GIRG_ITEM_WORK")) a.item_work = strtoull(e, nullptr, 10);
        a.wprof = nullptr;
        a.dev_flags = 0;
        a.T = hp.p.T;
        a.s = hp.p.s;
        a.invT = hp.p.invT;
        a.sl = hp.p.sl;
        a.blo = hp.p.blo;
        a.bhi = hp.p.bhi;
        a.nranks = nranks;
        a.rank = rank;
        a.sharded = nranks > 0 || blo > 0 || bhi < (1ull << (d * sl)) || sl * d >= 64;
        a.p0 = 0;
        if (const char* e = getenv("GIRG_DEV_FLAGS")) a.dev_flags = (unsigned)atoi(e);
        PE.record(2, st);
        sample_and_fetch();
    }

    void sample_and_fetch()
    {
        switch (d) {
            case 1: launch_sample<1>(a, scheme, st); break;
            case 2: launch_sample<2>(a, scheme, st); break;
            case 3: launch_sample<3>(a, scheme, st); break;
            case 4: launch_sample<4>(a, scheme, st); break;
            default: launch_sample<5>(a, scheme, st); break;
        }
        PE.record(3, st);
        GCHECK(cudaMemcpyAsync(hmisc, misc, 256, cudaMemcpyDeviceToHost, st));
    }

    int stage_c()
    {
        if (rc != GIRG_OK) return rc;
        for (int attempt = 0;; ++attempt) {
            int e0;
            unsigned int need;
            std::memcpy(&e0, hmisc, sizeof(int));
            std::memcpy(&need, hmisc + 28, sizeof(need));
            if (!(e0 & ERR_ITEMS) || attempt > 4) break;
            // the big-event item queue overflowed: grow it and re-run the (deterministic) sampler
            a.items_cap = need + (need >> 2) + 1024;
            a.items = S.alloc<BigItem>(a.items_cap);
            GCHECK(cudaMemsetAsync(misc, 0, 256, st));
            PE.record(2, st);
            sample_and_fetch();
            GCHECK(cudaStreamSynchronize(st));
        }
        g_timings.ms_wstats = PE.ms(0, 1);
        g_timings.ms_index = PE.ms(1, 2);
        g_timings.ms_sample = PE.ms(2, 3);
        g_timings.ms_total = PE.ms(0, 3);
        g_timings.launches = 11;  // k_wstats, k_keys, 3 x scan, k_scatter, k_order, k_order_big, k_place, k_sample, k_big
        g_timings.n = n;
        g_timings.key_space = hp.K;
        g_timings.d = d;
        int derr;
        unsigned long long m;
        Counters hc;
        std::memcpy(&derr, hmisc, sizeof(int));
        std::memcpy(&m, hmisc + 16, sizeof(m));
        std::memcpy(&hc, hmisc + 32, sizeof(hc));
        g_timings.m = m;
        if (derr & ERR_POS) return GIRG_EINVAL;
        if (derr & ERR_ITEMS) return GIRG_ENOMEM;
        *m_out = m;
        if (stats_out) {
            stats_out->cand1 = hc.cand1;
            stats_out->ev2 = hc.ev2;
            stats_out->chunks = hc.chunks;
            stats_out->draws = hc.draws;
            stats_out->landings = hc.landings;
            stats_out->edges1 = hc.edges1;
            stats_out->edges2 = hc.edges2;
            stats_out->neartie1 = hc.nt1;
            stats_out->neartie2 = hc.nt2;
            stats_out->fast_fallback = hc.fb;
            stats_out->fast_mismatch = hc.mm;
            stats_out->neartie_jump = hc.ntj;
            stats_out->layers = (uint64_t)hp.p.L;
            stats_out->key_space = hp.K;
        }
        return m > cap ? GIRG_ECAPACITY : GIRG_OK;
    }
};

static int edges_impl(const double* w, const double* x, uint64_t n, int d, double T, double kappa,
                      uint64_t seed, int sl, uint64_t blo, uint64_t bhi, int scheme, uint32_t* edges, uint64_t cap,
                      uint64_t* m_out, girg_stats* stats_out, cudaStream_t st, uint32_t nranks = 0,
                      uint32_t rank = 0, double s_override = 0.0)
{
    if (nranks > 0) {  // interleaved ownership: the block range is unused
        if (rank >= nranks) return GIRG_EINVAL;
        blo = 0;
        bhi = 1;
    }
    int v = EdgeCall::validate(w, x, n, d, T, kappa, sl, blo, bhi, scheme, edges, cap, m_out);
    if (v != GIRG_OK) return v;
    try {
        EdgeCall E(w, x, n, d, T, kappa, seed, sl, blo, bhi, scheme, edges, cap, m_out, stats_out, st);
        E.nranks = nranks;
        E.rank = rank;
        E.s_override = s_override;
        E.stage_a();
        GCHECK(cudaStreamSynchronize(st));
        E.stage_b();
        if (E.rc != GIRG_OK) return E.rc;
        GCHECK(cudaStreamSynchronize(st));
        return E.stage_c();
    } catch (const CudaFail& f) {
        return map_cuda(f.e);
    } catch (const std::bad_alloc&) {
        return GIRG_ENOMEM;
    } catch (...) {
        g_last_cuda = "internal error: unexpected exception";
        return GIRG_ECUDA;
    }
}

// ======================================================================================
// Average-degree estimation (Sec. 5.1, App. B.2), boundary call, not
// on the timed edge path.  Device: exact W and wmax (k_wstats), then one pass that sums over
// the vertices with w <= tau (the tail, never saturated for the kappas tried) and compacts the
// heavier candidates; host: the monotone search on f with E_R evaluated in O(|R|) over the
// sorted candidates (same decomposition as DESIGN.md R12).
// ======================================================================================
// Device part: ONE cooperative launch (grid-wide barriers) and one synchronisation:
//   1  global e_min / w_max / input checks;  2  exact W (192-bit per-thread fixed point relative
//   to e_min, block partials summed in 256 bits by block 0 and rounded once, R3);  3  kappa0,
//   a0 = 2^d kappa0 / W and the tail threshold tau = 1/(2 a0 w_max): vertices with w <= tau are
//   never saturated for kappa <= 2 kappa0, so their power sums (sum w, w^2, (w/wmax)^(1/T),
//   (w/wmax)^(2/T)) are kappa-independent and summed once (fixed order: thread, warp, block,
//   blocks in index order); heavier vertices are compacted.
// Host part: the exponential search and bisection on f (same decomposition as the oracle's
// or_f, R12) with E_R in O(|R|) over a LAZILY sorted prefix of the candidates (the
// paper's App. B.2 device): each f(kappa) needs only R(kappa) = {w > 1/(a w_max)}
// sorted; the unsorted rest enters through its sums.  A kappa outside the range covered by tau
// re-launches the device pass with a smaller tau.
constexpr int SC_THREADS = 256;
struct Acc192 {
    unsigned long long v[3];
};
struct TailSums {
    double s1, s2, z1, z2;  // sum w, sum w^2, sum (w/wmax)^(1/T), sum (w/wmax)^(2/T) over w <= tau
};
struct ScaleCtl {
    int emin;  // global minimum exponent (atomicMin)
    int err;   // ERR_WEIGHT / ERR_WRANGE
    unsigned long long wmax_bits;
    unsigned int ncand;  // candidates (w > tau) seen
    int pad;
    double W, wmax, tau, kappa0;
    TailSums tail;
};

__device__ __forceinline__ void add192(Acc192& a, unsigned long long lo, unsigned long long hi)
{
    const unsigned long long t0 = a.v[0] + lo;
    const unsigned long long c0 = t0 < lo;
    const unsigned long long t1 = a.v[1] + hi;
    const unsigned long long c1 = t1 < hi;
    const unsigned long long t1b = t1 + c0;
    const unsigned long long c1b = t1b < t1;
    a.v[0] = t0;
    a.v[1] = t1b;
    a.v[2] += c1 + c1b;
}
__device__ __forceinline__ void add192(Acc192& a, const Acc192& b)
{
    add192(a, b.v[0], b.v[1]);
    a.v[2] += b.v[2];
}

__global__ void __launch_bounds__(SC_THREADS) k_scale(const double* __restrict__ w, uint32_t n, int d, double T,
                                                      double avg_deg, double beta, double tau_in,
                                                      Acc192* __restrict__ wpart, TailSums* __restrict__ tpart,
                                                      double* __restrict__ cand, uint32_t cap, ScaleCtl* ctl)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const unsigned tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + tid, gstride = (size_t)gridDim.x * blockDim.x;
    __shared__ Acc192 sh_a[SC_THREADS / 32];
    __shared__ double sh_t[4][SC_THREADS / 32];
    // ---- 1: e_min, w_max, input checks ----
    {
        int emin = INT_MAX, bad = 0;
        unsigned long long wmb = 0;
        for (size_t v = gtid; v < n; v += gstride) {
            const unsigned long long bits = __double_as_longlong(w[v]);
            const int ef = (int)((bits >> 52) & 0x7ff);
            if ((bits >> 63) || ef == 0 || ef == 0x7ff) { bad |= ERR_WEIGHT; continue; }
            emin = min(emin, ef - EXP_BIAS);
            wmb = max(wmb, bits);
        }
        for (int o = 16; o; o >>= 1) {
            emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
            wmb = max(wmb, __shfl_xor_sync(0xffffffffu, wmb, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
        if (lane == 0) {
            atomicMin(&ctl->emin, emin);
            atomicMax(&ctl->wmax_bits, wmb);
            if (bad) atomicOr(&ctl->err, bad);
        }
    }
    grid.sync();
    const int emin = ctl->emin;
    // ---- 2: exact W partials (192-bit per thread, relative to the global e_min) ----
    {
        Acc192 acc = {{0, 0, 0}};
        int bad = 0;
        for (size_t v = gtid; v < n; v += gstride) {
            const unsigned long long bits = __double_as_longlong(w[v]);
            const int ef = (int)((bits >> 52) & 0x7ff);
            if ((bits >> 63) || ef == 0 || ef == 0x7ff) continue;
            const int sh = ef - EXP_BIAS - emin;
            if (sh > 63) { bad = ERR_WRANGE; continue; }
            const unsigned long long m = (bits & ((1ull << 52) - 1)) | (1ull << 52);
            add192(acc, m << sh, sh ? (m >> (64 - sh)) : 0ull);
        }
        if (bad) atomicOr(&ctl->err, bad);
        for (int o = 16; o; o >>= 1) {
            Acc192 b;
            for (int k = 0; k < 3; ++k) b.v[k] = __shfl_down_sync(0xffffffffu, acc.v[k], o);
            add192(acc, b);
        }
        if (lane == 0) sh_a[wid] = acc;
        __syncthreads();
        if (tid == 0) {
            Acc192 t = {{0, 0, 0}};
            for (int k = 0; k < SC_THREADS / 32; ++k) add192(t, sh_a[k]);
            wpart[blockIdx.x] = t;
        }
    }
    grid.sync();
    // ---- 3: W, kappa0, tau (block 0, thread 0) ----
    if (blockIdx.x == 0 && tid == 0) {
        unsigned long long acc4[4] = {0, 0, 0, 0};
        for (unsigned b = 0; b < gridDim.x; ++b) {
            const Acc192& q = wpart[b];
            unsigned long long carry = 0;
            for (int k = 0; k < 4; ++k) {
                const unsigned long long add = k < 3 ? q.v[k] : 0ull;
                const unsigned long long s1 = acc4[k] + add;
                const unsigned long long c1 = s1 < acc4[k];
                const unsigned long long s2 = s1 + carry;
                const unsigned long long c2 = s2 < s1;
                acc4[k] = s2;
                carry = c1 + c2;
            }
        }
        ctl->W = round_u256(acc4, emin - 52);
        ctl->wmax = __longlong_as_double((long long)ctl->wmax_bits);
        const double Ew = (beta - 1.0) / (beta - 2.0);
        const double k0 = avg_deg * (1.0 - T) / (ldexp(1.0, d) * Ew);
        ctl->kappa0 = k0;
        const double a0 = ldexp(k0, d) / ctl->W;
        ctl->tau = tau_in > 0.0 ? tau_in : 0.5 / (a0 * ctl->wmax);
        ctl->ncand = 0;
    }
    grid.sync();
    if (ctl->err) return;
    const double tau = ctl->tau, wmax = ctl->wmax, invT = T > 0.0 ? 1.0 / T : 0.0;
    // ---- 4: tail power sums and candidates ----
    double a1 = 0, a2 = 0, b1 = 0, b2 = 0;
    for (size_t v = gtid; v < n; v += gstride) {
        const double wv = w[v];
        if (wv <= tau) {
            a1 += wv;
            a2 += wv * wv;
            if (invT > 0.0) {
                const double z = pow(wv / wmax, invT);
                b1 += z;
                b2 += z * z;
            }
        } else {
            const uint32_t k = atomicAdd(&ctl->ncand, 1u);
            if (k < cap) {
                cand[k] = wv;
                cand[cap + k] = invT > 0.0 ? pow(wv / wmax, invT) : 0.0;  // zeta (the host search's power terms)
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        a1 += __shfl_down_sync(0xffffffffu, a1, o);
        a2 += __shfl_down_sync(0xffffffffu, a2, o);
        b1 += __shfl_down_sync(0xffffffffu, b1, o);
        b2 += __shfl_down_sync(0xffffffffu, b2, o);
    }
    if (lane == 0) { sh_t[0][wid] = a1; sh_t[1][wid] = a2; sh_t[2][wid] = b1; sh_t[3][wid] = b2; }
    __syncthreads();
    if (tid == 0) {
        TailSums t = {0, 0, 0, 0};
        for (int k = 0; k < SC_THREADS / 32; ++k) { t.s1 += sh_t[0][k]; t.s2 += sh_t[1][k]; t.z1 += sh_t[2][k]; t.z2 += sh_t[3][k]; }
        tpart[blockIdx.x] = t;
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {  // fixed-order sum of the block partials
        TailSums t = {0, 0, 0, 0};
        for (unsigned b = 0; b < gridDim.x; ++b) { t.s1 += tpart[b].s1; t.s2 += tpart[b].s2; t.z1 += tpart[b].z1; t.z2 += tpart[b].z2; }
        ctl->tail = t;
    }
}

// host: f(kappa) over the candidates with a lazily sorted prefix
struct LazyEstimator {
    uint64_t n;
    int d;
    double T, W, wmax, tau;
    TailSums tail;
    std::vector<double> C;  // candidates: C[0, L) sorted decreasing, C[L, end) unsorted and < C[L-1]
    std::vector<double> Z;  // their zeta = (c / wmax)^(1/T), computed by the device pass, permuted with C
    size_t L = 0;
    std::vector<double> zeta, suf1, suf2, sufz1, sufz2;  // over C[0, L): zeta and suffix sums (from k to L)
    std::vector<double> pre1, prez;                      // prefix sums of C and zeta over C[0, L)
    double r1 = 0, r2 = 0, rz1 = 0, rz2 = 0;             // sums over the unsorted rest
    double rest_max = 0;                                 // largest unsorted candidate

    void reset()
    {
        // all candidates sorted once (radix_desc: a few linear passes, no comparison sort of the
        // growing prefix), so cover() below has nothing left to do
        radix_desc(C, Z);
        L = C.size();
        zeta = Z;
        suf1.assign(L + 1, 0.0);
        suf2.assign(L + 1, 0.0);
        sufz1.assign(L + 1, 0.0);
        sufz2.assign(L + 1, 0.0);
        for (size_t k = L; k-- > 0;) {  // ascending weights: small terms first
            suf1[k] = suf1[k + 1] + C[k];
            suf2[k] = suf2[k + 1] + C[k] * C[k];
            sufz1[k] = sufz1[k + 1] + zeta[k];
            sufz2[k] = sufz2[k + 1] + zeta[k] * zeta[k];
        }
        pre1.assign(L + 1, 0.0);
        prez.assign(L + 1, 0.0);
        for (size_t k = 0; k < L; ++k) {
            pre1[k + 1] = pre1[k] + C[k];
            prez[k + 1] = prez[k] + zeta[k];
        }
        rest_sums();
    }
    // sort the candidates (positive doubles: their bit patterns order like their values)
    // decreasingly, their zeta along: LSD radix on ~bits, 11-bit digits, passes that keep every key
    // in one bucket skipped
    static void radix_desc(std::vector<double>& C, std::vector<double>& Z)
    {
        const size_t N = C.size();
        if (N < 2) return;
        std::vector<uint64_t> k(N), k2(N);
        std::vector<double> z2(N);
        for (size_t i = 0; i < N; ++i) {
            uint64_t b;
            std::memcpy(&b, &C[i], 8);
            k[i] = ~b;
        }
        constexpr int BITS = 11;
        constexpr uint64_t NB = 1ull << BITS;
        std::vector<uint32_t> cnt(NB);
        // digits of the top 33 bits only (sign, exponent, 21 mantissa bits: keys equal there differ
        // by < 2^-21 relative and are rare); the insertion pass below orders them by the full key
        for (int sh = 31; sh < 64; sh += BITS) {
            std::fill(cnt.begin(), cnt.end(), 0u);
            for (size_t i = 0; i < N; ++i) ++cnt[(k[i] >> sh) & (NB - 1)];
            if (cnt[(k[0] >> sh) & (NB - 1)] == N) continue;
            uint32_t acc = 0;
            for (uint64_t b = 0; b < NB; ++b) {
                const uint32_t c = cnt[b];
                cnt[b] = acc;
                acc += c;
            }
            for (size_t i = 0; i < N; ++i) {
                const uint32_t p = cnt[(k[i] >> sh) & (NB - 1)]++;
                k2[p] = k[i];
                z2[p] = Z[i];
            }
            k.swap(k2);
            Z.swap(z2);
        }
        for (size_t i = 1; i < N; ++i) {  // full-key order inside runs of equal top bits
            const uint64_t ki = k[i];
            if (!(k[i - 1] > ki)) continue;
            const double zi = Z[i];
            size_t j = i;
            while (j > 0 && k[j - 1] > ki) {
                k[j] = k[j - 1];
                Z[j] = Z[j - 1];
                --j;
            }
            k[j] = ki;
            Z[j] = zi;
        }
        for (size_t i = 0; i < N; ++i) {
            const uint64_t b = ~k[i];
            std::memcpy(&C[i], &b, 8);
        }
    }
    void rest_sums()
    {
        r1 = r2 = rz1 = rz2 = 0.0;
        rest_max = 0.0;
        for (size_t k = L; k < C.size(); ++k) {
            const double z = Z[k];
            r1 += C[k];
            r2 += C[k] * C[k];
            rz1 += z;
            rz2 += z * z;
            rest_max = std::max(rest_max, C[k]);
        }
    }
    // make C[0, L) hold every candidate > t, sorted decreasingly (the rest stays unsorted and
    // below every sorted element, so a smaller t only appends)
    void cover(double t)
    {
        if (L == C.size() || !(rest_max > t)) return;
        std::vector<std::pair<double, double>> cz(C.size() - L);
        for (size_t k = L; k < C.size(); ++k) cz[k - L] = {C[k], Z[k]};
        auto mid = std::partition(cz.begin(), cz.end(), [t](const std::pair<double, double>& c) { return c.first > t; });
        std::sort(cz.begin(), mid, [](const std::pair<double, double>& x, const std::pair<double, double>& y) {
            return x.first > y.first;
        });
        for (size_t k = L; k < C.size(); ++k) {
            C[k] = cz[k - L].first;
            Z[k] = cz[k - L].second;
        }
        const size_t L2 = L + (size_t)(mid - cz.begin());
        zeta.resize(L2);
        for (size_t k = L; k < L2; ++k) zeta[k] = Z[k];
        L = L2;
        suf1.assign(L + 1, 0.0);
        suf2.assign(L + 1, 0.0);
        sufz1.assign(L + 1, 0.0);
        sufz2.assign(L + 1, 0.0);
        for (size_t k = L; k-- > 0;) {  // ascending weights: small terms first
            suf1[k] = suf1[k + 1] + C[k];
            suf2[k] = suf2[k + 1] + C[k] * C[k];
            sufz1[k] = sufz1[k + 1] + zeta[k];
            sufz2[k] = sufz2[k + 1] + zeta[k] * zeta[k];
        }
        pre1.assign(L + 1, 0.0);
        prez.assign(L + 1, 0.0);
        for (size_t k = 0; k < L; ++k) {
            pre1[k + 1] = pre1[k] + C[k];
            prez[k + 1] = prez[k] + zeta[k];
        }
        rest_sums();
    }
    bool f(double kappa, double& out)
    {
        const double a = std::ldexp(kappa, d) / W;
        if ((a * tau) * wmax > 1.0) return false;
        const double invT = T > 0.0 ? 1.0 / T : 0.0;
        const double G = T > 0.0 ? std::pow(std::sqrt(a) * wmax, invT) : 0.0;
        cover(1.0 / (a * wmax));
        size_t nr = 0;  // R = prefix of the sorted candidates with (a w) wmax > 1
        while (nr < L && (a * C[nr]) * wmax > 1.0) ++nr;
        const double Wsmall = tail.s1 + r1 + suf1[nr], Zs = tail.z1 + rz1 + sufz1[nr],
                     W2s = tail.s2 + r2 + suf2[nr], Z2s = tail.z2 + rz2 + sufz2[nr];
        // sums over R[m, nr) from the prefix sums of the sorted candidates
        const double Wt = Wsmall + pre1[nr], Zt = Zs + prez[nr];
        double Lsum = Wt * Wsmall - W2s;  // pairs (u outside R, any v != u): all non-E_R
        double Psum = Zt * Zs - Z2s;      // in units of G^2
        double nER = 0.0;
        size_t m = nr;
        for (size_t t = 0; t < nr; ++t) {
            while (m > 0 && !((a * C[t]) * C[m - 1] > 1.0)) --m;
            const bool self = t < m;
            nER += (double)(m - (self ? 1 : 0));
            Lsum += C[t] * (Wsmall + (pre1[nr] - pre1[m]) - (self ? 0.0 : C[t]));
            Psum += zeta[t] * (Zs + (prez[nr] - prez[m]) - (self ? 0.0 : zeta[t]));
        }
        const double tot = T == 0.0 ? a * Lsum + nER : (a * Lsum - T * (G * G) * Psum) / (1.0 - T) + nER;
        out = tot / (double)n;
        return std::isfinite(out);
    }
};

static int scale_impl(const double* w, uint64_t n, double avg_deg, int d, double T, double beta, double* kappa_out,
                      cudaStream_t st)
{
    if (!w || !kappa_out || n < 2 || n >= (1ull << 32) || d < 1 || d > 5) return GIRG_EINVAL;
    if (!(T >= 0.0 && T < 1.0) || !(beta > 2.0) || !std::isfinite(beta)) return GIRG_EINVAL;
    if (!(avg_deg > 0.0 && avg_deg < (double)(n - 1))) return GIRG_EINVAL;
    try {
        static int occ = [] {
            int v = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_scale, SC_THREADS, 0);
            return std::max(1, std::min(v, 4));
        }();
        const unsigned nb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)device_sms() * occ,
                                                                                  (n + SC_THREADS - 1) / SC_THREADS));
        uint32_t cap = (uint32_t)std::max<uint64_t>(1u << 16, n / 32);
        double tau = 0.0;
        LazyEstimator E;
        E.n = n;
        E.d = d;
        E.T = T;
        for (int attempt = 0; attempt < 24; ++attempt) {
            // ---- device pass ----
            {
                const auto tp0 = std::chrono::steady_clock::now();
                Scratch S(st);
                const size_t o1 = Scratch::rounded(sizeof(ScaleCtl)), o2 = o1 + Scratch::rounded(nb * sizeof(Acc192)),
                             o3 = o2 + Scratch::rounded(nb * sizeof(TailSums));
                char* blk = S.alloc<char>(o3 + 2 * (size_t)cap * sizeof(double));  // candidates, then their zeta
                ScaleCtl* ctl = (ScaleCtl*)blk;
                Acc192* wpart = (Acc192*)(blk + o1);
                TailSums* tpart = (TailSums*)(blk + o2);
                double* cand = (double*)(blk + o3);
                ScaleCtl init;
                std::memset(&init, 0, sizeof(init));
                init.emin = INT_MAX;
                GCHECK(cudaMemcpyAsync(ctl, &init, sizeof(init), cudaMemcpyHostToDevice, st));
                const double* wp = w;
                uint32_t n32 = (uint32_t)n;
                double avg = avg_deg, Tv = T, bv = beta, tv = tau;
                int dv = d;
                void* args[] = {(void*)&wp, &n32, &dv, &Tv, &avg, &bv, &tv, &wpart, &tpart, &cand, &cap, &ctl};
                GCHECK(cudaLaunchCooperativeKernel((const void*)k_scale, dim3(nb), dim3(SC_THREADS), args, 0, st));
                ScaleCtl out;
                GCHECK(cudaMemcpyAsync(&out, ctl, sizeof(out), cudaMemcpyDeviceToHost, st));
                GCHECK(cudaStreamSynchronize(st));
                if (out.err & ERR_WEIGHT) return GIRG_EINVAL;
                if (out.err & ERR_WRANGE) return GIRG_ERANGE;
                if (out.ncand > cap) {  // candidate buffer too small: grow and repeat the pass
                    cap = out.ncand + (out.ncand >> 3) + 64;
                    tau = out.tau;
                    continue;
                }
                E.W = out.W;
                E.wmax = out.wmax;
                E.tau = out.tau;
                E.tail = out.tail;
                E.C.resize(out.ncand);
                E.Z.resize(out.ncand);
                if (out.ncand) {
                    GCHECK(cudaMemcpyAsync(E.C.data(), cand, out.ncand * sizeof(double), cudaMemcpyDeviceToHost, st));
                    GCHECK(cudaMemcpyAsync(E.Z.data(), cand + cap, out.ncand * sizeof(double), cudaMemcpyDeviceToHost,
                                           st));
                    GCHECK(cudaStreamSynchronize(st));
                }
                const auto tp1 = std::chrono::steady_clock::now();
                E.reset();
                const auto tp1b = std::chrono::steady_clock::now();
                // ---- host search (exponential bracket, bisection in log kappa, R12) ----
                const double k0 = out.kappa0;
                double lo = 0, hi = 0, fv = 0, bad_kappa = 0;
                bool ok = true;
                auto F = [&](double kappa) {
                    if (!ok) return false;
                    if (!E.f(kappa, fv)) {
                        const double a = std::ldexp(kappa, d) / E.W;
                        if ((a * E.tau) * E.wmax > 1.0) bad_kappa = kappa;
                        ok = false;
                    }
                    return ok;
                };
                int it = 0;
                if (F(k0) && fv < avg_deg) {
                    lo = k0;
                    hi = 2.0 * k0;
                    while (F(hi) && fv < avg_deg) {
                        lo = hi;
                        hi *= 2.0;
                        if (++it > 2000) return GIRG_ERANGE;
                    }
                } else if (ok) {
                    hi = k0;
                    lo = 0.5 * k0;
                    while (F(lo) && !(fv < avg_deg)) {
                        hi = lo;
                        lo *= 0.5;
                        if (++it > 2000) return GIRG_ERANGE;
                    }
                }
                // root of f(kappa) = avg_deg in [lo, hi] to a relative width of 1e-13 (R12): false
                // position in log kappa with the Illinois rule, a bisection every third step
                double glo = 0, ghi = 0;
                if (ok && F(lo)) glo = fv - avg_deg;
                if (ok && F(hi)) ghi = fv - avg_deg;
                int side = 0;
                for (it = 0; ok && it < 200 && hi / lo - 1.0 >= 1e-13; ++it) {
                    double mid = std::sqrt(lo * hi);
                    if (it % 3 != 2 && ghi > glo) {
                        const double xl = std::log(lo), xh = std::log(hi);
                        const double xm = xl - glo * (xh - xl) / (ghi - glo);
                        const double cand = std::exp(xm);
                        if (cand > lo && cand < hi) mid = cand;
                    }
                    if (!F(mid)) break;
                    const double g = fv - avg_deg;
                    if (g < 0) {
                        lo = mid;
                        glo = g;
                        if (side == -1) ghi *= 0.5;
                        side = -1;
                    } else {
                        hi = mid;
                        ghi = g;
                        if (side == 1) glo *= 0.5;
                        side = 1;
                    }
                }
                static const bool dbg = getenv("GIRG_SCALE_DEBUG") != nullptr;
                if (dbg) {
                    const auto tp2 = std::chrono::steady_clock::now();
                    fprintf(stderr, "[girg scale] attempt %d ncand %u sorted %zu tau %g ok %d iters %d kappa0 %g device+copy %.3f ms sort %.3f search %.3f ms\n",
                            attempt, out.ncand, E.L, E.tau, (int)ok, it, k0,
                            std::chrono::duration<double, std::milli>(tp1 - tp0).count(),
                            std::chrono::duration<double, std::milli>(tp1b - tp1).count(),
                            std::chrono::duration<double, std::milli>(tp2 - tp1b).count());
                }
                if (ok) {
                    *kappa_out = 0.5 * (lo + hi);
                    return GIRG_OK;
                }
                if (bad_kappa == 0) return GIRG_ERANGE;  // f not finite
                // kappa beyond the range covered by tau: a smaller tau (up to 16x the failing kappa)
                tau = 1.0 / (16.0 * (std::ldexp(bad_kappa, d) / E.W) * E.wmax);
            }
        }
        return GIRG_ERANGE;
    } catch (const CudaFail& fl) {
        return map_cuda(fl.e);
    } catch (const std::bad_alloc&) {
        return GIRG_ENOMEM;
    } catch (...) {
        g_last_cuda = "internal error: unexpected exception";
        return GIRG_ECUDA;
    }
}

#include "hrg.cuh"

}  // namespace girg

// ======================================================================================
// C ABI
// ======================================================================================
using namespace girg;

extern "C" int girg_weights(uint64_t n, double beta, uint64_t seed, double* w_dev, void* stream)
{
    if (n == 0 || n >= (1ull << 32) || !(beta > 2.0) || !std::isfinite(beta) || !w_dev) return GIRG_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_weights<<<grid_for(n, 256), 256, 0, st>>>((uint32_t)n, -1.0 / (beta - 1.0), (uint32_t)seed,
                                                (uint32_t)(seed >> 32), w_dev);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GIRG_OK : map_cuda(e);
}

extern "C" int girg_positions(uint64_t n, int d, uint64_t seed, double* x_dev, void* stream)
{
    if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5 || !x_dev) return GIRG_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    k_positions<<<grid_for(n, 256), 256, 0, st>>>((uint32_t)n, d, (uint32_t)seed, (uint32_t)(seed >> 32), x_dev);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GIRG_OK : map_cuda(e);
}

extern "C" int girg_scale_weights(const double* w_dev, uint64_t n, double avg_deg, int d, double T, double beta,
                                  double* kappa_out, void* stream)
{
    return scale_impl(w_dev, n, avg_deg, d, T, beta, kappa_out, (cudaStream_t)stream);
}

extern "C" int girg_edges(const double* w_dev, const double* x_dev, uint64_t n, int d, double T, double kappa,
                          uint64_t seed, uint32_t* edges_dev, uint64_t cap, uint64_t* m_out, void* stream)
{
    return edges_impl(w_dev, x_dev, n, d, T, kappa, seed, 0, 0, 1, SCHEME_MERGED, edges_dev, cap, m_out, nullptr,
                      (cudaStream_t)stream);
}

extern "C" int girg_edges_shard(const double* w_dev, const double* x_dev, uint64_t n, int d, double T,
                                double kappa, uint64_t seed, int shard_level, uint64_t blk_lo, uint64_t blk_hi,
                                uint32_t* edges_dev, uint64_t cap, uint64_t* m_out, girg_stats* stats_out,
                                void* stream)
{
    return edges_impl(w_dev, x_dev, n, d, T, kappa, seed, shard_level, blk_lo, blk_hi, SCHEME_MERGED, edges_dev,
                      cap, m_out, stats_out, (cudaStream_t)stream);
}

extern "C" int girg_edges_ex(const double* w_dev, const double* x_dev, uint64_t n, int d, double T, double kappa,
                             uint64_t seed, const girg_options* opt, uint32_t* edges_dev, uint64_t cap,
                             uint64_t* m_out, girg_stats* stats_out, void* stream)
{
    girg_options o = {GIRG_SCHEME_MERGED, 0, 0, 1, 0, 0};
    if (opt) o = *opt;
    return edges_impl(w_dev, x_dev, n, d, T, kappa, seed, o.shard_level, o.blk_lo, o.blk_hi, o.scheme, edges_dev, cap,
                      m_out, stats_out, (cudaStream_t)stream, o.nranks, o.rank);
}

extern "C" int girg_edges_host(const double* w_host, const double* x_host, uint64_t n, int d, double T,
                               double kappa, uint64_t seed, uint32_t* edges_host, uint64_t cap, uint64_t* m_out,
                               void* stream)
{
    if (!w_host || !x_host || !m_out || (cap && !edges_host)) return GIRG_EINVAL;
    if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5) return GIRG_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    try {
        Scratch S(st);
        double* w = S.alloc<double>(n);
        double* x = S.alloc<double>((size_t)d * n);
        GCHECK(cudaMemcpyAsync(w, w_host, n * sizeof(double), cudaMemcpyHostToDevice, st));
        GCHECK(cudaMemcpyAsync(x, x_host, (size_t)d * n * sizeof(double), cudaMemcpyHostToDevice, st));
        // page-locked output: the sampling kernels write their staged edge blocks straight into
        // host memory over the bus while they run (no device edge buffer, no trailing D2H copy)
        uint32_t* mapped = nullptr;
        if (cap) {
            cudaPointerAttributes pa;
            if (cudaPointerGetAttributes(&pa, edges_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                pa.devicePointer)
                mapped = (uint32_t*)pa.devicePointer;
            cudaGetLastError();  // pageable memory: not an error, use the copy path
        }
        uint32_t* e = mapped ? mapped : S.alloc<uint32_t>(2 * std::max<uint64_t>(cap, 1));
        int rc = edges_impl(w, x, n, d, T, kappa, seed, 0, 0, 1, SCHEME_MERGED, e, cap, m_out, nullptr, st);
        if (rc != GIRG_OK) return rc;
        if (*m_out && !mapped)
            GCHECK(cudaMemcpyAsync(edges_host, e, *m_out * 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        GCHECK(cudaStreamSynchronize(st));
        return GIRG_OK;
    } catch (const CudaFail& f) {
        return map_cuda(f.e);
    } catch (const std::bad_alloc&) {
        return GIRG_ENOMEM;
    } catch (...) {
        g_last_cuda = "internal error: unexpected exception";
        return GIRG_ECUDA;
    }
}

// Fused batch: B graphs of n points as ONE problem.  One launch
// computes every graph's weight statistics (blockIdx.y = graph); after the single read-back the
// host makes the B plans and offsets each graph's cell space into one concatenated key space, so
// that ONE counting sort (keys, scan, scatter, in-cell order, records) builds every graph's
// Lemma-1 index at once (graph g's sorted points are entries g n .. g n + n - 1, its vertex ids
// local); the sampling kernels run all graphs in one launch each (blockIdx.y = graph, per-graph
// arguments in device memory).  Two host synchronisations for the whole batch.  Graph g's edge
// set is exactly its girg_edges result: the plan, index and keyed draws are the same.
template <int D>
static int batch_fused(int B, const double* const* w_dev, const double* const* x_dev, uint64_t n, double T,
                       const double* kappa, const uint64_t* seed, uint32_t* const* edges_dev, const uint64_t* cap,
                       uint64_t* m_out, int* status, cudaStream_t st)
{
    constexpr int d = D;
    const uint32_t n32 = (uint32_t)n;
    const uint64_t N = (uint64_t)B * n;
    static const bool dbg = getenv("GIRG_BATCH_DEBUG") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    auto lap = [&](const char* what) {
        if (!dbg) return;
        const auto t = now();
        fprintf(stderr, "[girg batch] %-28s %8.1f us\n", what, std::chrono::duration<double, std::micro>(t - t0).count());
        t0 = t;
    };
    PhaseEvents PE;
    Scratch S(st);
    // ---- weight statistics of every graph (one launch, one read-back) ----
    const unsigned tiles = grid_for(n, WS_TILE);
    const size_t o_err = (size_t)B * HIST_BINS * 4, o_part = Scratch::rounded(o_err + (size_t)B * 16),
                 wst_bytes = o_part + (size_t)B * tiles * sizeof(WPartial);
    char* wst = S.alloc<char>(wst_bytes);
    const double** d_ptr = (const double**)S.alloc<char>(2 * (size_t)B * sizeof(void*));
    {
        std::vector<const double*> hp(2 * (size_t)B);
        for (int g = 0; g < B; ++g) {
            hp[g] = w_dev[g];
            hp[B + g] = x_dev[g];
        }
        GCHECK(cudaMemcpyAsync(d_ptr, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice, st));
        GCHECK(cudaStreamSynchronize(st));  // pageable source
    }
    const double* const* d_w = d_ptr;
    const double* const* d_x = d_ptr + B;
    GCHECK(cudaMemsetAsync(wst, 0, o_part, st));
    k_wstats<<<dim3(tiles, B), WS_THREADS, 0, st>>>(nullptr, n32, (uint32_t*)wst, (WPartial*)(wst + o_part),
                                                    (int*)(wst + o_err), d_w, 4);
    GCHECK(cudaGetLastError());
    char* hw = PE.staging(std::max<size_t>(wst_bytes, 1 << 20));
    std::vector<char> hw_pageable;
    if (!hw) {
        hw_pageable.resize(wst_bytes);
        hw = hw_pageable.data();
    }
    GCHECK(cudaMemcpyAsync(hw, wst, wst_bytes, cudaMemcpyDeviceToHost, st));
    GCHECK(cudaStreamSynchronize(st));
    lap("weight statistics + sync");
    // ---- plans (host threads for large batches), concatenated cell space ----
    // the plans live in a per-thread cache: a fresh 2 MB of HostPlans per call costs more in page
    // faults than making the plans
    static thread_local std::vector<HostPlan> hp_cache;
    if (hp_cache.size() < (size_t)B) hp_cache.resize(B);
    HostPlan* hp = hp_cache.data();
    std::vector<int> prc(B, GIRG_OK);
    auto plan_one = [&](int g) {
        const int herr = ((const int*)(hw + o_err))[4 * g];
        if (herr & ERR_WEIGHT) { prc[g] = GIRG_EINVAL; return; }
        if (herr & ERR_WRANGE) { prc[g] = GIRG_ERANGE; return; }
        std::vector<uint32_t> hist((const uint32_t*)hw + (size_t)g * HIST_BINS,
                                   (const uint32_t*)hw + (size_t)(g + 1) * HIST_BINS);
        std::vector<WPartial> parts((const WPartial*)(hw + o_part) + (size_t)g * tiles,
                                    (const WPartial*)(hw + o_part) + (size_t)(g + 1) * tiles);
        prc[g] = make_plan(hist, parts, n, d, T, kappa[g], hp[g]);
        hp[g].p.sl = 0;
        hp[g].p.blo = 0;
        hp[g].p.bhi = 1;
    };
    {
        static const int nth_env = getenv("GIRG_BATCH_PLAN_THREADS") ? atoi(getenv("GIRG_BATCH_PLAN_THREADS")) : 0;
        const int nth = nth_env > 0 ? nth_env : (B >= 16 ? std::min(8, B / 8) : 1);
        std::atomic<int> next{0};
        auto work = [&]() {
            for (int g; (g = next.fetch_add(1)) < B;) plan_one(g);
        };
        std::vector<std::thread> pool;
        for (int k = 1; k < nth; ++k) pool.emplace_back(work);
        work();
        for (std::thread& t : pool) t.join();
    }
    lap("plans");
    for (int g = 0; g < B; ++g)
        if (prc[g] != GIRG_OK) return 1;  // the caller runs the per-graph path, which reports it
    std::vector<uint64_t> gbase(B + 1, 0);
    for (int g = 0; g < B; ++g) gbase[g + 1] = gbase[g] + hp[g].K;
    const uint64_t K = gbase[B];
    if (K + 1 >= 0xFFFFFFFFull) return 1;
    size_t ntab = 0, ntask = 0;
    std::vector<size_t> tab_off(B), task_off(B);
    for (int g = 0; g < B; ++g) {
        Plan& p = hp[g].p;
        for (int i = 0; i <= p.L; ++i) p.base[i] += (uint32_t)gbase[g];
        tab_off[g] = ntab;
        task_off[g] = ntask;
        ntab += hp[g].tab.size();
        ntask += hp[g].tasks.size();
    }
    // ---- scratch ----
    const int recw = Geo<D>::RECW;
    const unsigned items_cap = std::max<unsigned>(4096u, n32 / 2);
    const size_t up_plan = Scratch::rounded((size_t)B * sizeof(Plan)), up_tab = Scratch::rounded(ntab * sizeof(TabEntry)),
                 up_task = Scratch::rounded(ntask * sizeof(uint16_t)), up_args = Scratch::rounded((size_t)B * sizeof(SampleArgs)),
                 up_bytes = up_plan + up_tab + up_task + up_args;
    S.reserve(Scratch::rounded(up_bytes) + Scratch::rounded((size_t)B * 256) + Scratch::rounded(16) +
              6 * Scratch::rounded(N * 4) + 2 * Scratch::rounded((K + 1) * 4) +
              Scratch::rounded((grid_for(K + 1, SCAN_TILE) + 1) * 4) + Scratch::rounded((size_t)recw * N * 8) +
              Scratch::rounded((size_t)B * items_cap * sizeof(BigItem)) + Scratch::rounded((2 * (N / (ORDER_SMALL + 1) + 1)) * 4));
    char* d_up = S.alloc<char>(up_bytes);
    Plan* d_plan = (Plan*)d_up;
    TabEntry* d_tab = (TabEntry*)(d_up + up_plan);
    uint16_t* d_tasks = (uint16_t*)(d_up + up_plan + up_tab);
    SampleArgs* d_args = (SampleArgs*)(d_up + up_plan + up_tab + up_task);
    char* misc = S.alloc<char>((size_t)B * 256);
    uint32_t* nbig = S.alloc<uint32_t>(4);
    uint32_t* key = S.alloc<uint32_t>(N);
    uint2* tk = S.alloc<uint2>(N);
    uint32_t* inv = S.alloc<uint32_t>(N);
    uint32_t* cnt = S.alloc<uint32_t>(K + 1);
    uint32_t* P = S.alloc<uint32_t>(K + 1);
    uint32_t* bsum = S.alloc<uint32_t>(grid_for(K + 1, SCAN_TILE) + 1);
    uint32_t* sid = S.alloc<uint32_t>(N);
    uint32_t* skey = S.alloc<uint32_t>(N);
    double* rec = S.alloc<double>((size_t)recw * N);
    BigItem* items = S.alloc<BigItem>((size_t)B * items_cap);
    uint32_t* big = S.alloc<uint32_t>(2 * (N / (ORDER_SMALL + 1) + 1));
    // ---- per-graph sampler arguments, written straight into page-locked staging, one upload ----
    char* stage = PE.staging(up_bytes + (size_t)B * 256);
    std::vector<char> up_pageable;
    char* up = stage;
    if (!up) {
        up_pageable.resize(up_bytes + (size_t)B * 256);
        up = up_pageable.data();
    }
    char* hmisc = up + up_bytes;
    for (int g = 0; g < B; ++g) {
        std::memcpy(up + (size_t)g * sizeof(Plan), &hp[g].p, plan_upload_bytes(hp[g].p));
        std::memcpy(up + up_plan + tab_off[g] * sizeof(TabEntry), hp[g].tab.data(), hp[g].tab.size() * sizeof(TabEntry));
        std::memcpy(up + up_plan + up_tab + task_off[g] * sizeof(uint16_t), hp[g].tasks.data(),
                    hp[g].tasks.size() * sizeof(uint16_t));
        SampleArgs a;
        std::memset(&a, 0, sizeof(a));
        char* mg = misc + (size_t)g * 256;
        a.pl = d_plan + g;
        a.tab = d_tab + tab_off[g];
        a.tasks = d_tasks + task_off[g];
        a.skey = skey + (size_t)g * n;
        a.rec = rec + (size_t)g * n * recw;
        a.sid = sid + (size_t)g * n;
        a.P = P;
        a.n = n32;
        a.tile_pts = 32u;  // the batch fills the GPU with graphs
        a.ntiles = (n32 + 31) / 32;
        a.k0 = (uint32_t)seed[g];
        a.k1 = (uint32_t)(seed[g] >> 32);
        a.edges = (uint2*)edges_dev[g];
        a.cap = cap[g];
        a.m = (unsigned long long*)(mg + 16);
        a.tile_ctr = (unsigned int*)(mg + 24);
        a.nitems = (unsigned int*)(mg + 28);
        a.item_ctr = (unsigned int*)(mg + 128);
        a.stats = nullptr;
        a.err = (int*)mg;
        a.items = items + (size_t)g * items_cap;
        a.items_cap = items_cap;
        a.nP = K + 1;
        a.ntab = (unsigned)hp[g].tab.size();
        a.ntasks = (unsigned)hp[g].tasks.size();
        a.big_work = big_work(d, n);
        a.item_work = item_work(d, n);
        a.T = hp[g].p.T;
        a.s = hp[g].p.s;
        a.invT = hp[g].p.invT;
        a.sl = 0;
        a.blo = 0;
        a.bhi = 1;
        a.nranks = 0;
        a.rank = 0;
        a.sharded = 0;
        a.p0 = (uint32_t)((uint64_t)g * n);
        std::memcpy(up + up_plan + up_tab + up_task + (size_t)g * sizeof(SampleArgs), &a, sizeof(a));
    }
    GCHECK(cudaMemcpyAsync(d_up, up, up_bytes, cudaMemcpyHostToDevice, st));
    if (!stage) GCHECK(cudaStreamSynchronize(st));  // pageable source must outlive the copy
    lap("scratch + args + upload");
    GCHECK(cudaMemsetAsync(misc, 0, (size_t)B * 256, st));
    GCHECK(cudaMemsetAsync(nbig, 0, 16, st));
    // ---- one index build over the concatenated problem ----
    GCHECK(cudaMemsetAsync(cnt, 0, (K + 1) * sizeof(uint32_t), st));
    k_keys<D><<<dim3(grid_for(n, 256), B), 256, 0, st>>>(nullptr, nullptr, n32, d_plan, key, cnt, (int*)misc, d_w,
                                                         d_x, 64);
    const unsigned nbs = grid_for(K + 1, SCAN_TILE);
    k_scan_reduce<<<nbs, SCAN_THREADS, 0, st>>>(cnt, K + 1, bsum);
    k_scan_top<<<1, 1024, 0, st>>>(bsum, nbs);
    k_scan_final<<<nbs, SCAN_THREADS, 0, st>>>(cnt, K + 1, bsum, P);
    k_scatter<<<grid_for(N, 256), 256, 0, st>>>(key, (uint32_t)N, cnt, tk);
    k_order<<<grid_for(N, 256), 256, 0, st>>>(tk, (uint32_t)N, P, sid, skey, inv, big, nbig, n32);
    {
        int bits = 1;
        while (bits < 32 && (1ull << bits) < N) ++bits;
        const unsigned gb = (unsigned)std::min<uint64_t>((uint64_t)device_sms() * 4u, N / (ORDER_SMALL + 1) + 1);
        k_order_big<<<gb, OB_THREADS, 0, st>>>(tk, (bits + 7) / 8, big, nbig, sid, skey, inv, key, n32);
    }
    k_place<D><<<dim3(grid_for(n, 256), B), 256, 0, st>>>(inv, n32, nullptr, nullptr, rec, d_w, d_x);
    GCHECK(cudaGetLastError());
    // ---- sampling, every graph in one launch per kernel ----
    {
        constexpr int WPB = Geo<D>::WPB, TPB = 32 * WPB;
        const size_t smem = sizeof(WarpSmem<D>) * WPB;
        smem_optin(k_sample_b<D, SCHEME_MERGED, false>, smem);
        smem_optin(k_big_b<D, SCHEME_MERGED, false>, smem);
        static const int occ = [] {
            int v = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_sample_b<D, SCHEME_MERGED, false>, TPB,
                                                          sizeof(WarpSmem<D>) * WPB);
            return std::max(v, 1);
        }();
        const unsigned wtiles = ((n32 + 31) / 32 + WPB - 1) / WPB;
        const unsigned per = std::max(1u, std::min<unsigned>(wtiles, (unsigned)((2ull * device_sms() * occ + B - 1) / B)));
        k_sample_b<D, SCHEME_MERGED, false><<<dim3(per, B), TPB, smem, st>>>(d_args);
        k_big_b<D, SCHEME_MERGED, false><<<dim3(per, B), TPB, smem, st>>>(d_args);
        GCHECK(cudaGetLastError());
    }
    lap("launches");
    GCHECK(cudaMemcpyAsync(hmisc, misc, (size_t)B * 256, cudaMemcpyDeviceToHost, st));
    GCHECK(cudaStreamSynchronize(st));
    lap("index + sampling + sync");
    for (int g = 0; g < B; ++g) {
        const char* mg = hmisc + (size_t)g * 256;
        int derr;
        unsigned long long m;
        std::memcpy(&derr, mg, sizeof(int));
        std::memcpy(&m, mg + 16, sizeof(m));
        if (derr & ERR_POS) {
            status[g] = GIRG_EINVAL;
            m_out[g] = 0;
            continue;
        }
        if (derr & ERR_ITEMS) {  // item queue overflow (rare for small graphs): this graph alone
            uint64_t mm = 0;
            status[g] = edges_impl(w_dev[g], x_dev[g], n, d, T, kappa[g], seed[g], 0, 0, 1, SCHEME_MERGED,
                                   edges_dev[g], cap[g], &mm, nullptr, st);
            m_out[g] = mm;
            continue;
        }
        m_out[g] = m;
        status[g] = m > cap[g] ? GIRG_ECAPACITY : GIRG_OK;
    }
    return 0;
}

// Batched small graphs: each graph is one unchanged girg_edges pipeline
// (EdgeCall: two host waits, for the weight statistics the plan needs and for the edge count).
// A pool of native host threads, each with its own stream, runs them concurrently, so one
// graph's host planning and waits overlap other graphs' kernels on the 148 SMs.  (Measured: a
// single thread driving all graphs in waves over several streams is slower -- the per-graph
// host work, not the waits, is what has to run in parallel.)
extern "C" int girg_edges_batch(int B, const double* const* w_dev, const double* const* x_dev, uint64_t n, int d,
                                double T, const double* kappa, const uint64_t* seed, uint32_t* const* edges_dev,
                                const uint64_t* cap, uint64_t* m_out, int* status_out, int nstreams, void* stream)
{
    if (B < 1 || !w_dev || !x_dev || !kappa || !seed || !edges_dev || !cap || !m_out) return GIRG_EINVAL;
    if (n == 0 || n >= (1ull << 32) || d < 1 || d > 5 || !(T >= 0.0 && T < 1.0)) return GIRG_EINVAL;
    for (int g = 0; g < B; ++g)  // per-graph arguments checked before any work is queued
        if (EdgeCall::validate(w_dev[g], x_dev[g], n, d, T, kappa[g], 0, 0, 1, SCHEME_MERGED, edges_dev[g], cap[g],
                               m_out + g) != GIRG_OK)
            return GIRG_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (B >= 2 && nstreams >= 0 && n <= (1ull << 22) && (uint64_t)B * n < (1ull << 31)) {  // fused batch
        std::vector<int> status(B, GIRG_OK);
        int used = 1;
        try {
            switch (d) {
                case 1: used = batch_fused<1>(B, w_dev, x_dev, n, T, kappa, seed, edges_dev, cap, m_out, status.data(), st); break;
                case 2: used = batch_fused<2>(B, w_dev, x_dev, n, T, kappa, seed, edges_dev, cap, m_out, status.data(), st); break;
                case 3: used = batch_fused<3>(B, w_dev, x_dev, n, T, kappa, seed, edges_dev, cap, m_out, status.data(), st); break;
                case 4: used = batch_fused<4>(B, w_dev, x_dev, n, T, kappa, seed, edges_dev, cap, m_out, status.data(), st); break;
                default: used = batch_fused<5>(B, w_dev, x_dev, n, T, kappa, seed, edges_dev, cap, m_out, status.data(), st); break;
            }
        } catch (const CudaFail& f) {
            return map_cuda(f.e);
        } catch (const std::bad_alloc&) {
            return GIRG_ENOMEM;
        } catch (...) {
            g_last_cuda = "internal error: unexpected exception";
            return GIRG_ECUDA;
        }
        if (used == 0) {
            int rc = GIRG_OK;
            for (int g = 0; g < B; ++g) {
                if (status_out) status_out[g] = status[g];
                if (rc == GIRG_OK && status[g] != GIRG_OK) rc = status[g];
            }
            return rc;
        }
    }
    const int nt = std::max(1, std::min(B, nstreams > 0 ? nstreams : (nstreams < 0 ? -nstreams : 8)));
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return map_cuda(cudaGetLastError());
    std::vector<cudaStream_t> ss(nt, nullptr);
    std::vector<cudaEvent_t> ev(nt + 1, nullptr);
    std::vector<int> status(B, GIRG_OK);
    auto cleanup = [&]() {
        for (cudaStream_t s2 : ss)
            if (s2) cudaStreamDestroy(s2);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
    };
    try {
        for (int k = 0; k <= nt; ++k) GCHECK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        GCHECK(cudaEventRecord(ev[nt], st));  // the batch starts after the caller's queued work
        for (int k = 0; k < nt; ++k) {
            GCHECK(cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking));
            GCHECK(cudaStreamWaitEvent(ss[k], ev[nt], 0));
        }
    } catch (const CudaFail& f) {
        cleanup();
        return map_cuda(f.e);
    }
    std::atomic<int> next{0};
    auto worker = [&](int k) {
        if (cudaSetDevice(dev) != cudaSuccess) {
            for (int g; (g = next.fetch_add(1)) < B;) status[g] = GIRG_ECUDA;
            return;
        }
        for (int g; (g = next.fetch_add(1)) < B;) {
            uint64_t m = 0;
            status[g] = edges_impl(w_dev[g], x_dev[g], n, d, T, kappa[g], seed[g], 0, 0, 1, SCHEME_MERGED,
                                   edges_dev[g], cap[g], &m, nullptr, ss[k]);
            m_out[g] = m;
        }
        cudaEventRecord(ev[k], ss[k]);
    };
    {
        std::vector<std::thread> pool;
        for (int k = 1; k < nt; ++k) pool.emplace_back(worker, k);
        worker(0);
        for (std::thread& t : pool) t.join();
    }
    int rc = GIRG_OK;
    for (int k = 0; k < nt; ++k)
        if (cudaStreamWaitEvent(st, ev[k], 0) != cudaSuccess && rc == GIRG_OK) rc = GIRG_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == GIRG_OK) rc = GIRG_ECUDA;
    cleanup();
    for (int g = 0; g < B; ++g) {
        if (status_out) status_out[g] = status[g];
        if (rc == GIRG_OK && status[g] != GIRG_OK) rc = status[g];
    }
    return rc;
}

extern "C" int girg_hrg_points(uint64_t n, double alpha, double C, uint64_t seed, double* r_dev, double* x_dev,
                               double* w_dev, void* stream)
{
    return girg::hrg_points_impl(n, alpha, C, seed, r_dev, x_dev, w_dev, (cudaStream_t)stream);
}

extern "C" int girg_hrg_edges(const double* r_dev, const double* x_dev, const double* w_dev, uint64_t n, double C,
                              double T, uint64_t seed, uint32_t* edges_dev, uint64_t cap, uint64_t* m_out,
                              girg_hrg_stats* stats_out, void* stream)
{
    return girg::hrg_edges_impl(r_dev, x_dev, w_dev, n, C, T, seed, edges_dev, cap, m_out, stats_out,
                                (cudaStream_t)stream);
}

extern "C" const char* girg_strerror(int status)
{
    switch (status) {
        case GIRG_OK: return "ok";
        case GIRG_EINVAL: return "invalid argument";
        case GIRG_ECAPACITY: return "edge buffer too small (m_out holds the required count)";
        case GIRG_ERANGE: return "input outside the supported range of the index";
        case GIRG_ENOMEM: return "out of device memory";
        case GIRG_ECUDA: return "CUDA runtime error";
        default: return "unknown status";
    }
}

extern "C" int girg_last_timings(girg_timings* out)
{
    if (!out) return GIRG_EINVAL;
    *out = girg::g_timings;
    return GIRG_OK;
}

extern "C" const char* girg_last_cuda_error(void) { return girg::g_last_cuda.c_str(); }

extern "C" int girg_version(void) { return 201; }
extern "C" int girg_debug_index(const double* w_dev, const double* x_dev, uint64_t n, int d, double T, double kappa,
                                uint32_t* sid_dev, uint32_t* P_dev, uint64_t P_cap, uint64_t* K_out, int* L_out,
                                uint32_t* base_out, uint32_t* lstart_out, uint8_t* I_out, void* stream)
{
    using namespace girg;
    uint64_t m = 0;
    cudaStream_t st = (cudaStream_t)stream;
    int v = EdgeCall::validate(w_dev, x_dev, n, d, T, kappa, 0, 0, 1, SCHEME_MERGED, nullptr, 0, &m);
    if (v != GIRG_OK) return v;
    if (!K_out || !L_out || !base_out || !lstart_out || !I_out) return GIRG_EINVAL;
    try {
        EdgeCall E(w_dev, x_dev, n, d, T, kappa, 0, 0, 0, 1, SCHEME_MERGED, nullptr, 0, &m, nullptr, st);
        E.dbg_sid = sid_dev;
        E.dbg_P = P_dev;
        E.dbg_Pcap = P_cap;
        E.stage_a();
        GCHECK(cudaStreamSynchronize(st));
        E.stage_b();
        if (E.rc != GIRG_OK) return E.rc;
        GCHECK(cudaStreamSynchronize(st));
        const int rc = E.stage_c();  // the sampler ran with capacity 0: ECAPACITY is the expected outcome
        if (rc != GIRG_OK && rc != GIRG_ECAPACITY) return rc;
        const Plan& p = E.hp.p;
        *K_out = E.hp.K;
        *L_out = p.L;
        for (int i = 0; i <= p.L; ++i) {
            base_out[i] = p.base[i];
            lstart_out[i] = p.lstart[i];
        }
        for (int i = 0; i < p.L; ++i) I_out[i] = p.I[i];
        return GIRG_OK;
    } catch (const CudaFail& f) {
        return map_cuda(f.e);
    } catch (const std::bad_alloc&) {
        return GIRG_ENOMEM;
    } catch (...) {
        g_last_cuda = "internal error: unexpected exception";
        return GIRG_ECUDA;
    }
}

extern "C" int girg_debug_set_ref_x(int x)
{
    girg::g_ref_x.store(x);
    return GIRG_OK;
}
