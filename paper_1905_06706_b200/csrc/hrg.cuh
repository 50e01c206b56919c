// hrg.cuh -- hyperbolic random graphs (Sec. 3.2) on the GIRG machinery
// (Sec. 3.3), included by girg.cu inside namespace girg.  DESIGN.md R25: the HRG is
// sampled as an exactly thinned DOMINATING GIRG.  With w'_v = e^((R - r_v)/2) / sqrt(1 - e^(-2 r_v))
// (e^(R/2) at r_v = 0), positions x_v = theta_v / (2 pi), d = 1 and s' = e^(-R/2)/sqrt(2) (1 + 2^-30),
// every HRG connection probability is at most the GIRG one (cosh d >= 2 sinh r_u sinh r_v
// sin^2(pi dx) >= 2 e^(2R) dx^2 / (w'_u w'_v)^2, e^(-d) <= 1/cosh d), so the girg_edges sampler
// (merged scheme, s fixed to s') draws a supergraph and each of its edges is kept with
// probability p_HRG / p_GIRG' -- every pair ends up an edge with probability p_HRG, independently.
#pragma once

struct HrgDevStats {
    unsigned long long m, nt, viol;
};

// Philox counter (v, 0, 0, 7): U = (o0, o1) -> r = acosh(1 + U (cosh(alpha R)
// - 1)) / alpha (inverse of the radial CDF), x = (o2, o3) (= theta / (2 pi)); w' as above
__global__ void k_hrg_points(uint32_t n, double alpha, double R, double K, uint32_t k0, uint32_t k1,
                             double* __restrict__ r, double* __restrict__ x, double* __restrict__ w)
{
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint4 o = philox4x32_10(make_uint4(v, 0u, 0u, 7u), k0, k1);
    const double U = u53(o.x, o.y);
    const double rv = __ddiv_rn(acosh(__dadd_rn(1.0, __dmul_rn(U, K))), alpha);
    r[v] = rv;
    x[v] = u53(o.z, o.w);
    w[v] = rv <= 0.0 ? exp(__dmul_rn(0.5, R))
                     : __ddiv_rn(exp(__dmul_rn(0.5, __dsub_rn(R, rv))), sqrt(-expm1(__dmul_rn(-2.0, rv))));
}

// thinning of the dominating GIRG's edges: keep (u, v) with probability p_HRG / p_GIRG'
// (T > 0: uniform of Philox counter (u, v, 0, 6), words (o0, o1); T = 0: iff cosh d < cosh R)
constexpr int HT_THREADS = 256;
__global__ void __launch_bounds__(HT_THREADS) k_hrg_thin(const uint2* __restrict__ sup, unsigned long long msup,
                                                        const double* __restrict__ r, const double* __restrict__ x,
                                                        const double* __restrict__ w, double R, double coshR,
                                                        double T, double invT, double s, uint32_t k0, uint32_t k1,
                                                        uint2* __restrict__ out, unsigned long long cap,
                                                        HrgDevStats* st)
{
    const unsigned lane = threadIdx.x & 31u;
    unsigned long long nt = 0, viol = 0;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long k0e = (unsigned long long)blockIdx.x * blockDim.x; k0e < msup; k0e += stride) {
        const unsigned long long k = k0e + threadIdx.x;
        bool keep = false;
        uint2 e = make_uint2(0u, 0u);
        if (k < msup) {
            e = sup[k];
            const uint32_t u = e.x, v = e.y;
            const double ru = r[u], rv = r[v];
            const double a = fabs(__dsub_rn(x[u], x[v]));
            const double t = fmin(a, __dsub_rn(1.0, a));
            const double cd = __dsub_rn(__dmul_rn(cosh(ru), cosh(rv)),
                                        __dmul_rn(__dmul_rn(sinh(ru), sinh(rv)), cos(__dmul_rn(6.283185307179586, t))));
            if (T == 0.0) {
                nt += fabs(__dsub_rn(cd, coshR)) < 1e-12 * coshR;
                keep = cd < coshR;
            } else {
                const double dd = acosh(cd < 1.0 ? 1.0 : cd);
                const double ph = __ddiv_rn(1.0, __dadd_rn(exp(__ddiv_rn(__dsub_rn(dd, R), __dmul_rn(2.0, T))), 1.0));
                const double pg = prob_uv(w[u], w[v], s, t, invT);  // d = 1: D = dist
                const double ratio = __ddiv_rn(ph, pg);
                viol += ratio > 1.0;
                const uint4 o = philox4x32_10(make_uint4(min(u, v), max(u, v), 0u, 6u), k0, k1);
                const double rr = u53(o.x, o.y);
                nt += fabs(__dsub_rn(rr, ratio)) < 1e-12;
                keep = rr < ratio;
            }
        }
        const unsigned bm = __ballot_sync(0xffffffffu, keep);
        unsigned long long base = 0;
        if (lane == 0 && bm) base = atomicAdd(&st->m, (unsigned long long)__popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const unsigned long long slot = base + __popc(bm & ((1u << lane) - 1u));
            if (slot < cap) out[slot] = e;
        }
    }
    for (int o = 16; o; o >>= 1) {
        nt += __shfl_xor_sync(0xffffffffu, nt, o);
        viol += __shfl_xor_sync(0xffffffffu, viol, o);
    }
    if (lane == 0 && (nt || viol)) {
        atomicAdd(&st->nt, nt);
        atomicAdd(&st->viol, viol);
    }
}

static int hrg_points_impl(uint64_t n, double alpha, double C, uint64_t seed, double* r, double* x, double* w,
                           cudaStream_t st)
{
    if (n < 2 || n >= (1ull << 32) || !(alpha > 0.5) || !std::isfinite(alpha) || !std::isfinite(C) || !r || !x || !w)
        return GIRG_EINVAL;
    const double R = 2.0 * std::log((double)n) + C;
    if (!(R > 0.0)) return GIRG_EINVAL;
    const double K = std::cosh(alpha * R) - 1.0;
    if (!std::isfinite(K)) return GIRG_ERANGE;
    k_hrg_points<<<grid_for(n, 256), 256, 0, st>>>((uint32_t)n, alpha, R, K, (uint32_t)seed, (uint32_t)(seed >> 32), r,
                                                   x, w);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GIRG_OK : map_cuda(e);
}

static int hrg_edges_impl(const double* r, const double* x, const double* w, uint64_t n, double C, double T,
                          uint64_t seed, uint32_t* edges, uint64_t cap, uint64_t* m_out, girg_hrg_stats* so,
                          cudaStream_t st)
{
    if (!r || !x || !w || !m_out || (cap && !edges) || n < 2 || n >= (1ull << 32)) return GIRG_EINVAL;
    if (!(T >= 0.0 && T < 1.0) || !std::isfinite(C)) return GIRG_EINVAL;
    const double R = 2.0 * std::log((double)n) + C;
    if (!(R > 0.0)) return GIRG_EINVAL;
    const double sd = std::exp(-0.5 * R) / std::sqrt(2.0) * (1.0 + 0x1p-30);  // s' (R25), as the oracle
    const double coshR = std::cosh(R);
    try {
        Scratch S(st);
        uint64_t scap = std::max<uint64_t>(4 * cap, 4 * n) + 1024, msup = 0;
        uint2* sup = nullptr;
        for (int attempt = 0;; ++attempt) {
            sup = S.alloc<uint2>(scap);
            const int rc = edges_impl(w, x, n, 1, T, 1.0, seed, 0, 0, 1, SCHEME_MERGED, (uint32_t*)sup, scap, &msup,
                                      nullptr, st, 0, 0, sd);
            if (rc == GIRG_ECAPACITY && attempt == 0) {
                scap = msup + 1;
                continue;
            }
            if (rc != GIRG_OK) return rc;
            break;
        }
        HrgDevStats* d_st = S.alloc<HrgDevStats>(1);
        GCHECK(cudaMemsetAsync(d_st, 0, sizeof(HrgDevStats), st));
        if (msup) {
            const unsigned nb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(grid_for(msup, HT_THREADS),
                                                                                    (uint64_t)device_sms() * 8));
            k_hrg_thin<<<nb, HT_THREADS, 0, st>>>(sup, msup, r, x, w, R, coshR, T, T > 0.0 ? 1.0 / T : 0.0, sd,
                                                  (uint32_t)seed, (uint32_t)(seed >> 32), (uint2*)edges, cap, d_st);
            GCHECK(cudaGetLastError());
        }
        HrgDevStats h;
        GCHECK(cudaMemcpyAsync(&h, d_st, sizeof(h), cudaMemcpyDeviceToHost, st));
        GCHECK(cudaStreamSynchronize(st));
        *m_out = h.m;
        if (so) {
            so->super_edges = msup;
            so->neartie = h.nt;
            so->violations = h.viol;
        }
        return h.m > cap ? GIRG_ECAPACITY : GIRG_OK;
    } catch (const CudaFail& f) {
        return map_cuda(f.e);
    } catch (const std::bad_alloc&) {
        return GIRG_ENOMEM;
    } catch (...) {
        g_last_cuda = "internal error: unexpected exception";
        return GIRG_ECUDA;
    }
}
