// fwl_kernel.cuh -- row f3: flow-compensated event image and the Flow Warping Loss
// (DESIGN readings R19, R20).
//
//   I_comp(q)   = sum over events e of s_e * bilinear weight of q at
//                 (x_e, y_e) + F(x_e, y_e) * (t_ref - t_e) / dt      (dropped if outside the frame)
//   I_uncomp(q) = sum over events at q of s_e                          (s_e = +1 if p_e > 0, else -1)
//   FWL         = var(I_comp) / var(I_uncomp), population variances over all W*H pixels.
//
// The warp is evaluated in fp64 with explicit round-to-nearest operations in the oracle's
// order (tau = (t_ref - t)/dt; xw = x + Fx*tau; x0 = floor(xw); fx = xw - x0; weights
// (1-fx)(1-fy), fx(1-fy), (1-fx)fy, fx*fy), so the drop/floor decisions and every weight are
// the oracle's bit for bit; only the order of the per-pixel sums differs (fp64 atomics).
// Both images live in a zero-initialised scratch of a few windows (L2-resident: 12 B/px).  The
// sums of I and I^2 come from the splat's atomics (each add's old value, see fwl_add), so the
// images are never read back; a memset re-zeroes the scratch for the next windows.
#pragma once
#include <cstdint>

namespace ieds {

constexpr int kFwlThreads = 256;

struct FwlParams {
    const uint32_t* __restrict__ xy;       // [n_events] x | y << 16
    const int64_t* __restrict__ t;         // [n_events] microseconds
    const int8_t* __restrict__ p;          // [n_events] polarity (> 0: +1, else -1)
    const int64_t* __restrict__ offsets;   // [nb + 1] absolute indices
    int64_t n_events;
    const float2* __restrict__ flow;       // [nb][H][W] (dx, dy) pixels per dt
    const int64_t* __restrict__ t_ref;     // [nb] reference times (microseconds)
    int64_t dt;                            // microseconds, > 0
    int W, H;
    int64_t stride;                        // pixels per window image in the scratch (>= W*H, % 4 == 0)
    double* __restrict__ Ic;               // [nb][stride] scratch, zero on entry
    int* __restrict__ Iu;                  // [nb][stride] scratch, zero on entry
    int* __restrict__ err;
};

// Per-window partial sums of I_comp, I_comp^2 (fp64) and I_uncomp, I_uncomp^2 (exact int64),
// one per splat block: part[b][blk] = {sum c, sum c^2, sum u, sum u^2}.
struct FwlPart {
    double c, c2;
    long long u, u2;
};

// The warp of one event (reading R19), in the oracle's fp64 order with explicit
// round-to-nearest operations: false if the warped position is dropped (outside [0, W-1] x
// [0, H-1], or NaN); else the top-left corner (ix, iy) and the bilinear weights.
struct FwlWarp {
    int ix, iy;
    double w00, w10, w01, w11;
};

__device__ __forceinline__ bool fwl_warp(const FwlParams& p, const float2* F, int64_t tref, int64_t i, int x, int y,
                                         FwlWarp& o) {
    const float2 f = __ldg(F + (size_t)y * p.W + x);
    const double dt = (double)p.dt;
    const double tau = __ddiv_rn((double)(tref - __ldg(p.t + i)), dt);
    const double xw = __dadd_rn((double)x, __dmul_rn((double)f.x, tau));
    const double yw = __dadd_rn((double)y, __dmul_rn((double)f.y, tau));
    if (!(xw >= 0.0 && xw <= (double)(p.W - 1) && yw >= 0.0 && yw <= (double)(p.H - 1))) return false;
    const double x0 = floor(xw), y0 = floor(yw);
    const double fx = __dsub_rn(xw, x0), fy = __dsub_rn(yw, y0);
    const double ax = __dsub_rn(1.0, fx), ay = __dsub_rn(1.0, fy);
    o.ix = (int)x0;
    o.iy = (int)y0;
    o.w00 = __dmul_rn(ax, ay);
    o.w10 = __dmul_rn(fx, ay);
    o.w01 = __dmul_rn(ax, fy);
    o.w11 = __dmul_rn(fx, fy);
    return true;
}

// Adds v to *a and returns its contribution to the sum of squares: new^2 - old^2, with old the
// atomic's return and new = old + v exactly as the atomic rounded it.  Over all adds to one
// pixel these terms sum to the pixel's final value squared (telescoping), so the image is
// never read back.  Also adds v to the plain sum.
__device__ __forceinline__ double fwl_add(double* a, double v, double& sc) {
    const double old = atomicAdd(a, v);
    const double nw = __dadd_rn(old, v);
    sc += v;
    return __dmul_rn(__dsub_rn(nw, old), __dadd_rn(nw, old));
}

// Splat: each event adds s_e = +-1 to I_uncomp at (x, y) and s_e * weight to the four corners
// of its warped position in I_comp; the block's threads accumulate sum I and sum I^2 of both
// images from the atomics' old values, and write one partial per block.  (Bound by the L2
// atomic rate: taking 2 or 4 events per thread with all their atomics in flight measured no gain.)
__global__ void __launch_bounds__(kFwlThreads) fwl_splat_kernel(FwlParams p, FwlPart* __restrict__ part) {
    const int b = blockIdx.y;
    int64_t o0 = p.offsets[b], o1 = p.offsets[b + 1];
    if (o0 < 0 || o1 < o0 || o1 > p.n_events) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.err, 2);   // kErrOrder
        o0 = o1 = 0;
    }
    const int W = p.W, H = p.H;
    double* Ic = p.Ic + (size_t)b * p.stride;
    int* Iu = p.Iu + (size_t)b * p.stride;
    const float2* F = p.flow + (size_t)b * W * H;
    const int64_t tref = p.t_ref[b];
    double sc = 0.0, sc2 = 0.0;
    long long su = 0, su2 = 0;
    int bad = 0;
    for (int64_t i = o0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < o1; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldg(p.xy + i);
        const int x = (int)(v & 0xFFFFu), y = (int)(v >> 16);
        if (x >= W || y >= H) {
            bad = 1;
            continue;
        }
        const int s = __ldg(p.p + i) > 0 ? 1 : -1;
        const int old = atomicAdd(Iu + (size_t)y * W + x, s);
        su += s;
        su2 += 2ll * s * old + 1;   // (old + s)^2 - old^2, exact
        FwlWarp wp;
        if (!fwl_warp(p, F, tref, i, x, y, wp)) continue;
        double* c = Ic + (size_t)wp.iy * W + wp.ix;
        const bool neg = s < 0;
        sc2 += fwl_add(c, neg ? -wp.w00 : wp.w00, sc);
        if (wp.ix + 1 < W) sc2 += fwl_add(c + 1, neg ? -wp.w10 : wp.w10, sc);
        if (wp.iy + 1 < H) {
            sc2 += fwl_add(c + W, neg ? -wp.w01 : wp.w01, sc);
            if (wp.ix + 1 < W) sc2 += fwl_add(c + W + 1, neg ? -wp.w11 : wp.w11, sc);
        }
    }
    if (bad) atomicOr(p.err, 1);   // kErrRange: dropped, latched
    for (int o = 16; o > 0; o >>= 1) {
        sc += __shfl_xor_sync(0xFFFFFFFFu, sc, o);
        sc2 += __shfl_xor_sync(0xFFFFFFFFu, sc2, o);
        su += __shfl_xor_sync(0xFFFFFFFFu, su, o);
        su2 += __shfl_xor_sync(0xFFFFFFFFu, su2, o);
    }
    __shared__ FwlPart s_p[kFwlThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_p[warp] = FwlPart{sc, sc2, su, su2};
    __syncthreads();
    if (threadIdx.x == 0) {
        FwlPart t = s_p[0];
        for (int k = 1; k < kFwlThreads / 32; ++k) {
            t.c += s_p[k].c;
            t.c2 += s_p[k].c2;
            t.u += s_p[k].u;
            t.u2 += s_p[k].u2;
        }
        part[(size_t)b * gridDim.x + blockIdx.x] = t;
    }
}

// One block per window: sums the partials (fixed order), var = E[I^2] - E[I]^2,
// FWL = var_c / var_u (NaN if var_u = 0)
__global__ void __launch_bounds__(kFwlThreads) fwl_finalize_kernel(const FwlPart* __restrict__ part, int nblk,
                                                                    int64_t npx, double* __restrict__ fwl,
                                                                    double* __restrict__ var_c,
                                                                    double* __restrict__ var_u) {
    const int b = blockIdx.x;
    double sc = 0.0, sc2 = 0.0;
    long long su = 0, su2 = 0;
    for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
        const FwlPart t = part[(size_t)b * nblk + k];
        sc += t.c;
        sc2 += t.c2;
        su += t.u;
        su2 += t.u2;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sc += __shfl_xor_sync(0xFFFFFFFFu, sc, o);
        sc2 += __shfl_xor_sync(0xFFFFFFFFu, sc2, o);
        su += __shfl_xor_sync(0xFFFFFFFFu, su, o);
        su2 += __shfl_xor_sync(0xFFFFFFFFu, su2, o);
    }
    __shared__ FwlPart s_p[kFwlThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_p[warp] = FwlPart{sc, sc2, su, su2};
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int k = 1; k < (int)(blockDim.x / 32); ++k) {
        sc += s_p[k].c;
        sc2 += s_p[k].c2;
        su += s_p[k].u;
        su2 += s_p[k].u2;
    }
    const double N = (double)npx;
    const double mc = sc / N;
    const double vc = fmax(sc2 / N - mc * mc, 0.0);
    // N * sum u^2 - (sum u)^2 is an exact integer (|sum u| <= n_events)
    const double vu = (double)(npx * su2 - su * su) / (N * N);
    fwl[b] = vu > 0.0 ? vc / vu : __longlong_as_double(0x7FF8000000000000LL);
    if (var_c) var_c[b] = vc;
    if (var_u) var_u[b] = vu;
}

}  // namespace ieds
