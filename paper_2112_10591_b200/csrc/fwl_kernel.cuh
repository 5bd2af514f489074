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
// Both images live in a zero-initialised scratch of a few windows (L2-resident: 12 B/px), the
// reduce pass re-zeroes it as it reads it.
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

__global__ void __launch_bounds__(kFwlThreads) fwl_splat_kernel(FwlParams p) {
    const int b = blockIdx.y;
    int64_t o0 = p.offsets[b], o1 = p.offsets[b + 1];
    if (o0 < 0 || o1 < o0 || o1 > p.n_events) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.err, 2);   // kErrOrder
        return;
    }
    const int W = p.W, H = p.H;
    const size_t npx = (size_t)W * H;
    double* Ic = p.Ic + (size_t)b * p.stride;
    int* Iu = p.Iu + (size_t)b * p.stride;
    const float2* F = p.flow + (size_t)b * npx;
    const int64_t tref = p.t_ref[b];
    const double dt = (double)p.dt, xmax = (double)(W - 1), ymax = (double)(H - 1);
    int bad = 0;
    for (int64_t i = o0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < o1; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldg(p.xy + i);
        const int x = (int)(v & 0xFFFFu), y = (int)(v >> 16);
        if (x >= W || y >= H) {
            bad = 1;
            continue;
        }
        const bool pos = __ldg(p.p + i) > 0;
        const size_t q = (size_t)y * W + x;
        atomicAdd(Iu + q, pos ? 1 : -1);
        const float2 f = __ldg(F + q);
        const double tau = __ddiv_rn((double)(tref - __ldg(p.t + i)), dt);
        const double xw = __dadd_rn((double)x, __dmul_rn((double)f.x, tau));
        const double yw = __dadd_rn((double)y, __dmul_rn((double)f.y, tau));
        if (!(xw >= 0.0 && xw <= xmax && yw >= 0.0 && yw <= ymax)) continue;   // dropped (also NaN)
        const double x0 = floor(xw), y0 = floor(yw);
        const double fx = __dsub_rn(xw, x0), fy = __dsub_rn(yw, y0);
        const double ax = __dsub_rn(1.0, fx), ay = __dsub_rn(1.0, fy);
        const int ix = (int)x0, iy = (int)y0;
        double* c = Ic + (size_t)iy * W + ix;
        const double w00 = __dmul_rn(ax, ay), w10 = __dmul_rn(fx, ay), w01 = __dmul_rn(ax, fy),
                     w11 = __dmul_rn(fx, fy);
        atomicAdd(c, pos ? w00 : -w00);
        if (ix + 1 < W) atomicAdd(c + 1, pos ? w10 : -w10);
        if (iy + 1 < H) {
            atomicAdd(c + W, pos ? w01 : -w01);
            if (ix + 1 < W) atomicAdd(c + W + 1, pos ? w11 : -w11);
        }
    }
    if (bad) atomicOr(p.err, 1);   // kErrRange: dropped, latched
}

// Per-window partial sums of I_comp, I_comp^2 (fp64) and I_uncomp, I_uncomp^2 (exact int64),
// one partial per block: part[b][blk] = {sum c, sum c^2, sum u, sum u^2}; re-zeroes both
// images.  Each window's scratch image has a stride that is a multiple of 4 pixels (the pad
// stays zero), so a thread takes 4 pixels with two 16-byte fp64 loads and one 16-byte int32
// load, all in flight at once.  With comp_out (tests), a plain per-pixel loop also copies
// I_comp out.
struct FwlPart {
    double c, c2;
    long long u, u2;
};

__global__ void __launch_bounds__(kFwlThreads) fwl_reduce_kernel(double* __restrict__ Ic, int* __restrict__ Iu,
                                                                  int64_t npx, int64_t stride,
                                                                  FwlPart* __restrict__ part, int nblk,
                                                                  double* __restrict__ comp_out) {
    const int b = blockIdx.y;
    double* c = Ic + (size_t)b * stride;
    int* u = Iu + (size_t)b * stride;
    double sc = 0.0, sc2 = 0.0;
    long long su = 0, su2 = 0;
    if (comp_out) {
        double* co = comp_out + (size_t)b * npx;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
            const double cv = c[i];
            const long long uv = u[i];
            sc += cv;
            sc2 = fma(cv, cv, sc2);
            su += uv;
            su2 += uv * uv;
            co[i] = cv;
            c[i] = 0.0;
            u[i] = 0;
        }
    } else {
        double2* c2 = reinterpret_cast<double2*>(c);
        int4* u4 = reinterpret_cast<int4*>(u);
        const int64_t n4 = stride >> 2;
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
            const double2 a = __ldcg(c2 + 2 * j), d = __ldcg(c2 + 2 * j + 1);
            const int4 w = __ldcg(u4 + j);
            sc += (a.x + a.y) + (d.x + d.y);
            sc2 = fma(a.x, a.x, fma(a.y, a.y, fma(d.x, d.x, fma(d.y, d.y, sc2))));
            su += (long long)w.x + w.y + w.z + w.w;
            su2 += (long long)w.x * w.x + (long long)w.y * w.y + (long long)w.z * w.z + (long long)w.w * w.w;
            c2[2 * j] = make_double2(0.0, 0.0);
            c2[2 * j + 1] = make_double2(0.0, 0.0);
            u4[j] = make_int4(0, 0, 0, 0);
        }
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
    if (threadIdx.x == 0) {
        FwlPart t = s_p[0];
        for (int k = 1; k < kFwlThreads / 32; ++k) {
            t.c += s_p[k].c;
            t.c2 += s_p[k].c2;
            t.u += s_p[k].u;
            t.u2 += s_p[k].u2;
        }
        part[(size_t)b * nblk + blockIdx.x] = t;
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
