// surface_kernel.cuh -- rows a4 + a5 in the saturation-aware streaming form (the default when
// the caller does not request D2).  One warp per (window, strip of 32 columns); lane = column.
//
// Eq. (1) saturates: in fp32, S = 1 - exp(-sqrt(D2)/alpha) is exactly 1.0f for
// D2 >= K_sat (K_sat = 353 for alpha = 6/ln 255).  Let c = ceil(sqrt(K_sat)).  Any E_df pixel
// at squared distance < K_sat lies within c-1 rows and c-1 columns, so
//   D2(x,y) = min over rows y' with h(x,y') < c of (y-y')^2 + h(x,y')^2   whenever D2 < K_sat,
// where h(x,y') = horizontal distance from (x,y') to the nearest E_df pixel of row y'
// (separable exact EDT, with the first pass capped -- SURVEY.md §8(c) "capping
// lemma").  Every candidate is a true squared distance, so when D2 >= K_sat the computed value
// is >= K_sat as well and S = 1.0f exactly: the fp32 surface equals the exact-EDT surface.
//
// Per warp the rows are streamed top to bottom: row yi's site (h < c) is pushed onto a
// Felzenszwalb-Huttenlocher lower envelope of parabolas (y - yi)^2 + h^2, then pixel
// yo = yi - (c-1) -- all of whose candidate rows are pushed -- is evaluated by walking the
// envelope and written (lanes = 32 consecutive columns: one coalesced 128-byte store per row).
// Sites c or more rows above yo can no longer matter, so the live envelope spans < 2c rows and
// lives in a 64-entry ring per lane in shared memory; all quantities stay below 2^24, so the
// intersection tests are exact in 32-bit integers.
#pragma once
#include <cstdint>

namespace ieds {

constexpr int kRing = 64;           // ring entries per lane (requires c <= 31)
constexpr int kSurfWarps = 8;       // warps (strips) per CTA

struct SurfParams {
    const uint32_t* __restrict__ Edf;   // [nb][H][NWP2] row-major E_df words, NWP2 = NW + 2,
                                        // word w of row y at index 1 + w, guard words are 0
    float* __restrict__ S;              // [nb][H][W]
    const float* __restrict__ lut;      // [K_lut]
    int W, H, NW;
    int K_lut, K_sat;
    int c;                              // ceil(sqrt(K_sat)) <= 31
    float c_exp;
};

// lane j of strip w: horizontal distance to the nearest set bit among words w-1, w, w+1
// (>= 32 when there is none within 31 columns; c <= 31 makes that sufficient).
//   left : the 32 columns x-31 .. x, column x in the MSB      -> count leading zeros
//   right: the 32 columns x .. x+31, column x in the LSB      -> count trailing zeros
__device__ __forceinline__ int hdist3(uint32_t tl, uint32_t t, uint32_t tr, int j) {
    const uint32_t left = __funnelshift_rc(tl, t, j + 1);
    const uint32_t right = __funnelshift_r(t, tr, j);
    return min(__clz(left), __clz(__brev(right)));
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}

struct Envelope {
    // live envelope = ring entries [flo, n) (a valid FH stack whose first entry is never
    // popped); the top two entries are cached in registers; pe = walk position
    uint32_t ring;   // shared address of this lane's ring column: entry i at ring + (i&63)*64
    int n, flo, pe;
    int sb, fb, sa, fa;   // sites and f = h^2 of the top (b) and second (a) entries
    int sflo;             // site of entry flo

    __device__ __forceinline__ uint32_t at(int i) const { return lds_u16(ring + ((i & (kRing - 1)) << 6)); }

    // push the parabola (y - yi)^2 + h^2 (Felzenszwalb-Huttenlocher).  The top b is popped
    // while z(b, yi) <= z(a, b), i.e. (k_yi - k_b)(s_b - s_a) <= (k_b - k_a)(yi - s_b) with keys
    // k = f + s^2; live sites lie in (yi - 2c, yi] so every product is < 2^24 (exact in int32).
    __device__ __forceinline__ void push(int yi, int h) {
        const int f = h * h;
        while (n - flo >= 2) {
            const int lhs = (f - fb + (yi - sb) * (yi + sb)) * (sb - sa);
            const int rhs = (fb - fa + (sb - sa) * (sb + sa)) * (yi - sb);
            if (lhs > rhs) break;
            --n;
            sb = sa;
            fb = fa;
            if (n - flo >= 2) {
                const uint32_t e = at(n - 2);
                sa = (int)(e >> 5);
                const int ha = (int)(e & 31u);
                fa = ha * ha;
            }
        }
        sts_u16(ring + ((n & (kRing - 1)) << 6), ((uint32_t)yi << 5) | (uint32_t)h);
        sa = sb;
        fa = fb;
        sb = yi;
        fb = f;
        if (n == flo) sflo = yi;
        ++n;
        pe = min(pe, n - 2);   // the walk restarts at or below the modified depth
    }

    // D2 at row yo over the live entries (0x7FFFFFFF if none)
    __device__ __forceinline__ int eval(int yo, int c) {
        // entries whose site is c or more rows above yo are dead for yo and every later row
        while (flo < n && sflo <= yo - c) {
            ++flo;
            sflo = (int)(at(flo) >> 5);
        }
        if (n <= flo) return 0x7FFFFFFF;
        pe = max(pe, flo);
        uint32_t e = at(pe);
        int dy = yo - (int)(e >> 5), hh = (int)(e & 31u);
        int d2 = dy * dy + hh * hh;
        while (pe + 1 < n) {   // the minimum over the envelope is unimodal along the stack
            const uint32_t e2 = at(pe + 1);
            const int dy2 = yo - (int)(e2 >> 5), h2 = (int)(e2 & 31u);
            const int v2 = dy2 * dy2 + h2 * h2;
            if (v2 >= d2) break;
            d2 = v2;
            ++pe;
        }
        return d2;
    }
};

__global__ void __launch_bounds__(kSurfWarps * 32) surface_kernel(SurfParams p) {
    __shared__ __align__(16) uint16_t ring_all[kSurfWarps][kRing][32];   // entry = site << 5 | h
    __shared__ __align__(16) float lut_s[1024];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < p.K_lut; i += blockDim.x) lut_s[i] = p.lut[i];
    __syncthreads();

    const int w = blockIdx.x * kSurfWarps + warp;
    if (w >= p.NW) return;
    const int b = blockIdx.y;
    const int W = p.W, H = p.H, c = p.c, K_lut = p.K_lut, K_sat = p.K_sat;
    const float c_exp = p.c_exp;
    const int NWP2 = p.NW + 2;
    const int lag = c - 1;
    const int x = 32 * w + lane;
    const bool xvalid = x < W;
    const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(lut_s);
    const uint32_t* rp = p.Edf + (size_t)b * H * NWP2 + 1 + w;
    float* sp = p.S + (size_t)b * H * W + (xvalid ? x : 0);

    Envelope env;
    env.ring = (uint32_t)__cvta_generic_to_shared(&ring_all[warp][0][lane]);
    env.n = env.flo = env.pe = 0;
    env.sb = env.fb = env.sa = env.fa = env.sflo = 0;

    auto store = [&](int d2) {
        float v;
        if ((unsigned)d2 < (unsigned)K_lut) v = lds_f32(lut_base + 4u * (uint32_t)d2);
        else if ((unsigned)d2 >= (unsigned)K_sat) v = 1.0f;
        else v = 1.0f - exp2f(c_exp * sqrtf((float)d2));
        if (xvalid) *sp = v;
        sp += W;
    };
    auto site = [&](int yi) {
        const uint32_t tl = rp[-1], t = rp[0], tr = rp[1];
        rp += NWP2;
        const int h = hdist3(tl, t, tr, lane);
        if (h < c) env.push(yi, h);
    };

    const int y_in_end = H;             // rows pushed: 0 .. H-1
    const int pre = min(lag, H);
    int yi = 0;
    for (; yi < pre; ++yi) site(yi);                      // prologue: push only
    for (; yi < y_in_end; ++yi) {                          // steady state: push row yi, emit yi - lag
        site(yi);
        store(env.eval(yi - lag, c));
    }
    for (int yo = max(0, H - lag); yo < H; ++yo) store(env.eval(yo, c));   // epilogue
}

}  // namespace ieds
