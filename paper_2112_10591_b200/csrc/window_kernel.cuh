// window_kernel.cuh -- rows a4 + a5, saturation-aware and branch-free (default surface path).
// One warp per (window, strip of 32 columns); lane = column; rows streamed top to bottom.
//
// Why it is exact (Eq. (1), separable exact EDT P:239):
// the fp32 surface 1 - exp(-sqrt(D2)/alpha) is exactly 1.0f once D2 >= K_sat.  With
// C >= ceil(sqrt(K_sat)), any E_df pixel at squared distance < K_sat lies fewer than C rows
// and C columns away, so for every pixel
//     D2(x,y) = min over |y-u| < C of (y-u)^2 + min(h(x,u), C)^2     whenever D2 < K_sat,
// h(x,u) = horizontal distance from (x,u) to the nearest E_df pixel of row u.  Every
// candidate is a true squared distance or >= C^2 >= K_sat, so a computed value >= K_sat can
// only occur when D2 >= K_sat: the fp32 surface is the exact-EDT surface, bit for bit.
//
// Each lane keeps the 2C pixels y in [u-C+1, u+C] of its column as 16-bit partial minima,
// two per register (slot y mod 2C).  Row u's site updates all of them with one packed add and
// one packed 3-way min (VIMNMX3.U16x2, two rows per instruction); pixel u-C+1 is final after
// row u and is emitted with one coalesced 128-byte store per warp.  The loop is unrolled over
// the 2C slot phases so every slot/distance is a compile-time constant: no stack, no
// divergence, no shared-memory traffic besides the 4-byte table lookup.  (Each update is one
// fused packed add+min instruction, VIADDMNMX.U16x2, per register and row.)
#pragma once
#include <cstdint>

namespace ieds {

constexpr int kWinWarps = 8;                  // warps (strips) per CTA
constexpr int kWinRowWords = kWinWarps + 2;   // E_df words of one row a CTA needs (strips +- 1)

struct WinParams {
    const uint32_t* __restrict__ Edf;   // [nb][H][NW+2], word w of row y at 1 + w, zero guards
    void* __restrict__ S;               // [nb][H][W] float32 or uint8 (OutT)
    const float* __restrict__ lut;      // [K_sat + 1], lut[K_sat] = 1.0f
    int W, H, NW;
    int K_sat;                          // <= 1024
};

// horizontal distance of lane j of a strip to the nearest set bit of words (tl, t, tr)
// (>= 32 when none within 31 columns)
__device__ __forceinline__ int hdist_words(uint32_t tl, uint32_t t, uint32_t tr, int j) {
    const uint32_t left = __funnelshift_rc(tl, t, j + 1);   // columns x-31..x, x in the MSB
    const uint32_t right = __funnelshift_r(t, tr, j);       // columns x..x+31, x in the LSB
    // trailing zeros of `right`; an empty word reads as 31, which is >= C for every C <= 31
    return min(__clz(left), __ffs(right | 0x80000000u) - 1);
}

// squared distance from row u (first of a pair) to pixel y0 + j of the window, y0 = u - C + 1
template <int C>
__device__ __forceinline__ constexpr uint32_t dsq(int j, int row_off) {
    const int d = j - (C - 1) - row_off;
    return (uint32_t)(d * d);
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// write-once output: streaming (evict-first) stores
__device__ __forceinline__ void st_cs(float* ptr, float v) { __stcs(ptr, v); }
__device__ __forceinline__ void st_cs(uint8_t* ptr, float v) {
    asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(ptr), "r"((uint32_t)v) : "memory");
}

template <int C, typename OutT>
struct WinState {
    int H, NWP2, lane;
    uint32_t words_sh;                 // shared address of this strip's words (w-1, w, w+1) of row 0
    OutT* op;                          // next pixel to emit (rows are emitted in order)
    size_t W;                          // row stride in elements
    uint32_t lut_sh, K_sat, xvalid;

    // h of row u for this lane: 3 broadcast shared loads (words w-1, w, w+1 of the row)
    __device__ __forceinline__ uint32_t h_of(int u) const {
        const uint32_t a = words_sh + (uint32_t)min(u, H) * (4u * kWinRowWords);
        uint32_t tl, t, tr;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tl) : "r"(a));
        asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(t) : "r"(a));
        asm volatile("ld.shared.u32 %0, [%1+8];" : "=r"(tr) : "r"(a));
        return (uint32_t)hdist_words(tl, t, tr, lane);   // <= 31; >= C contributes >= C^2
    }
    __device__ __forceinline__ void emit(uint32_t v) {
        const float f = lds_f32(lut_sh + 4u * min(v, K_sat));
        if (xvalid) st_cs(op, f);
        op += W;
    }

    // Rotating window: before a pair step of phase S, logical register j (pixels y0+2j,
    // y0+2j+1 with y0 = u-C+1) lives in P[(j + S) % C].  The step applies the sites of rows
    // u, u+1 and shifts the window by one register, in place: logical j of the new window is
    // old logical j+1 min the two parabolas, and the freed register P[S % C] becomes the new
    // last register.  Then pixels y0, y0+1 are final -- a site C or more rows away cannot
    // bring a value below C^2 >= K_sat -- and are emitted.  Unrolled over S = 0..C-1 (one
    // rotation) every register index is static and a skipped row pair costs one reset.
    template <int S>
    __device__ __forceinline__ void step(int u, uint32_t (&P)[C]) {
        const uint32_t ha = h_of(u), hb = h_of(u + 1);   // rows >= H are zero words: no site
        if (__any_sync(0xFFFFFFFFu, (ha < (uint32_t)C) | (hb < (uint32_t)C))) {
            const uint32_t h2a = ha * ha * 0x10001u, h2b = hb * hb * 0x10001u;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const uint32_t sqa = dsq<C>(2 * j, 0) | (dsq<C>(2 * j + 1, 0) << 16);
                const uint32_t sqb = dsq<C>(2 * j, 1) | (dsq<C>(2 * j + 1, 1) << 16);
                const int m = (j + S + 1) % C;
                const uint32_t prev = (j + 1 < C) ? P[m] : 0xFFFFFFFFu;
                // two fused packed add+min (VIADDMNMX.U16x2 with an immediate): no carries
                // cross the halves because every sum stays below 2 * 31^2 < 2^16
                P[m] = __vminu2(__vminu2(prev, __vadd2(h2a, sqa)), __vadd2(h2b, sqb));
            }
        } else {
            P[S % C] = 0xFFFFFFFFu;   // the new last register starts empty
        }
        const int y0 = u - (C - 1);
        const uint32_t v = P[(S + 1) % C];
        if (y0 >= 0 && y0 < H) emit(v & 0xFFFFu);
        if (y0 + 1 >= 0 && y0 + 1 < H) emit(v >> 16);
    }

    template <int S>
    __device__ __forceinline__ void block(int u0, int total, uint32_t (&P)[C]) {
        if constexpr (S < C) {
            if (u0 + 2 * S < total) {
                step<S>(u0 + 2 * S, P);
                block<S + 1>(u0, total, P);
            }
        }
    }
};

template <int C, typename OutT>
__global__ void __launch_bounds__(kWinWarps * 32, (C <= 22 ? 5 : 3)) window_kernel(WinParams p) {
    static_assert(C >= 2 && C <= 31, "window size (hdist_words reports empty words as 31)");
    extern __shared__ __align__(16) uint32_t wsm[];   // [H + 2][kWinRowWords] E_df words, then the table
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y, H = p.H, w0 = blockIdx.x * kWinWarps;
    const int NWP2 = p.NW + 2;
    // stage words w0-1 .. w0+8 of every row (guard words / columns beyond the frame read 0)
    // plus two zero rows past the end for the row pair straddling H
    {
        const uint32_t* src = p.Edf + (size_t)b * H * NWP2 + w0;
        const int n = (H + 2) * kWinRowWords;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int y = i / kWinRowWords, c = i - y * kWinRowWords;
            wsm[i] = (y < H && w0 + c < NWP2) ? __ldg(src + (size_t)y * NWP2 + c) : 0u;
        }
    }
    float* lut_s = reinterpret_cast<float*>(wsm + (H + 2) * kWinRowWords);
    for (int i = threadIdx.x; i <= p.K_sat; i += blockDim.x) lut_s[i] = p.lut[i];
    __syncthreads();

    const int w = w0 + warp;
    if (w >= p.NW) return;
    const int x = 32 * w + lane;
    WinState<C, OutT> st;
    st.H = H;
    st.NWP2 = NWP2;
    st.lane = lane;
    st.W = (size_t)p.W;
    st.xvalid = x < p.W ? 1u : 0u;
    st.op = reinterpret_cast<OutT*>(p.S) + (size_t)b * H * p.W + (x < p.W ? x : 0);
    st.K_sat = (uint32_t)p.K_sat;
    uint32_t lut_sh = (uint32_t)__cvta_generic_to_shared(lut_s);
    asm volatile("" : "+r"(lut_sh));   // keep the shared address in a register
    st.lut_sh = lut_sh;
    st.words_sh = (uint32_t)__cvta_generic_to_shared(wsm + warp);

    // Window of 2C pixels of this lane's column as 16-bit partial minima, two per register.
    uint32_t P[C];
#pragma unroll
    for (int k = 0; k < C; ++k) P[k] = 0xFFFFFFFFu;
    const int total = H + C - 1;   // row pairs u = 0, 2, ... < total
    for (int u = 0; u < total; u += 2 * C) st.template block<0>(u, total, P);
}

}  // namespace ieds
