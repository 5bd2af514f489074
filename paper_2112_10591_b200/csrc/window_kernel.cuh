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
// divergence, no shared-memory traffic besides the 4-byte table lookup.
#pragma once
#include <cstdint>

namespace ieds {

constexpr int kWinWarps = 8;   // warps (strips) per CTA

struct WinParams {
    const uint32_t* __restrict__ Edf;   // [nb][H][NW+2], word w of row y at 1 + w, zero guards
    float* __restrict__ S;              // [nb][H][W]
    const float* __restrict__ lut;      // [K_sat + 1], lut[K_sat] = 1.0f
    int W, H, NW;
    int K_sat;                          // <= 1024
};

// horizontal distance of lane j of a strip to the nearest set bit of words (tl, t, tr)
// (>= 32 when none within 31 columns)
__device__ __forceinline__ int hdist_words(uint32_t tl, uint32_t t, uint32_t tr, int j) {
    const uint32_t left = __funnelshift_rc(tl, t, j + 1);   // columns x-31..x, x in the MSB
    const uint32_t right = __funnelshift_r(t, tr, j);       // columns x..x+31, x in the LSB
    return min(__clz(left), __clz(__brev(right)));
}

template <int C>
__device__ __forceinline__ constexpr uint32_t slot_sq(int slot, int u_phase) {
    // distance from row u (u == u_phase mod 2C) to the window pixel held in `slot`
    // (window = [u-C+1, u+C]): d = ((slot - u_phase + C - 1) mod 2C) - (C - 1)
    const int d = ((slot - u_phase + C - 1) % (2 * C) + 2 * C) % (2 * C) - (C - 1);
    return (uint32_t)(d * d);
}

template <int C>
__global__ void __launch_bounds__(kWinWarps * 32, (C <= 22 ? 6 : 3)) window_kernel(WinParams p) {
    static_assert(C >= 2 && C <= 64, "window size");
    constexpr int NS = 2 * C;   // slots
    __shared__ float lut_s[1025];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i <= p.K_sat; i += blockDim.x) lut_s[i] = p.lut[i];
    __syncthreads();

    const int w = blockIdx.x * kWinWarps + warp;
    if (w >= p.NW) return;
    const int b = blockIdx.y;
    const int W = p.W, H = p.H;
    const uint32_t K_sat = (uint32_t)p.K_sat;
    const int NWP2 = p.NW + 2;
    const int x = 32 * w + lane;
    const bool xvalid = x < W;
    const uint32_t* rp = p.Edf + (size_t)b * H * NWP2 + w;   // words w-1, w, w+1 at rp[0..2]
    float* op = p.S + (size_t)b * H * W + (xvalid ? x : 0);  // next pixel to emit (rows in order)
    const size_t wstride = (size_t)W;

    uint32_t R[C];
#pragma unroll
    for (int k = 0; k < C; ++k) R[k] = 0xFFFFFFFFu;

    // The strip's three words of 32 consecutive rows are fetched lane-parallel (lane i holds
    // row base+i) one batch ahead and broadcast with shuffles when the row is processed.
    uint32_t cl = 0, cm = 0, cr = 0, nl = 0, nm = 0, nr = 0;
    auto fetch = [&](int row0, uint32_t& a, uint32_t& m, uint32_t& z) {
        const int r = row0 + lane;
        if (r < H) {
            const uint32_t* q = rp + (size_t)r * NWP2;
            a = __ldg(q);
            m = __ldg(q + 1);
            z = __ldg(q + 2);
        } else {
            a = m = z = 0u;
        }
    };
    fetch(0, cl, cm, cr);
    fetch(32, nl, nm, nr);
    auto h_of = [&](int u) -> uint32_t {   // h of row u clamped to C (rows >= H: no site)
        const int src = u & 31;
        const uint32_t tl = __shfl_sync(0xFFFFFFFFu, cl, src);
        const uint32_t t = __shfl_sync(0xFFFFFFFFu, cm, src);
        const uint32_t tr = __shfl_sync(0xFFFFFFFFu, cr, src);
        return (uint32_t)min(hdist_words(tl, t, tr, lane), C);
    };

    const int total = H + C - 1;   // rows u = 0 .. total-1: push site u (< H), emit u-C+1 (>= 0)
    for (int base = 0; base < total; base += NS) {
#pragma unroll
        for (int ph = 0; ph < NS; ph += 2) {
            const int u0 = base + ph;
            if (u0 >= total) break;
            if (u0 > 0 && (u0 & 31) == 0) {   // rows u0.. start a new batch of 32
                cl = nl;
                cm = nm;
                cr = nr;
                fetch(u0 + 32, nl, nm, nr);
            }
            const uint32_t ha = h_of(u0), hb = h_of(u0 + 1);   // rows >= H read zero words
            // skip the update when no lane of either row has a site within C-1 columns
            if (__any_sync(0xFFFFFFFFu, (ha < (uint32_t)C) | (hb < (uint32_t)C))) {
                const uint32_t h2a = ha * ha * 0x10001u, h2b = hb * hb * 0x10001u;
#pragma unroll
                for (int k = 0; k < C; ++k) {
                    // rows u0 (phase ph) and u0+1 (phase ph+1); slots 2k (low half), 2k+1 (high)
                    const uint32_t sqa = slot_sq<C>(2 * k, ph) | (slot_sq<C>(2 * k + 1, ph) << 16);
                    const uint32_t sqb = slot_sq<C>(2 * k, ph + 1) | (slot_sq<C>(2 * k + 1, ph + 1) << 16);
                    R[k] = __vminu2(R[k], __vminu2(sqa + h2a, sqb + h2b));
                }
            }
            // pixels u0-C+1 and u0-C+2 are final: a row C or more away cannot bring a value
            // below C^2 >= K_sat.  Their slots are reset for pixels u0+C+1, u0+C+2.
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int yo = u0 + e - (C - 1);
                const int so = ((ph + e - (C - 1)) % NS + NS) % NS;   // compile-time slot of yo
                if (yo >= 0 && yo < H) {
                    const uint32_t v = (so & 1) ? (R[so >> 1] >> 16) : (R[so >> 1] & 0xFFFFu);
                    const float f = lut_s[min(v, K_sat)];
                    // write-once output: streaming store, predicated off for lanes beyond W
                    asm volatile(
                        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}"
                        ::"l"(op), "f"(f), "r"((uint32_t)xvalid) : "memory");
                    op += wstride;
                }
                R[so >> 1] |= (so & 1) ? 0xFFFF0000u : 0x0000FFFFu;
            }
        }
    }
}

}  // namespace ieds
