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
// Each lane keeps the 2C pixels y in [u-C+1, u+C] of its column as 16-bit partial minima of
// 4*D2, two per register (slot y mod 2C).  Row u's site updates all of them with one fused
// packed add+min (VIADDMNMX.U16x2 with an immediate) per register and row; pixel u-C+1 is
// final after row u and is emitted with one coalesced 128-byte store per warp.  The loop is
// unrolled over the C register phases of one rotation so every slot/distance is a
// compile-time constant: no stack, no divergence.  (win_split(C) of the C registers take their two
// adds on the FMA pipe instead, then one 3-way packed min: the kernel is co-limited by the ALU
// pipe and by issue.)  The rotations in the middle of the frame
// (all emitted rows inside the frame) run without any range check; only the first and the
// last rotation carry them.  Instruction budget per row pair (2 pixels), see DESIGN.md §6:
//   activity      uniform bit test + BRA (one ballot per rotation gives the C pair bits)
//   active only:  h of 2 rows: 3 LDS.64 + 2 x (2 SHF + BREV + LOP3 + FLO.SH) + 4 IMAD (h^2),
//                 2 (C - k) VIADDMNMX.U16x2 + k x (2 IMAD + VIMNMX3.U16x2), k = win_split(C)
//   emit          2 IMAD extracts + 2 LDS (table) + 2 STG + 2 32-bit pointer adds
#pragma once
#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

namespace ieds {

constexpr int kWinWarps = 8;                      // warps (strips) per CTA
constexpr int kWinMaxC = 40;                      // C <= 31: h from 1 word per side; 31 < C <= 40: 2 words
constexpr int kWinLutMax = 2048;                  // K_sat bound of the window path
// E_df words of one staged row: the CTA's strips plus 1 word per side (C <= 31) or 2 (C > 31)
__host__ __device__ constexpr int window_row_words(int C) { return kWinWarps + (C > 31 ? 4 : 2); }
// registers per step whose two adds run on the FMA pipe (then one 3-way min on the ALU).  Measured
// (round 2, sensor-width kernels): 8 of 19 registers for the fp32 window (C3 window kernel -0.4 %,
// C5 +2.8 % vs 4), 4 for the small 8-bit / fp16 windows (8 loses 3.6 % / 4.8 % there)
__host__ __device__ constexpr int win_split(int C) {
#ifdef IEDS_WIN_SPLIT
    return IEDS_WIN_SPLIT;
#elif defined(IEDS_WIN_SPLIT_SMALL)
    return C >= 16 ? 8 : IEDS_WIN_SPLIT_SMALL;
#else
    return C >= 16 ? 8 : 4;
#endif
}

struct WinParams {
    const uint32_t* __restrict__ Edf;   // [nb][H][NW+2], word w of row y at 1 + w, zero guards
    void* __restrict__ S;               // [nb][H][W] float32, uint8 or float16 bits (OutT)
    const float* __restrict__ lut;      // [K_sat + 1], lut[K_sat] = the saturated value
    uint32_t* __restrict__ dummy;       // [nb][32] sink for the lanes of a ragged strip (x >= W)
    int W, H, NW;
    int RB;                             // rows per band (blockIdx.z); >= H: one band (the bulk path)
    int K_sat;                          // <= kWinLutMax
    uint32_t one;                       // 1 (runtime, so 0x10000 = one << 16 stays an IMAD operand)
    int nb;                             // windows of this launch (the packed grid's item count)
};

// row pairs a CTA stages: H rows plus zero rows for the reads past H (steps read pairs
// q < (H + C) / 2)
__host__ __device__ constexpr int window_staged_pairs(int H) { return (H + 2 * kWinMaxC + 2) / 2; }
// Packed CTAs (narrow frames, C <= 31): the 8 warps take 8 consecutive (window, strip) items
// of the launch, so no warp idles when the strips per window are not a multiple of 8; each warp
// stages its own words w-1, w, w+1 of every row.
constexpr int kWinPackedWords = 3;
// dynamic shared memory: [pairs][row words] uint2 {row 2q, row 2q+1}; packed: one such array
// of 3-word rows per warp
__host__ __device__ constexpr size_t window_smem_bytes(int H, int C, bool packed = false) {
    return packed ? 8ull * window_staged_pairs(H) * kWinPackedWords * kWinWarps
                  : 8ull * window_staged_pairs(H) * window_row_words(C);
}

// squared distance x4 from row u (first of a pair) to pixel y0 + j of the window, y0 = u - C + 1
template <int C>
__device__ __forceinline__ constexpr uint32_t dsq4(int j, int row_off) {
    const int d = j - (C - 1) - row_off;
    return (uint32_t)(4 * d * d);
}

__device__ __forceinline__ uint32_t clz_shiftamt(uint32_t x) {   // FLO.U32.SH; x != 0
    uint32_t r;
    asm("bfind.shiftamt.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}

// write-once output: streaming (evict-first) stores of the table's raw 32-bit pattern
__device__ __forceinline__ void st_cs_bits(float*, uint64_t addr, uint32_t bits) {
    asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(addr), "r"(bits) : "memory");
}
__device__ __forceinline__ void st_cs_bits(uint8_t*, uint64_t addr, uint32_t bits) {
    asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(addr), "r"(bits) : "memory");
}
__device__ __forceinline__ void st_cs_bits(uint16_t*, uint64_t addr, uint32_t bits) {   // float16 bits
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(addr), "h"((unsigned short)bits) : "memory");
}

// the same store at a compile-time byte offset from the base address (STG [R.64 + imm]): used by
// the width-specialised instantiations, whose row stride is a compile-time constant
template <int OFF>
__device__ __forceinline__ void st_cs_bits_at(float*, uint64_t addr, uint32_t bits) {
    asm volatile("st.global.cs.b32 [%0+%2], %1;" ::"l"(addr), "r"(bits), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void st_cs_bits_at(uint8_t*, uint64_t addr, uint32_t bits) {
    asm volatile("st.global.cs.u8 [%0+%2], %1;" ::"l"(addr), "r"(bits), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void st_cs_bits_at(uint16_t*, uint64_t addr, uint32_t bits) {
    asm volatile("st.global.cs.u16 [%0+%2], %1;" ::"l"(addr), "h"((unsigned short)bits), "n"(OFF) : "memory");
}

// WIDTH > 0: a sensor-width instantiation (row stride WIDTH * sizeof(OutT) bytes known at
// compile time).  When WIDTH % 32 != 0 the lanes of the last strip beyond the frame skip the
// rotations' stores (a loop-invariant predicate) and keep the ragged-strip sink for the rest.
template <int C, typename OutT, int PS = window_row_words(C), int WIDTH = 0>
struct WinState {
    static constexpr bool WIDE = C > 31;                  // h needs a second word per side
    static constexpr int RW = window_row_words(C);        // staged words per row (CTA-shared staging)
    static constexpr int OFF = WIDE ? 2 : 1;              // this strip's word w is at index OFF
    using ActT = typename std::conditional<(C > 32), uint64_t, uint32_t>::type;   // a bit per step
    int H, lane;
    int ya, yb;                        // rows this CTA emits (its band)
    uint64_t op;                       // byte address of the next pixel to emit (rows in order)
    uint32_t wb;                       // row stride in bytes (0 for lanes beyond W)
    uint32_t k65536;                   // 0x10000 (runtime: the half extracts stay IMADs)
    uint32_t one;                      // 1 (runtime: the split updates' adds stay IMADs)
    uint32_t ksat4x2;                  // 4*K_sat in both halves: the start value of every slot
    const uint32_t* lut;               // shared table, raw output bit patterns
    bool xok;                          // this lane's column lies inside the frame

    // h of a row for this lane from its strip's words (w-1, w, w+1), clamped to <= 31:
    // clz of (columns x-31..x with x at the MSB) | bitreverse(columns x..x+31) -- the leading
    // zero count of an OR is the min of the two one-sided distances; bit 0 bounds it by 31.
    __device__ __forceinline__ uint32_t h_of(uint32_t tl, uint32_t t, uint32_t tr) const {
        const uint32_t left = __funnelshift_rc(tl, t, lane + 1);
        const uint32_t right = __funnelshift_r(t, tr, lane);
        return clz_shiftamt(left | __brev(right) | 1u);
    }
    // WIDE (C > 31): words w-2 .. w+2; distances 0..31 from the inner pair of words (no guard
    // bit: an empty window reads 0xFFFFFFFF), 32..63 from the outer pair (guard bit: <= 63)
    __device__ __forceinline__ uint32_t h_of5(uint32_t tl2, uint32_t tl, uint32_t t, uint32_t tr, uint32_t tr2) const {
        const uint32_t near = __funnelshift_rc(tl, t, lane + 1) | __brev(__funnelshift_r(t, tr, lane));
        const uint32_t far = __funnelshift_rc(tl2, tl, lane + 1) | __brev(__funnelshift_r(tr, tr2, lane));
        return min(clz_shiftamt(near), 32u + clz_shiftamt(far | 1u));
    }
    // h of rows 2q, 2q+1 from this strip's staged words of pair q
    __device__ __forceinline__ void h_pair(const uint2* q, uint32_t& ha, uint32_t& hb) const {
        if constexpr (WIDE) {
            const uint2 a = q[0], l = q[1], c = q[2], r = q[3], z = q[4];
            ha = h_of5(a.x, l.x, c.x, r.x, z.x);
            hb = h_of5(a.y, l.y, c.y, r.y, z.y);
        } else {
            const uint2 l = q[0], c = q[1], r = q[2];
            ha = h_of(l.x, c.x, r.x);
            hb = h_of(l.y, c.y, r.y);
        }
    }
    // store table[idx4 / 4] at op and step op one row down; FAST: the rows left in this
    // window do not cross a 4 GB boundary, so only the low address word moves
    template <bool FAST>
    __device__ __forceinline__ void emit(uint32_t idx4) {
        const uint32_t bits = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(lut) + idx4);
        st_cs_bits(static_cast<OutT*>(nullptr), op, bits);
        if constexpr (FAST) {
            asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %0;\n\tadd.u32 lo, lo, %1;\n\t"
                "mov.b64 %0, {lo, hi};\n\t}" : "+l"(op) : "r"(wb));
        } else {
            op += wb;
        }
    }

    // Rotating window (steady state): before a pair step of phase S, logical register j
    // (pixels y0+2j, y0+2j+1 with y0 = u-C+1) lives in P[(j + S) % C].  The step applies the
    // sites of rows u, u+1 and shifts the window by one register, in place: logical j of the
    // new window is old logical j+1 min the two parabolas, and the freed register P[S % C]
    // becomes the new last register.  Then pixels y0, y0+1 are final -- a site C or more rows
    // away cannot bring a value below C^2 >= K_sat -- and are emitted.  Slots start at 4*K_sat
    // and only decrease, so every emitted value is a valid table offset.  `pr` points at this
    // strip's words of pair u0/2 (the rotation's first), so the row reads use immediate
    // offsets; bit S of `act` says whether rows u, u+1 hold a site fewer than C columns from
    // the strip.  All emitted rows lie inside the frame (the caller guarantees it).
    // sensor-width instantiations: table[idx4 / 4] stored at row ROW of the current rotation
    // (op = the rotation's first row), an immediate offset -- no per-pixel address arithmetic
    template <int ROW>
    __device__ __forceinline__ void emit_row(uint32_t idx4) {
        const uint32_t bits = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(lut) + idx4);
        if (WIDTH % 32 == 0 || xok) st_cs_bits_at<ROW * WIDTH * (int)sizeof(OutT)>(static_cast<OutT*>(nullptr), op, bits);
    }

    template <int S>
    __device__ __forceinline__ void step(const uint2* pr, ActT act, uint32_t (&P)[C]) {
        if (act & (ActT(1) << S)) {   // warp-uniform: a ballot result
            uint32_t ha, hb;
            h_pair(pr + S * PS, ha, hb);   // PS: uint2 stride between staged row pairs
            const uint32_t h2a = ha * ha * 0x40004u, h2b = hb * hb * 0x40004u;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const int m = (j + S + 1) % C;
                const uint32_t prev = (j + 1 < C) ? P[m] : ksat4x2;
                if (j < win_split(C)) {
                    // FMA-pipe adds (a plain 32-bit add is the packed add: no carry crosses
                    // the halves) and one 3-way packed min on the ALU
                    const uint32_t ta = h2a * one + sq2<0>(j), tb = h2b * one + sq2<1>(j);
                    P[m] = __vimin3_u16x2(prev, ta, tb);
                } else {
                    // two fused packed add+min: no carries cross the halves because every sum
                    // stays below 4 * (31^2 + 31^2) < 2^16
                    P[m] = __vminu2(__vminu2(prev, __vadd2(h2a, sq2<0>(j))), __vadd2(h2b, sq2<1>(j)));
                }
            }
        } else {
            P[S % C] = ksat4x2;   // the new last register starts empty
        }
        const uint32_t v = P[(S + 1) % C];
        const uint32_t hi = __umulhi(v, k65536), lo = v - hi * 0x10000u;
        if constexpr (WIDTH > 0) {
            emit_row<2 * S>(lo);
            emit_row<2 * S + 1>(hi);
            if constexpr (S == C - 1) op += (uint64_t)(2 * C) * wb;   // next rotation's rows (sink lanes: wb = 0)
        } else {
            emit<true>(lo);
            emit<true>(hi);
        }
    }

    // A rotation with no site in reach while every slot is still saturated (4 K_sat): its 2C
    // rows are the saturated value and the slots stay as they are -- store them directly.
    // sensor-width 8-bit / fp16 path: the warp's 2C x 32 outputs as 16-byte stores (the strip's
    // rows are 16-byte aligned: W * sizeof(OutT) % 16 == 0), 16 / sizeof(OutT) rows per store
    template <int K = 0>
    __device__ __forceinline__ void saturated_rows_v4(uint64_t base, uint32_t rep) {
        constexpr int LPR = 2 * (int)sizeof(OutT);   // lanes per row (16 bytes each)
        constexpr int RPI = 32 / LPR;                // rows per store instruction
        if constexpr (K * RPI < 2 * C) {
            if (K * RPI + lane / LPR < 2 * C) {
                asm volatile("st.global.cs.v4.b32 [%0+%1], {%2, %2, %2, %2};" ::"l"(base),
                             "n"(K * RPI * WIDTH * (int)sizeof(OutT)), "r"(rep) : "memory");
            }
            saturated_rows_v4<K + 1>(base, rep);
        }
    }

    template <int R = 0>
    __device__ __forceinline__ void saturated_rows(uint32_t bits) {
        if constexpr (WIDTH > 0 && sizeof(OutT) < 4 && R == 0) {
            constexpr int LPR = 2 * (int)sizeof(OutT);
            const uint32_t rep = sizeof(OutT) == 1 ? bits * 0x01010101u : bits * 0x00010001u;
            const uint64_t base = op - (uint64_t)(lane * sizeof(OutT)) +
                                  (uint64_t)(lane / LPR) * (WIDTH * sizeof(OutT)) + (uint64_t)(lane % LPR) * 16u;
            saturated_rows_v4(base, rep);
            op += (uint64_t)(2 * C) * wb;
        } else if constexpr (R < 2 * C) {
            if constexpr (WIDTH > 0) {
                st_cs_bits_at<R * WIDTH * (int)sizeof(OutT)>(static_cast<OutT*>(nullptr), op, bits);
            } else {
                st_cs_bits(static_cast<OutT*>(nullptr), op, bits);
                asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %0;\n\tadd.u32 lo, lo, %1;\n\t"
                    "mov.b64 %0, {lo, hi};\n\t}" : "+l"(op) : "r"(wb));
            }
            saturated_rows<R + 1>(bits);
        } else if constexpr (WIDTH > 0) {
            op += (uint64_t)(2 * C) * wb;
        }
    }

    template <int S>
    __device__ __forceinline__ void rotation(const uint2* pr, ActT act, uint32_t (&P)[C]) {
        if constexpr (S < C) {
            step<S>(pr, act, P);
            rotation<S + 1>(pr, act, P);
        }
    }

    // One pair step outside the steady state (the first rows, the last rows, or every row when
    // the fast address stepping is not allowed): a rolled loop body that keeps logical j in
    // P[j] by shifting the registers explicitly, checks the emitted rows against the frame and
    // steps the full 64-bit address.  Its code is one step long, so the hot rotation above is
    // the only large body in the instruction cache.
    __device__ __forceinline__ void step_rolled(const uint2* pq, int u, uint32_t (&P)[C]) {
        uint32_t ha, hb;
        h_pair(pq, ha, hb);
        if (__any_sync(0xFFFFFFFFu, min(ha, hb) < (uint32_t)C)) {
            const uint32_t h2a = ha * ha * 0x40004u, h2b = hb * hb * 0x40004u;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const uint32_t prev = (j + 1 < C) ? P[j + 1] : ksat4x2;
                P[j] = __vminu2(__vminu2(prev, __vadd2(h2a, sq2<0>(j))), __vadd2(h2b, sq2<1>(j)));
            }
        } else {
#pragma unroll
            for (int j = 0; j < C; ++j) P[j] = (j + 1 < C) ? P[j + 1] : ksat4x2;
        }
        const uint32_t v = P[0];
        const uint32_t hi = __umulhi(v, k65536), lo = v - hi * 0x10000u;
        const int y0 = u - (C - 1);
        if (y0 >= ya && y0 < yb) emit<false>(lo);
        if (y0 + 1 >= ya && y0 + 1 < yb) emit<false>(hi);
    }

    // The remaining n pair steps from u on lie beyond the frame (u >= H: staged zero rows, no
    // sites), so each would only shift the window and emit: step i would emit today's
    // P[i + 1] as rows u + 2i - C + 1, +1.  Emit them in place instead -- no h, no vote, no
    // shift.  Rows are checked against the band as in step_rolled, and emitted in the same order.
    __device__ __forceinline__ void flush(int u, int n, const uint32_t (&P)[C]) {
#pragma unroll
        for (int i = 0; i < C; ++i) {
            if (i >= n) break;
            const uint32_t v = (i + 1 < C) ? P[i + 1] : ksat4x2;
            const uint32_t hi = __umulhi(v, k65536), lo = v - hi * 0x10000u;
            const int y0 = u + 2 * i - (C - 1);
            if (y0 >= ya && y0 < yb) emit<false>(lo);
            if (y0 + 1 >= ya && y0 + 1 < yb) emit<false>(hi);
        }
    }

    // packed squared distances x4 from row u + R of a pair to pixels y0 + 2j, y0 + 2j + 1
    template <int R>
    __device__ __forceinline__ static constexpr uint32_t sq2(int j) {
        return dsq4<C>(2 * j, R) | (dsq4<C>(2 * j + 1, R) << 16);
    }
};

// CTAs per SM the register budget is sized for.  Measured (ms per C3 / C2 launch; 8-bit and
// fp16 surfaces/s at C3): C = 19 unpacked 5 / 4 / 3 CTAs: 0.827 / 0.82 / 0.828; C = 19 packed
// (C2): 0.166 / 0.158 / 0.150; C = 8 / 10 (8-bit / fp16): 1.50 / 1.42 M at 5, 1.46 / 1.36 M at 4,
// 1.48 / 1.40 M at 3; C = 31 / 40 (d_sat 9 / 12): 389 / 152 k at 2, 404 / 172 k at 3, 430 /
// 176 k at 4.  (6 CTAs: 40 registers with spills, slower everywhere.)
__host__ __device__ constexpr int window_min_ctas(int C, bool packed) {
#ifdef IEDS_WIN_CTAS_UNPACKED
    if (!packed && C > 12) return IEDS_WIN_CTAS_UNPACKED;
#endif
    return packed ? (C <= 12 ? 4 : 3) : (C <= 12 ? 5 : 4);
}

template <int C, typename OutT, bool PACKED = false, int WIDTH = 0>
__global__ void __launch_bounds__(kWinWarps * 32, window_min_ctas(C, PACKED)) window_kernel(WinParams p) {
    static_assert(!PACKED || C <= 31, "packed CTAs stage one word per side");
    static_assert(C >= 2 && C <= kWinMaxC, "window size (h: <= 31 from one word, <= 63 from two)");
    static_assert(C <= 31 || C >= 34, "two-word windows start at C = 34 (the activity masks)");
    static_assert(2 * C * WIDTH * (int)sizeof(OutT) < (1 << 23), "sensor width: immediate store offsets");
    constexpr int kWinRowWords = PACKED ? kWinPackedWords : window_row_words(C);   // uint2 stride between pairs
    using St = WinState<C, OutT, kWinRowWords, WIDTH>;
    __shared__ uint32_t lut_s[(C <= 31 ? 1024 : kWinLutMax) + 1];   // table, raw output bit patterns
    extern __shared__ __align__(16) uint32_t wsm[];      // row pairs of E_df words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = p.H, w0 = blockIdx.x * kWinWarps;
    const int NWP2 = p.NW + 2;
    // this warp's strip: word w of window b (packed: item blockIdx.x * 8 + warp of the launch)
    int b, w;
    bool valid;
    if constexpr (PACKED) {
        const int item = w0 + warp;
        valid = item < p.nb * p.NW;
        b = valid ? item / p.NW : 0;
        w = item - b * p.NW;
    } else {
        b = blockIdx.y;
        w = w0 + warp;
        valid = w < p.NW;
    }
    // this CTA's band of emitted rows [ya, yb) and the row pairs u in [u_first, u_last) it
    // steps over: every row within C - 1 of the band (the first ones only warm the window up)
    const int ya = blockIdx.z * p.RB, yb = min(H, ya + p.RB);
    const int u_first = max(0, ya - (C - 1)) & ~1;
    const int u_last = min(H + C - 1, yb + C - 1);
    const int NPS = window_staged_pairs(min(H, p.RB));
    const uint2* pairs = reinterpret_cast<const uint2*>(wsm);
    // stage words w0-1 .. w0+8 of every row (guard words / columns beyond the frame read 0)
    // plus zero rows past the end, interleaved by row pair: asynchronous 4-byte copies,
    // zero-filled where out of range, all in flight at once
    if constexpr (PACKED) {
        // each warp its own words w-1, w, w+1 (scratch indices w .. w+2, guards included)
        if (valid) {
            const uint32_t* src = p.Edf + ((size_t)b * H + u_first) * NWP2 + w;
            constexpr int kRowsPerPass = 32 / kWinPackedWords;   // 10 rows x 3 words per pass
            const int c = lane % kWinPackedWords, y_first = lane / kWinPackedWords;
            const uint32_t base =
                (uint32_t)__cvta_generic_to_shared(wsm) + 8u * (uint32_t)(warp * NPS * kWinPackedWords);
            if (y_first < kRowsPerPass) {
                for (int y = y_first; y < 2 * NPS; y += kRowsPerPass) {
                    const bool ok = u_first + y < H;
                    const uint32_t* g = ok ? src + (size_t)y * NWP2 + c : src;
                    const uint32_t dst =
                        base + 8u * (uint32_t)((y >> 1) * kWinPackedWords + c) + 4u * (uint32_t)(y & 1);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(g), "r"(ok ? 4 : 0)
                                 : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    } else {
        // staged word c of a row = scratch index w0 - OFF + 1 + c (word w0 - OFF + c; guards at
        // 0 and NW + 1, anything beyond the row reads 0); staged row 0 = row u_first
        const uint32_t* src = p.Edf + ((size_t)b * H + u_first) * NWP2;
        constexpr int kRowsPerPass = (kWinWarps * 32) / kWinRowWords;   // 25 rows x 10 words (21 x 12)
        const int c = threadIdx.x % kWinRowWords, y_first = threadIdx.x / kWinRowWords;
        const int sidx = w0 - St::OFF + 1 + c;
        const bool col_ok = sidx >= 0 && sidx < NWP2;
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(wsm);
        if (y_first < kRowsPerPass) {
            for (int y = y_first; y < 2 * NPS; y += kRowsPerPass) {
                const bool ok = col_ok && u_first + y < H;
                const uint32_t* g = ok ? src + (size_t)y * NWP2 + sidx : src;
                const uint32_t dst = base + 8u * (uint32_t)((y >> 1) * kWinRowWords + c) + 4u * (uint32_t)(y & 1);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(g), "r"(ok ? 4 : 0)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int i = threadIdx.x; i <= p.K_sat; i += blockDim.x) {
        const float f = p.lut[i];
        // the table holds values exactly representable in the output type
        if constexpr (std::is_same<OutT, uint8_t>::value) lut_s[i] = (uint32_t)f;
        else if constexpr (std::is_same<OutT, uint16_t>::value) lut_s[i] = __half_as_ushort(__float2half_rn(f));
        else lut_s[i] = __float_as_uint(f);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    if (!valid) return;
    const int x = 32 * w + lane;
    St st;
    st.H = H;
    st.lane = lane;
    st.ya = ya;
    st.yb = yb;
    st.k65536 = p.one << 16;
    st.one = p.one;
    st.ksat4x2 = (4u * (uint32_t)p.K_sat) * 0x10001u;
    st.lut = lut_s;
    st.xok = x < p.W;
    if (x < p.W) {
        st.op = reinterpret_cast<uint64_t>(reinterpret_cast<OutT*>(p.S) + (((size_t)b * H + ya) * p.W + x));
        st.wb = (uint32_t)(p.W * sizeof(OutT));
    } else {   // lanes of a ragged last strip write to a private sink, stride 0
        st.op = reinterpret_cast<uint64_t>(reinterpret_cast<OutT*>(p.dummy + 32 * (size_t)b) + lane);
        st.wb = 0;
    }
    // the unchecked rotations step only the low address word: every lane's column of this
    // window must lie inside one 4 GB-aligned range (else all rotations take the checked path)
    const uint64_t last = st.op + (uint64_t)st.wb * (uint64_t)(yb - ya - 1);
    const bool fast_ok = __all_sync(0xFFFFFFFFu, (last >> 32) == (st.op >> 32));
    // this strip's words w-OFF .. w+OFF of staged pair 0 (row u_first)
    const uint2* pr = PACKED ? pairs + warp * NPS * kWinPackedWords : pairs + warp;
    // columns within C-1 of the strip [32w - (C-1), 32w + 31 + (C-1)]: the outermost staged
    // words contribute their bits nearest the strip
    constexpr int kReach = St::WIDE ? C - 33 : C - 1;   // bits of the outermost word on each side
    constexpr uint32_t kLeft = ~0u << (32 - kReach);
    constexpr uint32_t kRight = (1u << kReach) - 1u;

    // Window of 2C pixels of this lane's column as 16-bit partial minima, two per register.
    uint32_t P[C];
#pragma unroll
    for (int k = 0; k < C; ++k) P[k] = st.ksat4x2;
    const int npairs = (u_last - u_first + 1) >> 1;   // staged row pairs this CTA steps over
    auto lp = [&](int uu) { return pr + ((uu - u_first) >> 1) * kWinRowWords; };
    int u = u_first;
    if (fast_ok) {
        // rows y0 = u - C + 1 < ya are not emitted: rolled steps until the first even u >= ya + C - 1
        for (; u < ya + C - 1 && u < u_last; u += 2) st.step_rolled(lp(u), u, P);
        // steady state: whole rotations whose emitted rows (up to u + C) all lie in the band
        for (; u + C < yb; u += 2 * C) {
            const int q0 = (u - u_first) >> 1;
            // activity of the rotation's C row pairs, lane j < C testing pair q0 + j: rows 2q,
            // 2q+1 hold a set pixel in columns [32w - (C-1), 32w + 31 + (C-1)], i.e. some lane
            // has h < C there (exactly the lanes' own test)
            // lanes j test pairs q0 + j (and q0 + 32 + j when C > 32)
            auto pair_any = [&](int q) -> bool {
                const uint2* qq = pr + q * kWinRowWords;
                if constexpr (St::WIDE) {
                    const uint2 a = qq[0], l = qq[1], m = qq[2], r = qq[3], z = qq[4];
                    return (((a.x | a.y) & kLeft) | l.x | l.y | m.x | m.y | r.x | r.y | ((z.x | z.y) & kRight)) != 0u;
                } else {
                    const uint2 a = qq[0], m = qq[1], r = qq[2];
                    return (((a.x | a.y) & kLeft) | m.x | m.y | ((r.x | r.y) & kRight)) != 0u;
                }
            };
            const bool lo = lane < C && q0 + lane < npairs && pair_any(q0 + lane);
            typename St::ActT act = __ballot_sync(0xFFFFFFFFu, lo);
            if constexpr (C > 32) {
                const bool hi = lane < C - 32 && q0 + 32 + lane < npairs && pair_any(q0 + 32 + lane);
                act |= (uint64_t)__ballot_sync(0xFFFFFFFFu, hi) << 32;
            }
            // (8-bit / fp16 only: 8-bit +5 %, fp16 +3 %; the fp32 window, bound by its stores
            // there, lost 0.4 % to the check and C5 1 %)
            if (sizeof(OutT) < 4 && act == 0) {   // warp-uniform: no site within reach of this rotation's rows
                uint32_t nz = 0;
#pragma unroll
                for (int k = 0; k < C; ++k) nz |= P[k] ^ st.ksat4x2;
                if (!__any_sync(0xFFFFFFFFu, nz != 0u)) {   // ... and nothing carried in either
                    st.saturated_rows(lut_s[p.K_sat]);
                    continue;
                }
            }
            st.template rotation<0>(pr + q0 * kWinRowWords, act, P);
        }
    }
    for (; u < u_last && u < H; u += 2) st.step_rolled(lp(u), u, P);
    if (u < u_last) st.flush(u, (u_last - u + 1) >> 1, P);   // pairs beyond the frame
}

}  // namespace ieds
