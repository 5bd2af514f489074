// edt_kernel.cuh -- rows a4 (exact EDT) and a5 (Eq. (1) surface), one CTA per (window, band
// of 32 rows).  Lane = row of the band, warp = segment of SEGW consecutive columns.
//
// Exact separable EDT (§III-C: Coeurjolly et al.'s separable exact EDT family):
//   pass A (columns): g(x,y) = distance from (x,y) to the nearest E_df pixel of column x,
//           read in O(1) from the transposed bit words T written by the frame kernel plus the
//           nearest non-empty word-rows above/below the band (per-column bitmap);
//   pass B (rows):    D2(x,y) = min_q (x-q)^2 + g(q,y)^2 = lower envelope of parabolas.
//           Each warp builds the envelope of its segment's parabolas (Felzenszwalb-
//           Huttenlocher stack, exact 64-bit integer intersection comparisons), the
//           segment envelopes are merged pairwise in a tree (an entry is removed while it is
//           dominated by its neighbours at the junction, as in Cao et al.'s PBA), and each
//           warp then evaluates its pixels by walking the merged envelope.
// Surface (Eq. (1)): S = 1 - exp(-sqrt(D2)/alpha) from an fp64-built fp32 table
// over the integer D2; S is exactly 1.0f from the saturation index K_sat on.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace ieds {

constexpr int kGInf = 0x8000;   // g >= kGInf: column has no E_df pixel

struct EdtParams {
    const uint32_t* __restrict__ T;                // [nb][NR][W]
    const unsigned long long* __restrict__ colmask;  // [nb][W]
    int W, H, NR, NS, SEGW;
    void* __restrict__ S;                           // [nb][H][W] float32 / uint8 / float16 (out_fmt), or null
    uint32_t* __restrict__ D2;                      // [nb][H][W] or null
    const float* __restrict__ lut;                  // [K_lut]
    int K_lut, K_sat;
    float c_exp;                                    // -log2(e) / alpha
    int transfer, out_fmt;                          // IEDS_TRANSFER_*, IEDS_OUT_*
    float bound, sat_value, empty_value;            // saturated value (D2 >= K_sat), empty frame
};

struct SmemLayout {
    uint32_t* tword;   // [W]
    uint32_t* gap;     // [W]  lo16: rows from band top to nearest E_df row above; hi16: below
    float* lut;        // [K_lut]
    uint16_t* lo;      // [NS][32] surviving entry range of each segment's stack, per row
    uint16_t* hi;
    float* stg;        // [NS][32*9]
    uint32_t* stgd;    // [NS][32*9] (only if D2 requested)
    uint8_t* stk;      // [NS][SEGW][32] envelope stacks, site offset within the segment
};

// g(x, y) for y = band top + lane, from the column word t and the gap word.
__device__ __forceinline__ int gval(uint32_t t, uint32_t gp, int lane, uint32_t mle, uint32_t mge) {
    const uint32_t ui = t & mle, di = t & mge;
    const int up = ui ? (lane - (31 - __clz(ui))) : (lane + (int)(gp & 0xFFFFu));
    const int dn = di ? (__ffs(di) - 1 - lane) : ((31 - lane) + (int)(gp >> 16));
    return min(up, dn);
}

struct Ent {
    int seg, idx;   // seg < 0: none
    int site, f;    // column, g^2
};

struct EdtCtx {
    const SmemLayout& sm;
    int SEGW, lane;
    uint32_t mle, mge;

    __device__ __forceinline__ int lo(int s) const { return sm.lo[s * 32 + lane]; }
    __device__ __forceinline__ int hi(int s) const { return sm.hi[s * 32 + lane]; }
    __device__ __forceinline__ int fval(int q) const {
        const int g = gval(sm.tword[q], sm.gap[q], lane, mle, mge);
        return g * g;
    }
    __device__ __forceinline__ Ent make(int s, int i) const {
        Ent e;
        e.seg = s;
        e.idx = i;
        e.site = s * SEGW + sm.stk[(s * SEGW + i) * 32 + lane];
        e.f = fval(e.site);
        return e;
    }
    __device__ __forceinline__ Ent none() const {
        Ent e;
        e.seg = -1; e.idx = 0; e.site = 0; e.f = 0;
        return e;
    }
    // previous surviving entry, not crossing below segment s0
    __device__ __forceinline__ Ent prev(const Ent& e, int s0) const {
        if (e.idx - 1 >= lo(e.seg)) return make(e.seg, e.idx - 1);
        for (int s = e.seg - 1; s >= s0; --s)
            if (hi(s) > lo(s)) return make(s, hi(s) - 1);
        return none();
    }
    // next surviving entry, not crossing segment s1 (exclusive)
    __device__ __forceinline__ Ent next(const Ent& e, int s1) const {
        if (e.idx + 1 < hi(e.seg)) return make(e.seg, e.idx + 1);
        for (int s = e.seg + 1; s < s1; ++s)
            if (hi(s) > lo(s)) return make(s, lo(s));
        return none();
    }
};

// q is not on the lower envelope of {p, q, r} (p < q < r): z(p,q) >= z(q,r)
__device__ __forceinline__ bool dominated(const Ent& p, const Ent& q, const Ent& r) {
    const long long kp = (long long)p.f + (long long)p.site * p.site;
    const long long kq = (long long)q.f + (long long)q.site * q.site;
    const long long kr = (long long)r.f + (long long)r.site * r.site;
    return (kq - kp) * (long long)(r.site - q.site) >= (kr - kq) * (long long)(q.site - p.site);
}

// transfer of an exact squared distance (Eq. (1) or a §IV-D ablation, see ieds.h): the
// fp64-built table below K_lut, the saturated value from K_sat, fp32 arithmetic in between
// (only reached for large alpha / unbounded transfers)
__device__ __forceinline__ float transfer_value(uint32_t d2, const float* lut, const EdtParams& p) {
    if (d2 < (uint32_t)p.K_lut) return lut[d2];
    if (d2 == 0xFFFFFFFFu) return p.empty_value;
    if (d2 >= (uint32_t)p.K_sat) return p.sat_value;
    const float d = sqrtf((float)d2);   // d2 < 2^24: exact input, correctly rounded
    switch (p.transfer) {
        case 0: return 1.0f - exp2f(p.c_exp * d);
        case 1: return d;
        case 2: return fminf(d, p.bound);
        default: return log1pf(d);
    }
}

__device__ __forceinline__ int envF(int x, const Ent& e) {
    const int d = x - e.site;
    return d * d + e.f;
}

__global__ void __launch_bounds__(512) edt_kernel(EdtParams p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int W = p.W, NS = p.NS, SEGW = p.SEGW;
    SmemLayout sm;
    {
        unsigned char* q = smraw;
        sm.tword = reinterpret_cast<uint32_t*>(q); q += 4 * W;
        sm.gap = reinterpret_cast<uint32_t*>(q); q += 4 * W;
        sm.lut = reinterpret_cast<float*>(q); q += 4 * ((p.K_lut + 3) & ~3);
        sm.lo = reinterpret_cast<uint16_t*>(q); q += 2 * 32 * NS;
        sm.hi = reinterpret_cast<uint16_t*>(q); q += 2 * 32 * NS;
        sm.stg = reinterpret_cast<float*>(q); q += 4 * 32 * 9 * NS;
        sm.stgd = reinterpret_cast<uint32_t*>(q); if (p.D2) q += 4 * 32 * 9 * NS;
        sm.stk = q;
    }
    const int r = blockIdx.x, b = blockIdx.y;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    const int y0 = 32 * r;

    // ---- phase 0: column words of this band and the gaps to the nearest E_df rows outside it
    {
        const uint32_t* Tb = p.T + (size_t)b * p.NR * W;
        const unsigned long long* cmb = p.colmask + (size_t)b * W;
        for (int x = tid; x < W; x += nthr) {
            const uint32_t t = Tb[(size_t)r * W + x];
            const unsigned long long m = cmb[x];
            uint32_t gu = 0xFFFFu, gd = 0xFFFFu;
            const unsigned long long above = m & ((1ull << r) - 1ull);
            if (above) {
                const int r2 = 63 - __clzll(above);
                const uint32_t t2 = Tb[(size_t)r2 * W + x];
                gu = (uint32_t)(y0 - (32 * r2 + 31 - __clz(t2)));
            }
            const unsigned long long below = (r + 1 < 64) ? (m >> (r + 1)) : 0ull;
            if (below) {
                const int r3 = r + __ffsll(below);
                const uint32_t t3 = Tb[(size_t)r3 * W + x];
                gd = (uint32_t)(32 * r3 + __ffs(t3) - 1 - (y0 + 31));
            }
            sm.tword[x] = t;
            sm.gap[x] = gu | (gd << 16);
        }
        for (int i = tid; i < p.K_lut; i += nthr) sm.lut[i] = p.lut[i];
    }
    __syncthreads();

    const uint32_t mle = (lane == 31) ? kFull : ((2u << lane) - 1u);   // bits 0..lane
    const uint32_t mge = kFull << lane;                                  // bits lane..31
    EdtCtx cx{sm, SEGW, lane, mle, mge};

    // ---- phase 1: lower envelope of each segment (warp = segment, lane = row)
    for (int s = warp; s < NS; s += nwarps) {
        const int a_s = s * SEGW, b_s = min(W, a_s + SEGW);
        uint8_t* st = sm.stk + (size_t)s * SEGW * 32;
        int n = 0, bt = 0, kb = 0, at = 0, ka = 0;
        for (int x = a_s; x < b_s; ++x) {
            const int g = gval(sm.tword[x], sm.gap[x], lane, mle, mge);
            if (g < kGInf) {
                const int k = g * g + x * x;
                while (n >= 2) {
                    // pop the top b if z(b, x) <= z(a, b)
                    if ((long long)(k - kb) * (bt - at) > (long long)(kb - ka) * (x - bt)) break;
                    --n;
                    bt = at;
                    kb = ka;
                    if (n >= 2) {
                        at = a_s + st[(n - 2) * 32 + lane];
                        ka = cx.fval(at) + at * at;
                    }
                }
                st[n * 32 + lane] = (uint8_t)(x - a_s);
                at = bt;
                ka = kb;
                bt = x;
                kb = k;
                ++n;
            }
        }
        sm.lo[s * 32 + lane] = 0;
        sm.hi[s * 32 + lane] = (uint16_t)n;
    }
    __syncthreads();

    // ---- phase 2: merge segment envelopes pairwise (tree over segments)
    for (int stride = 1; stride < NS; stride *= 2) {
        for (int m = warp; stride * (2 * m + 1) < NS; m += nwarps) {
            const int j = stride * (2 * m + 1);
            const int jl = j - stride, jr = min(NS, j + stride);
            int sl = -1, sr = -1;
            for (int s = j - 1; s >= jl; --s)
                if (cx.hi(s) > cx.lo(s)) { sl = s; break; }
            for (int s = j; s < jr; ++s)
                if (cx.hi(s) > cx.lo(s)) { sr = s; break; }
            if (sl >= 0 && sr >= 0) {
                Ent eb = cx.make(sl, cx.hi(sl) - 1);
                Ent ec = cx.make(sr, cx.lo(sr));
                Ent ea = cx.prev(eb, jl);
                Ent ed = cx.next(ec, jr);
                for (;;) {
                    if (ea.seg >= 0 && dominated(ea, eb, ec)) {
                        sm.hi[eb.seg * 32 + lane] = (uint16_t)eb.idx;   // drop b (last of left)
                        eb = ea;
                        ea = cx.prev(eb, jl);
                        continue;
                    }
                    if (ed.seg >= 0 && dominated(eb, ec, ed)) {
                        sm.lo[ec.seg * 32 + lane] = (uint16_t)(ec.idx + 1);   // drop c (first of right)
                        ec = ed;
                        ed = cx.next(ec, jr);
                        continue;
                    }
                    break;
                }
            }
        }
        __syncthreads();
    }

    // ---- phase 3: evaluate D2 on each segment by walking the merged envelope; write S
    const size_t plane = (size_t)p.H * W;
    float* Sb = reinterpret_cast<float*>(p.S) + (size_t)b * plane;
    uint8_t* Qb = reinterpret_cast<uint8_t*>(p.S) + (size_t)b * plane;
    __half* Hb = reinterpret_cast<__half*>(p.S) + (size_t)b * plane;
    uint32_t* Db = p.D2 ? p.D2 + (size_t)b * plane : nullptr;
    for (int s = warp; s < NS; s += nwarps) {
        const int a_s = s * SEGW, b_s = min(W, a_s + SEGW);
        float* stg = sm.stg + s * 32 * 9;
        uint32_t* stgd = sm.stgd + s * 32 * 9;
        // start at the tail of segments [0, s), else the head of [s, NS)
        Ent cur = cx.none();
        for (int q = s - 1; q >= 0; --q)
            if (cx.hi(q) > cx.lo(q)) { cur = cx.make(q, cx.hi(q) - 1); break; }
        if (cur.seg < 0)
            for (int q = s; q < NS; ++q)
                if (cx.hi(q) > cx.lo(q)) { cur = cx.make(q, cx.lo(q)); break; }
        const bool empty = cur.seg < 0;   // E_df of this window is empty
        Ent nxt = cx.none();
        if (!empty) {
            for (;;) {
                Ent pv = cx.prev(cur, 0);
                if (pv.seg >= 0 && envF(a_s, pv) <= envF(a_s, cur)) cur = pv;
                else break;
            }
            nxt = cx.next(cur, NS);
        }
        for (int x = a_s; x < b_s; ++x) {
            uint32_t d2 = 0xFFFFFFFFu;
            if (!empty) {
                while (nxt.seg >= 0 && envF(x, nxt) < envF(x, cur)) {
                    cur = nxt;
                    nxt = cx.next(cur, NS);
                }
                d2 = (uint32_t)envF(x, cur);
            }
            const float v = transfer_value(d2, sm.lut, p);
            const int c = (x - a_s) & 7;
            stg[lane * 9 + c] = v;
            if (Db) stgd[lane * 9 + c] = d2;
            if (c == 7 || x == b_s - 1) {
                __syncwarp();
                const int xb = x - c;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int row = 4 * k + (lane >> 3), col = lane & 7;
                    const int y = y0 + row;
                    if (y < p.H && col <= c) {
                        if (p.S) {
                            const size_t o = (size_t)y * W + xb + col;
                            const float v = stg[row * 9 + col];
                            if (p.out_fmt == 1) Qb[o] = (uint8_t)v;
                            else if (p.out_fmt == 2) Hb[o] = __float2half_rn(v);   // table values: exact
                            else Sb[o] = v;
                        }
                        if (Db) Db[(size_t)y * W + xb + col] = stgd[row * 9 + col];
                    }
                }
                __syncwarp();
            }
        }
    }
}

}  // namespace ieds
