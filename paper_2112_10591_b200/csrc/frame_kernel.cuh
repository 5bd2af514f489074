// frame_kernel.cuh -- rows a1..a3 of the hot path, one CTA per window (per row band).
//
//   a1 scatter   events -> bit-packed edge image E in shared memory      (§III-A)
//   a2 denoise   E_d  = E   & [n4_E   >= N_d]                            (Alg. 1)
//   a3 fill      E_df = E_d | [n4_E_d >= N_f]                            (Alg. 2)
//   then, default path: E_df rows into the row-major scratch the window kernel reads (a2 and a3
//                fused into one read-only walk per word column, see df_walk);
//   exact path:  E_df transposed into column words T (bit i of T[r][x] = E_df(x, 32r+i)) plus a
//                per-column bitmap of non-empty word-rows, which is all the exact EDT needs.
//
// Layout: one CTA per (window, row band).  Band k covers frame rows [ylo, yhi) =
// [k * BR, min(H, (k + 1) * BR)) (BR = band_rows, a multiple of 32 when there are several bands;
// one band = the whole frame for every frame that fits, 1280x720 included).  Its shared-memory
// frame holds rows ylo - 3 .. yhi + 2 (a zero guard row, the two-row halo Alg. 1 + Alg. 2
// need on each side, and a zero guard row), BR + 6 rows of NWP words, after 4 zero words (so
// word -1 of the first row reads 0).  NWP = the smallest odd number > ceil(W/32): an odd row
// stride makes the "lane = row" accesses bank-conflict free and leaves at least one zero pad
// word per row.  fr1 points where frame row 0 would be, so frame row y is fr1 + y * NWP for
// every row the band touches; rows outside the frame and the pad words are zero, so
// out-of-frame neighbours read as non-edge (reading R1) without bounds checks.  Bit (x % 32)
// of word x / 32 is pixel x; bits beyond W stay 0.
#pragma once
#include <cstdint>

namespace ieds {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kErrRange = 1;   // an event outside the frame (dropped)
constexpr int kErrOrder = 2;   // window offsets not non-decreasing / out of range

struct FrameParams {
    const uint32_t* __restrict__ xy;        // [n_events] x | y << 16
    const int64_t* __restrict__ offsets;    // [nb + 1] absolute indices into xy
    int64_t n_events;
    int W, H, NW, NWP, NR, n_d, n_f;
    int band_rows, nbands;                  // rows per band (see Layout), bands per window
    int vec_ok;                             // xy is 16-byte aligned
    uint32_t* __restrict__ T;               // [nb][NR][W] transposed E_df
    unsigned long long* __restrict__ colmask;  // [nb][W] bit r = T[r][x] != 0
    uint32_t* __restrict__ E_out;           // [nb][H][NW] or null
    uint32_t* __restrict__ Ed_out;
    uint32_t* __restrict__ Edf_out;
    uint32_t* __restrict__ Edf_scratch;     // [nb][H][NW+2] E_df for the streaming surface kernel,
                                            // word w at 1 + w, zero guard words at 0 and NW + 1
    int* __restrict__ err;
    int nb;                                 // windows of this launch
    int prefetch_ahead;                     // > 0: L2-prefetch the events of window b + this (one wave later)
    int64_t prefetch_max;                   // bytes prefetched per window at most (a wave's share of L2)
};

// bulk prefetch of [p, p + bytes) into L2 (cp.async.bulk.prefetch; 16-byte granules, one thread)
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
    const uintptr_t a0 = (reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15;
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + (uintptr_t)bytes) & ~(uintptr_t)15;
    for (uintptr_t a = a0; a < a1; a += 65536) {
        const uint32_t n = (uint32_t)min((uintptr_t)65536, a1 - a);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    }
}

// bit-sliced "at least n of the four neighbour words are set", per bit position
__device__ __forceinline__ uint32_t at_least(int n, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    switch (n) {
        case 0: return kFull;
        case 1: return a | b | c | d;
        case 2: return (a & b) | (c & d) | ((a | b) & (c | d));
        case 3: return (a & b & (c | d)) | (c & d & (a | b));
        case 4: return a & b & c & d;
        default: return 0u;
    }
}

// frame word (y, w) through fr1 (frame row 0; see Layout), 0 outside the frame
__device__ __forceinline__ uint32_t frame_word(const uint32_t* fr1, const FrameParams& p, int y, int w) {
    return (y >= 0 && y < p.H && w >= 0 && w < p.NW) ? fr1[y * p.NWP + w] : 0u;
}

// E_d word (y, w): Alg. 1 on 32 pixels at once.
__device__ __forceinline__ uint32_t denoised_word(const uint32_t* fr, const FrameParams& p, int y, int w) {
    uint32_t c = frame_word(fr, p, y, w);
    uint32_t up = frame_word(fr, p, y - 1, w);
    uint32_t dn = frame_word(fr, p, y + 1, w);
    uint32_t lf = (c << 1) | (frame_word(fr, p, y, w - 1) >> 31);   // neighbour x-1
    uint32_t rt = (c >> 1) | (frame_word(fr, p, y, w + 1) << 31);   // neighbour x+1
    return c & at_least(p.n_d, up, dn, lf, rt);
}

// Sets the event's pixel if its row is one of the band's (ylo - 2 <= y < yhi + 2); returns
// nonzero if the event is outside the frame.  Branch-free: the coordinates are clamped into the
// frame with one packed min (lim = (H-1) << 16 | (W-1)), the row into the band, and an event
// outside either ORs nothing.
template <bool BANDED>
__device__ __forceinline__ uint32_t scatter_event(uint32_t* fr1, uint32_t lim, int NWP, int ya, int yb, uint32_t v) {
    const uint32_t c = __vminu2(v, lim);
    const int x = (int)(c & 0xFFFFu), y = (int)(c >> 16);
    if constexpr (BANDED) {
        const int yc = min(max(y, ya), yb);
        atomicOr(&fr1[yc * NWP + (x >> 5)], (c == v && yc == y) ? 1u << (x & 31) : 0u);
    } else {   // one band holds every row
        atomicOr(&fr1[y * NWP + (x >> 5)], c == v ? 1u << (x & 31) : 0u);
    }
    return c ^ v;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* ptr) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
    return r;
}

// 32x32 bit-matrix transpose across a warp: lane i holds row i on entry, column i on exit.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t v, int lane) {
#define IEDS_TSTEP(s, m)                                                              \
    {                                                                                 \
        uint32_t o = __shfl_xor_sync(kFull, v, s);                                    \
        v = (lane & s) ? ((v & ~(m)) | ((o & ~(m)) >> s)) : ((v & (m)) | ((o & (m)) << s)); \
    }
    IEDS_TSTEP(16, 0x0000FFFFu)
    IEDS_TSTEP(8, 0x00FF00FFu)
    IEDS_TSTEP(4, 0x0F0F0F0Fu)
    IEDS_TSTEP(2, 0x33333333u)
    IEDS_TSTEP(1, 0x55555555u)
#undef IEDS_TSTEP
    return v;
}

// E_d / E_df of one frame word from its shared-memory neighbourhood (guard rows/pad words = 0)
template <int N>
__device__ __forceinline__ uint32_t stencil_word(const uint32_t* fr, int i, int NWP) {
    const uint32_t c = fr[i];
    const uint32_t lf = (c << 1) | (fr[i - 1] >> 31);
    const uint32_t rt = (c >> 1) | (fr[i + 1] << 31);
    return at_least(N, fr[i - NWP], fr[i + NWP], lf, rt);
}

// (a & 0x80000000) | (b & 0x7FFFFFFF): bit 31 from a, the rest from b (one LOP3)
__device__ __forceinline__ uint32_t sel31(uint32_t a, uint32_t b) { return (a & 0x80000000u) | (b & 0x7FFFFFFFu); }

// E rows of one word column and its neighbours: l = word w-1, c = word w, r = word w+1
struct Row3 {
    uint32_t l, c, r;
};

// E_d (Alg. 1) of row r from E rows r-1 (a), r (m), r+1 (n):
//   d = word w;  s = bit 31: pixel 31 of word w-1, bit 0: pixel 0 of word w+1 (other bits junk)
template <int ND>
__device__ __forceinline__ void denoise_row(const Row3& a, const Row3& m, const Row3& n, uint32_t& d, uint32_t& s) {
    d = m.c & at_least(ND, a.c, n.c, __funnelshift_l(m.l, m.c, 1), __funnelshift_r(m.c, m.r, 1));
    // the neighbours of pixel 31 of word w-1 (bit 31) and of pixel 0 of word w+1 (bit 0):
    // left of (w-1, 31) is (w-1, 30); left of (w+1, 0) is (w, 31); right of (w-1, 31) is
    // (w, 0); right of (w+1, 0) is (w+1, 1)
    s = sel31(m.l, m.r) & at_least(ND, sel31(a.l, a.r), sel31(n.l, n.r), sel31(m.l << 1, m.c >> 31),
                                   sel31(m.c << 31, m.r >> 1));
}

// Alg. 1 then Alg. 2 for word column w of rows [y0, y1), fused as one top-to-bottom walk over
// the read-only E frame: E rows y-1..y+2 and E_d rows y-1..y+1 live in registers, each step
// loads one E row (3 words) and writes one E_df word.  fr1 = shared row 1 (frame row 0).
template <int ND, int NF, bool DBG>
__device__ __forceinline__ void df_walk(const uint32_t* fr1, const FrameParams& p, int b, int w, int y0, int y1,
                                        uint32_t wmask) {
    const int NWP = p.NWP;
    const uint32_t* q = fr1 + y0 * NWP + w;   // frame row y0, word w
    auto ld = [&](int dr) {                   // E row y0 + dr (rows -1, H, H+1 are zero guards)
        const uint32_t* t = q + dr * NWP;
        return Row3{t[-1], t[0], t[1]};
    };
    Row3 e0 = y0 > 0 ? ld(-2) : Row3{0u, 0u, 0u};   // row -2 does not exist: E_d(-1) = 0 anyway
    Row3 e1 = ld(-1), e2 = ld(0), e3 = ld(1);
    uint32_t dP, sP, dC, sC;
    denoise_row<ND>(e0, e1, e2, dP, sP);   // E_d(y0 - 1) (only its word w is used)
    denoise_row<ND>(e1, e2, e3, dC, sC);   // E_d(y0)
    Row3 eA = e2, eB = e3;                 // E rows y, y+1
    const size_t NW2 = (size_t)p.NW + 2;
    uint32_t* out = p.Edf_scratch + ((size_t)b * p.H + y0) * NW2 + 1 + w;
    const uint32_t* qn = q + 2 * NWP;      // E row y + 2
    for (int y = y0; y < y1; ++y) {
        const Row3 eN{qn[-1], qn[0], qn[1]};
        qn += NWP;
        uint32_t dN, sN;
        denoise_row<ND>(eA, eB, eN, dN, sN);   // E_d(y + 1)
        const uint32_t df =
            (dC | at_least(NF, dP, dN, __funnelshift_l(sC, dC, 1), __funnelshift_r(dC, sC, 1))) & wmask;
        *out = df;
        out += NW2;
        if constexpr (DBG) {
            const size_t o = ((size_t)b * p.H + y) * p.NW + w;
            if (p.Ed_out) p.Ed_out[o] = dC;
            if (p.Edf_out) p.Edf_out[o] = df;
        }
        dP = dC;
        dC = dN;
        sC = sN;
        eA = eB;
        eB = eN;
    }
}

// the default path's a2 + a3: word columns x row bands over the CTA's threads
template <int ND, int NF>
__device__ __forceinline__ void denoise_fill_walk(const uint32_t* fr1, const FrameParams& p, int b, int ylo, int yhi,
                                                  int tid, int nthr) {
    const int NW = p.NW;
    const int nbands = nthr / NW;   // >= 1 (host: NW <= threads)
    const int band = tid / NW, w = tid - band * NW;
    if (band >= nbands) return;
    const int rows = (yhi - ylo + nbands - 1) / nbands;
    const int y0 = ylo + band * rows, y1 = min(yhi, y0 + rows);
    if (y0 >= y1) return;
    const uint32_t wmask = (w == NW - 1 && (p.W & 31)) ? ((1u << (p.W & 31)) - 1u) : kFull;
    if (p.Ed_out || p.Edf_out)
        df_walk<ND, NF, true>(fr1, p, b, w, y0, y1, wmask);
    else
        df_walk<ND, NF, false>(fr1, p, b, w, y0, y1, wmask);
}

template <int ND>
__device__ __forceinline__ void denoise_fill_nf(const uint32_t* fr1, const FrameParams& p, int b, int ylo, int yhi,
                                                int tid, int nthr) {
    switch (p.n_f) {
        case 1: denoise_fill_walk<ND, 1>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 2: denoise_fill_walk<ND, 2>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 3: denoise_fill_walk<ND, 3>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 4: denoise_fill_walk<ND, 4>(fr1, p, b, ylo, yhi, tid, nthr); break;
        default: denoise_fill_walk<ND, 5>(fr1, p, b, ylo, yhi, tid, nthr); break;
    }
}

__device__ __forceinline__ void streaming_denoise_fill(const uint32_t* fr1, const FrameParams& p, int b, int ylo,
                                                       int yhi, int tid, int nthr) {
    switch (p.n_d) {
        case 0: denoise_fill_nf<0>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 1: denoise_fill_nf<1>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 2: denoise_fill_nf<2>(fr1, p, b, ylo, yhi, tid, nthr); break;
        case 3: denoise_fill_nf<3>(fr1, p, b, ylo, yhi, tid, nthr); break;
        default: denoise_fill_nf<4>(fr1, p, b, ylo, yhi, tid, nthr); break;
    }
}

// a1 for one window (and band): every event of [o0, o1), 16-byte streaming loads with
// kScatterLoads in flight per thread; returns nonzero if any event lies outside the frame
#ifndef IEDS_SCATTER_LOADS
#define IEDS_SCATTER_LOADS 8
#endif
constexpr int kScatterLoads = IEDS_SCATTER_LOADS;
template <bool BANDED>
__device__ __forceinline__ uint32_t scatter_window(uint32_t* fr1, const FrameParams& p, int64_t o0, int64_t o1, int ya,
                                                   int yb, int tid, int nthr) {
    uint32_t bad = 0;
    const uint32_t lim = ((uint32_t)(p.H - 1) << 16) | (uint32_t)(p.W - 1);
    const int NWP = p.NWP;
    if (p.vec_ok) {
        int64_t h1 = o1 < ((o0 + 3) & ~3ll) ? o1 : ((o0 + 3) & ~3ll);
        int64_t v1 = h1 > (o1 & ~3ll) ? h1 : (o1 & ~3ll);
        for (int64_t i = o0 + tid; i < h1; i += nthr) bad |= scatter_event<BANDED>(fr1, lim, NWP, ya, yb, __ldg(p.xy + i));
        const uint4* x4 = reinterpret_cast<const uint4*>(p.xy);
        int64_t j = (h1 >> 2) + tid;
        const int64_t j1 = v1 >> 2;
        auto apply4 = [&](const uint4& q) {
            return scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.x) | scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.y) |
                   scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.z) | scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.w);
        };
        for (; j + (kScatterLoads - 1) * nthr < j1; j += kScatterLoads * nthr) {   // kScatterLoads loads in flight
            uint4 q[kScatterLoads];
#pragma unroll
            for (int r = 0; r < kScatterLoads; ++r) q[r] = ld_stream_u4(x4 + j + r * nthr);
#pragma unroll
            for (int r = 0; r < kScatterLoads; ++r) bad |= apply4(q[r]);
        }
        for (; j < j1; j += nthr) {
            uint4 q = ld_stream_u4(x4 + j);
            bad |= scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.x) | scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.y) | scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.z) | scatter_event<BANDED>(fr1, lim, NWP, ya, yb, q.w);
        }
        for (int64_t i = v1 + tid; i < o1; i += nthr) bad |= scatter_event<BANDED>(fr1, lim, NWP, ya, yb, __ldg(p.xy + i));
    } else {
        for (int64_t i = o0 + tid; i < o1; i += nthr) bad |= scatter_event<BANDED>(fr1, lim, NWP, ya, yb, __ldg(p.xy + i));
    }
    return bad;
}

__global__ void __launch_bounds__(1024, 1) frame_kernel(FrameParams p) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int nframe = 4 + (p.band_rows + 6) * p.NWP;   // 4 zero words, then the band's rows (see Layout)
    uint32_t* fr = smem + 4;
    unsigned long long* cm = reinterpret_cast<unsigned long long*>(smem + ((nframe + 3) & ~3));
    const int b = blockIdx.x;
    const int ylo = blockIdx.y * p.band_rows, yhi = min(p.H, ylo + p.band_rows);
    const int ya = max(0, ylo - 2), yb = min(p.H - 1, yhi + 1);   // frame rows this band stores
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;

    // ---- clear the frame and the column bitmap
    {
        uint4 z = make_uint4(0, 0, 0, 0);
        uint4* f4 = reinterpret_cast<uint4*>(smem);   // from the 4 zero words on (see Layout)
        const int n4 = (nframe + 3) >> 2;
        for (int i = tid; i < n4; i += nthr) f4[i] = z;
        if (p.T)
            for (int i = tid; i < p.W; i += nthr) cm[i] = 0ull;
    }
    __syncthreads();

    // ---- a1: scatter this window's events (duplicates are idempotent; polarity absent)
    int64_t o0 = p.offsets[b], o1 = p.offsets[b + 1];
    if (o0 < 0 || o1 < o0 || o1 > p.n_events) {
        if (tid == 0) atomicOr(p.err, kErrOrder);
        o0 = o1 = 0;
    }
    uint32_t* fr1 = fr + (3 - ylo) * p.NWP;   // where frame row 0 would be (shared row 3 - ylo)
    const uint32_t bad = p.nbands == 1 ? scatter_window<false>(fr1, p, o0, o1, ya, yb, tid, nthr)
                                       : scatter_window<true>(fr1, p, o0, o1, ya, yb, tid, nthr);
    if (bad) atomicOr(p.err, kErrRange);
    __syncthreads();
    // the window one wave later starts when this wave's CTAs finish: stage its events in L2 now,
    // while this CTA's walk keeps the SM busy without HBM reads
    if (p.prefetch_ahead > 0 && tid == 0 && blockIdx.y == 0 && b + p.prefetch_ahead < p.nb) {
        const int64_t q0 = p.offsets[b + p.prefetch_ahead], q1 = p.offsets[b + p.prefetch_ahead + 1];
        if (q0 >= 0 && q1 > q0 && q1 <= p.n_events) prefetch_l2(p.xy + q0, min(4 * (q1 - q0), p.prefetch_max));
    }

    if (p.E_out) {
        uint32_t* out = p.E_out + (size_t)b * p.H * p.NW;
        const int n = (yhi - ylo) * p.NW;
        for (int i = tid; i < n; i += nthr) {
            const int y = ylo + i / p.NW, w = i % p.NW;
            out[(size_t)y * p.NW + w] = fr1[y * p.NWP + w];
        }
    }

    if (!p.T) {   // streaming surface path: row-major E_df only
        streaming_denoise_fill(fr1, p, b, ylo, yhi, tid, nthr);
        return;
    }

    // ---- a2 + a3 on 32x32 blocks (lane = row), then transpose the block into T
    const uint32_t lastmask = (p.W & 31) ? ((1u << (p.W & 31)) - 1u) : kFull;
    const int r0 = ylo / 32, nitems = ((yhi + 31) / 32 - r0) * p.NW;   // this band's word rows
    for (int item = warp; item < nitems; item += nwarps) {
        const int r = r0 + item / p.NW, w = item % p.NW;
        const int y = 32 * r + lane;
        const uint32_t cd = denoised_word(fr1, p, y, w);
        const uint32_t ld = denoised_word(fr1, p, y, w - 1);
        const uint32_t rd = denoised_word(fr1, p, y, w + 1);
        const uint32_t xd = denoised_word(fr1, p, lane == 0 ? 32 * r - 1 : 32 * r + 32, w);
        uint32_t up = __shfl_up_sync(kFull, cd, 1);
        uint32_t dn = __shfl_down_sync(kFull, cd, 1);
        if (lane == 0) up = xd;
        if (lane == 31) dn = xd;
        const uint32_t lf = (cd << 1) | (ld >> 31), rt = (cd >> 1) | (rd << 31);
        uint32_t df = cd | at_least(p.n_f, up, dn, lf, rt);
        if (w == p.NW - 1) df &= lastmask;
        if (y >= p.H) df = 0u;
        if (y < p.H) {
            const size_t o = ((size_t)b * p.H + y) * p.NW + w;
            if (p.Ed_out) p.Ed_out[o] = cd;
            if (p.Edf_out) p.Edf_out[o] = df;
        }
        const uint32_t t = warp_transpose32(df, lane);
        const int x = 32 * w + lane;
        if (x < p.W) {
            p.T[((size_t)b * p.NR + r) * p.W + x] = t;
            if (t) atomicOr(&cm[x], 1ull << r);
        }
    }
    __syncthreads();
    for (int x = tid; x < p.W; x += nthr) {
        if (p.nbands == 1) p.colmask[(size_t)b * p.W + x] = cm[x];
        else if (cm[x]) atomicOr(&p.colmask[(size_t)b * p.W + x], cm[x]);   // zeroed by the host
    }
}

}  // namespace ieds
