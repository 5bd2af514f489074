// surface_kernel.cuh -- rows a4 + a5 in the saturation-aware streaming form (the default when
// the caller does not request D2).  One warp per (window, strip of 32 columns); lane = column.
//
// Eq. (1) saturates: in fp32, S = 1 - exp(-sqrt(D2)/alpha) is exactly 1.0f for
// D2 >= K_sat (K_sat = 353 for alpha = 6/ln 255).  Let c = ceil(sqrt(K_sat)).  Any E_df pixel
// at squared distance < K_sat lies within c-1 rows and c-1 columns, so
//   D2(x,y) = min over rows y' with h(x,y') < c of (y-y')^2 + h(x,y')^2   whenever D2 < K_sat,
// where h(x,y') = horizontal distance from (x,y') to the nearest E_df pixel of row y'
// (separable exact EDT, with the column pass capped -- SURVEY.md §8(c) "capping
// lemma").  Every candidate is a true squared distance, so when D2 >= K_sat the computed value
// is >= K_sat as well and S = 1.0f exactly: the fp32 surface equals the exact-EDT surface.
//
// Per warp the rows are streamed top to bottom: row y_in's site (h < c) is pushed onto a
// Felzenszwalb-Huttenlocher lower envelope of parabolas (y - y')^2 + h^2 (exact 64-bit integer
// intersection test), then pixel y_out = y_in - (c-1) -- whose candidate rows are all pushed
// -- is evaluated by walking the envelope and written (lanes = 32 consecutive columns: one
// coalesced 128-byte store per row).  Sites more than c-1 rows above y_out can no longer
// matter, so the envelope lives in a 64-entry ring per lane in shared memory.
#pragma once
#include <cstdint>

namespace ieds {

constexpr int kRing = 64;           // ring entries per lane (c <= 32)
constexpr int kSurfWarps = 8;       // warps (strips) per CTA

struct SurfParams {
    const uint32_t* __restrict__ Edf;   // [nb][H][NW] row-major E_df words
    float* __restrict__ S;              // [nb][H][W]
    const float* __restrict__ lut;      // [K_lut]
    int W, H, NW;
    int K_lut, K_sat;
    int c;                              // ceil(sqrt(K_sat)) <= 32
    float c_exp;
};

// horizontal distance from column 32w+j to the nearest set bit of (tl | t | tr) within the
// three words; >= 32 means "none within 32 columns" (c <= 32 makes that sufficient).
__device__ __forceinline__ int hdist(uint32_t t, int fl, int fr, int j, uint32_t mle, uint32_t mge) {
    const uint32_t ui = t & mle, di = t & mge;
    const int left = ui ? (j - (31 - __clz(ui))) : (j + fl);      // fl = 32 - hibit(tl), or big
    const int right = di ? (__ffs(di) - 1 - j) : ((31 - j) + fr); // fr = lobit(tr) + 1, or big
    return min(left, right);
}

__device__ __forceinline__ uint32_t ring_pack(int site, int h) { return ((uint32_t)site << 5) | (uint32_t)h; }

__global__ void __launch_bounds__(kSurfWarps * 32) surface_kernel(SurfParams p) {
    __shared__ uint16_t ring_all[kSurfWarps][kRing][32];
    __shared__ float lut_s[1024];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < p.K_lut; i += blockDim.x) lut_s[i] = p.lut[i];
    __syncthreads();

    const int w = blockIdx.x * kSurfWarps + warp;
    if (w >= p.NW) return;
    const int b = blockIdx.y;
    const int W = p.W, H = p.H, NW = p.NW, c = p.c;
    const int lag = c - 1;
    const int x = 32 * w + lane;
    const bool xvalid = x < W;
    uint16_t (*ring)[32] = ring_all[warp];
    const uint32_t* Eb = p.Edf + (size_t)b * H * NW;
    float* Sb = p.S + (size_t)b * H * W + x;
    const uint32_t mle = (lane == 31) ? 0xFFFFFFFFu : ((2u << lane) - 1u);
    const uint32_t mge = 0xFFFFFFFFu << lane;
    const int kBig = 1 << 12;

    // envelope state (per lane): entries [flo, n) of the ring are live; top two cached
    int n = 0, flo = 0;
    int sb = 0, kb = 0, sa = 0, ka = 0;       // top (b) and second (a): site, key = h^2 + site^2
    // eval state: pointer pe, cached cur/nxt (site, f = h^2)
    int pe = 0, cs = 0, cf = 0, ns = 0, nf = 0;
    bool have_cur = false, have_nxt = false;
    int sflo = 0;                              // site of entry flo (cached)

    const uint32_t* rowp = Eb + w;
    for (int yi = 0; yi < H + lag; ++yi) {
        // ---------------- push site yi (rows with an E_df pixel within c-1 columns)
        if (yi < H) {
            const uint32_t t = rowp[(size_t)yi * NW];
            const uint32_t tl = (w > 0) ? rowp[(size_t)yi * NW - 1] : 0u;
            const uint32_t tr = (w + 1 < NW) ? rowp[(size_t)yi * NW + 1] : 0u;
            if ((t | tl | tr) != 0u) {
                const int fl = tl ? (32 - (31 - __clz(tl))) : kBig;
                const int fr = tr ? __ffs(tr) : kBig;
                const int h = hdist(t, fl, fr, lane, mle, mge);
                if (h < c) {
                    const int k = h * h + yi * yi;
                    int touched = n;   // lowest depth modified
                    while (n - flo >= 2) {
                        // pop top b if z(b, yi) <= z(a, b)
                        if ((long long)(k - kb) * (sb - sa) > (long long)(kb - ka) * (yi - sb)) break;
                        --n;
                        sb = sa;
                        kb = ka;
                        if (n - flo >= 2) {
                            const uint32_t e = ring[(n - 2) & (kRing - 1)][lane];
                            sa = (int)(e >> 5);
                            const int ha = (int)(e & 31u);
                            ka = ha * ha + sa * sa;
                        }
                    }
                    touched = min(touched, n);
                    ring[n & (kRing - 1)][lane] = (uint16_t)ring_pack(yi, h);
                    if (n - flo >= 1) {
                        sa = sb;
                        ka = kb;
                    }
                    sb = yi;
                    kb = k;
                    if (n == flo) sflo = yi;
                    ++n;
                    // the owner of the last pixel may have been popped: restart the walk from the
                    // (unchanged) entry just below the modified depth
                    if (touched <= pe) {
                        pe = max(flo, touched - 1);
                        have_cur = false;
                        have_nxt = false;
                    } else if (touched == pe + 1) {
                        have_nxt = false;
                    }
                }
            }
        }
        // ---------------- evaluate pixel yo
        const int yo = yi - lag;
        if (yo < 0) continue;
        // drop entries that can no longer reach a near pixel (site <= yo - c)
        // (the live entries [flo, n) stay a valid FH stack: its first entry is never popped)
        while (flo < n && sflo <= yo - c) {
            ++flo;
            if (flo < n) sflo = (int)(ring[flo & (kRing - 1)][lane] >> 5);
        }
        uint32_t d2 = 0xFFFFFFFFu;
        if (n > flo) {
            if (pe < flo) {
                pe = flo;
                have_cur = false;
                have_nxt = false;
            }
            if (pe >= n) {
                pe = n - 1;
                have_cur = false;
                have_nxt = false;
            }
            if (!have_cur) {
                const uint32_t e = ring[pe & (kRing - 1)][lane];
                cs = (int)(e >> 5);
                const int hc = (int)(e & 31u);
                cf = hc * hc;
                have_cur = true;
                have_nxt = false;
            }
            int dc = (yo - cs) * (yo - cs) + cf;
            for (;;) {
                if (pe + 1 >= n) break;
                if (!have_nxt) {
                    const uint32_t e = ring[(pe + 1) & (kRing - 1)][lane];
                    ns = (int)(e >> 5);
                    const int hn = (int)(e & 31u);
                    nf = hn * hn;
                    have_nxt = true;
                }
                const int dn = (yo - ns) * (yo - ns) + nf;
                if (dn >= dc) break;
                ++pe;
                cs = ns;
                cf = nf;
                dc = dn;
                have_nxt = false;
            }
            d2 = (uint32_t)dc;
        }
        float v;
        if (d2 < (uint32_t)p.K_lut) v = lut_s[d2];
        else if (d2 >= (uint32_t)p.K_sat) v = 1.0f;
        else v = 1.0f - exp2f(p.c_exp * sqrtf((float)d2));
        if (xvalid) Sb[(size_t)yo * W] = v;
    }
}

}  // namespace ieds
