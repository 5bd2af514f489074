// flow.cu -- row f4: the flow consumer of the surfaces and the edge masking
// of P:248, on the GPU.  The estimator is the substitute of DESIGN reading R21 (
// the paper's own flow library gives no equations), step for step as oracle_flow_step:
//
//   J = scale * S; 2x2-mean pyramid;                   coarse to fine over the levels l:
//   Pt_l   = P_l(p - P_l(p))                            (previous flow transported by itself)
//   init   = Pt_{L-1} (coarsest) | 2 * bilinear upsample of F_{l+1}
//   J1     = J_prev,l sampled at p - init(p)            (border-clamped bilinear)
//   Ix, Iy = central differences of J1 (one-sided on the border), It = J_cur,l - J1
//   w      = K_l Jacobi sweeps from init:  w <- wbar - g (g . (wbar - init) + It) / (lambda_l + |g|^2)
//   F_l    = (1 - gamma) w + gamma Pt_l ;  P_l <- F_l
//   output = F_0, restricted to the denoised edge pixels E_d when given.
//
// fp32 throughout (the oracle is fp64; DESIGN states the tolerance).  Per level: one prep pass
// (transport, upsample, warp), one gradient pass, then the sweeps 4 at a time on shared-memory
// halo tiles with the temporal filter in the last launch's epilogue.  One step is 3 launches from the host: the level-0 scale (reads the caller's
// surface), one CUDA graph with every per-level kernel (captured once per pyramid parity,
// replayed each window), and the output / masking pass (writes the caller's buffers).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/ieds.h"

namespace cg = cooperative_groups;

namespace {

constexpr int kFT = 256;   // threads per block for the per-pixel kernels
constexpr int kMaxLevels = 8;

__device__ __forceinline__ float bl1(const float* __restrict__ I, int W, int H, float sx, float sy) {
    sx = fminf(fmaxf(sx, 0.f), (float)(W - 1));
    sy = fminf(fmaxf(sy, 0.f), (float)(H - 1));
    const int x0 = (int)floorf(sx), y0 = (int)floorf(sy);
    const float fx = sx - (float)x0, fy = sy - (float)y0;
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    return (1.f - fx) * (1.f - fy) * I[(size_t)y0 * W + x0] + fx * (1.f - fy) * I[(size_t)y0 * W + x1] +
           (1.f - fx) * fy * I[(size_t)y1 * W + x0] + fx * fy * I[(size_t)y1 * W + x1];
}

__device__ __forceinline__ float2 bl2(const float2* __restrict__ I, int W, int H, float sx, float sy) {
    sx = fminf(fmaxf(sx, 0.f), (float)(W - 1));
    sy = fminf(fmaxf(sy, 0.f), (float)(H - 1));
    const int x0 = (int)floorf(sx), y0 = (int)floorf(sy);
    const float fx = sx - (float)x0, fy = sy - (float)y0;
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const float2 a = I[(size_t)y0 * W + x0], b = I[(size_t)y0 * W + x1], c = I[(size_t)y1 * W + x0],
                 d = I[(size_t)y1 * W + x1];
    const float wa = (1.f - fx) * (1.f - fy), wb = fx * (1.f - fy), wc = (1.f - fx) * fy, wd = fx * fy;
    return make_float2(wa * a.x + wb * b.x + wc * c.x + wd * d.x, wa * a.y + wb * b.y + wc * c.y + wd * d.y);
}

#define IEDS_PIX(W, H)                                                  \
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y; \
    if (x >= (W) || y >= (H)) return;                                    \
    const size_t p = (size_t)y * (W) + x;

__global__ void scale_kernel(const float* __restrict__ S, float* __restrict__ J, int W, int H, float s) {
    IEDS_PIX(W, H)
    J[p] = s * S[p];
}

__global__ void down_kernel(const float* __restrict__ src, int Ws, float* __restrict__ dst, int W, int H) {
    IEDS_PIX(W, H)
    const float* a = src + (size_t)(2 * y) * Ws + 2 * x;
    dst[p] = (a[0] + a[1] + a[Ws] + a[Ws + 1]) * 0.25f;
}

// The per-level inputs of the sweeps, one pass per pixel:
//   Pt   = P_l(p - P_l(p))                        (the previous flow transported by itself)
//   init = Pt (coarsest level) | 2 * bilinear upsample of the coarser level's new flow
//   J1   = J_prev,l sampled at p - init(p)       (border-clamped bilinear)
__global__ void prep_kernel(const float2* __restrict__ P, const float2* __restrict__ Fc, int Wc, int Hc,
                            const float* __restrict__ Jprev, float2* __restrict__ Pt, float2* __restrict__ init,
                            float* __restrict__ J1, int W, int H) {
    IEDS_PIX(W, H)
    const float2 f = P[p];
    const float2 pt = bl2(P, W, H, (float)x - f.x, (float)y - f.y);
    Pt[p] = pt;
    float2 in = pt;
    if (Fc) {
        const float2 v = bl2(Fc, Wc, Hc, ((float)x + 0.5f) * 0.5f - 0.5f, ((float)y + 0.5f) * 0.5f - 0.5f);
        in = make_float2(2.f * v.x, 2.f * v.y);
    }
    init[p] = in;
    J1[p] = bl1(Jprev, W, H, (float)x - in.x, (float)y - in.y);
}

// G = (Ix, Iy, It, 1 / (lambda + Ix^2 + Iy^2)) at pixel (x, y): central differences of J1
// (one-sided on the border), It = Jc - J1; the last entry is 0 where the denominator is 0
// (w = wbar there)
__device__ __forceinline__ float4 flow_grad(const float* __restrict__ J1, const float* __restrict__ Jc, size_t p, int x,
                                            int y, int W, int H, float lam) {
    float ix, iy;
    if (W == 1) ix = 0.f;
    else if (x == 0) ix = J1[p + 1] - J1[p];
    else if (x == W - 1) ix = J1[p] - J1[p - 1];
    else ix = (J1[p + 1] - J1[p - 1]) * 0.5f;
    if (H == 1) iy = 0.f;
    else if (y == 0) iy = J1[p + W] - J1[p];
    else if (y == H - 1) iy = J1[p] - J1[p - W];
    else iy = (J1[p + W] - J1[p - W]) * 0.5f;
    const float den = lam + ix * ix + iy * iy;
    return make_float4(ix, iy, Jc[p] - J1[p], den > 0.f ? 1.f / den : 0.f);
}

__global__ void grad_kernel(const float* __restrict__ J1, const float* __restrict__ Jc, float4* __restrict__ G, int W,
                            int H, float lam) {
    IEDS_PIX(W, H)
    G[p] = flow_grad(J1, Jc, p, x, y, W, H, lam);
}

// K Jacobi sweeps in one launch (temporal blocking): a CTA loads its tile plus a K-pixel halo
// of w into shared memory (G and init of its cells stay in registers), runs K sweeps on a
// shrinking region and writes the tile.  After sweep s every cell at least s cells inside the
// region is exact, so the tile (K inside) equals K plain sweeps over the whole level, operation
// for operation: the same clamped (replicate) border neighbours and the same fp32 expressions:
//   w <- wbar - g (g . (wbar - init) + It) / (lambda + |g|^2),  G = (Ix, Iy, It, 1/(lambda + |g|^2)).
// Region of 64 x 32 cells per CTA (threads 32 x 8; a thread owns columns tx, tx + 32 and rows
// ty + 8j, j < 4), tile = region minus K on every side.
constexpr int kTbRX = 64, kTbRY = 32, kTbThreads = 256, kTbMaxK = 4;

struct TbParams {
    const float2* win;     // w before these sweeps (init for the first launch)
    float2* wout;          // w after them, or with blend: F = (1 - gamma) w + gamma Pt
    const float2* init;
    const float4* G;       // (Ix, Iy, It, 1 / (lambda + Ix^2 + Iy^2)) per pixel
    const float2* Pt;      // with blend: the transported previous flow
    float gamma;
    int W, H;
    int kk;                // sweeps of this launch, 1..kTbMaxK
    int blend;             // last launch of the level: write F into the level's flow state
};

// tile of a CTA: the region minus a kTbMaxK-pixel halo on every side
constexpr int kTbTX = kTbRX - 2 * kTbMaxK, kTbTY = kTbRY - 2 * kTbMaxK;
inline dim3 tb_grid(int W, int H) { return dim3((W + kTbTX - 1) / kTbTX, (H + kTbTY - 1) / kTbTY); }

// One CTA's part of q.kk sweeps (see above): load the region of q.win, sweep, write the tile.
__device__ __forceinline__ void tb_body(const TbParams& q, float2 (&sw)[2][kTbRY][kTbRX]) {
    constexpr int K = kTbMaxK;
    const int W = q.W, H = q.H, kk = q.kk;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * kTbTX - K, y0 = blockIdx.y * kTbTY - K;
    float4 g[2][4];
    float2 i0[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int rx = tx + 32 * a, ry = ty + 8 * j, gx = x0 + rx, gy = y0 + ry;
            if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
                const size_t p = (size_t)gy * W + gx;
                sw[0][ry][rx] = q.win[p];
                g[a][j] = q.G[p];
                i0[a][j] = q.init[p];
            }
        }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < K; ++s) {
        if (s >= kk) break;
        const float2(*src)[kTbRX] = sw[s & 1];
        float2(*dst)[kTbRX] = sw[(s + 1) & 1];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int rx = tx + 32 * a, ry = ty + 8 * j, gx = x0 + rx, gy = y0 + ry;
                if (rx <= s || rx >= kTbRX - 1 - s || ry <= s || ry >= kTbRY - 1 - s) continue;   // not exact
                if (gx < 0 || gx >= W || gy < 0 || gy >= H) continue;
                const float2 l = src[ry][gx > 0 ? rx - 1 : rx], r = src[ry][gx < W - 1 ? rx + 1 : rx];
                const float2 u = src[gy > 0 ? ry - 1 : ry][rx], d = src[gy < H - 1 ? ry + 1 : ry][rx];
                const float mx = (l.x + r.x + u.x + d.x) * 0.25f, my = (l.y + r.y + u.y + d.y) * 0.25f;
                const float4 gg = g[a][j];
                const float res = gg.x * (mx - i0[a][j].x) + gg.y * (my - i0[a][j].y) + gg.z;
                dst[ry][rx] = make_float2(mx - gg.x * res * gg.w, my - gg.y * res * gg.w);
            }
        __syncthreads();
    }
    const float2(*fin)[kTbRX] = sw[kk & 1];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int rx = tx + 32 * a, ry = ty + 8 * j, gx = x0 + rx, gy = y0 + ry;
            if (rx < K || rx >= K + kTbTX || ry < K || ry >= K + kTbTY || gx >= W || gy >= H) continue;
            const size_t p = (size_t)gy * W + gx;
            const float2 w = fin[ry][rx];
            if (q.blend) {
                const float2 b = q.Pt[p];
                q.wout[p] = make_float2((1.f - q.gamma) * w.x + q.gamma * b.x, (1.f - q.gamma) * w.y + q.gamma * b.y);
            } else {
                q.wout[p] = w;
            }
        }
}

__global__ void __launch_bounds__(kTbThreads) jacobi_tb_kernel(TbParams q) {
    __shared__ float2 sw[2][kTbRY][kTbRX];
    tb_body(q, sw);
}

// All of a level's sweeps in one cooperative launch (levels whose tiles are all co-resident):
// chunks of kTbMaxK sweeps with a grid-wide barrier between them, ping-ponging w0 / w1 from
// init, the last chunk writing the filtered flow F.  Same tiles, same operations.
__global__ void __launch_bounds__(kTbThreads) jacobi_coop_kernel(TbParams q, int sweeps, float2* w0, float2* w1,
                                                                 float2* F) {
    __shared__ float2 sw[2][kTbRY][kTbRX];
    cg::grid_group grid = cg::this_grid();
    const float2* a = q.init;
    for (int k = 0; k < sweeps; k += kTbMaxK) {
        const bool last = k + kTbMaxK >= sweeps;
        TbParams c = q;
        c.win = a;
        c.wout = last ? F : (a == w0 ? w1 : w0);
        c.kk = min(kTbMaxK, sweeps - k);
        c.blend = last ? 1 : 0;
        tb_body(c, sw);
        if (!last) grid.sync();
        a = c.wout;
    }
}

__global__ void blend_kernel(const float2* __restrict__ w, const float2* __restrict__ Pt, float2* __restrict__ F,
                             int64_t n, float gamma) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float2 a = w[i], b = Pt[i];
    F[i] = make_float2((1.f - gamma) * a.x + gamma * b.x, (1.f - gamma) * a.y + gamma * b.y);
}

// caller's outputs: the level-0 flow, restricted to E_d (bit (x % 32) of word [y][x / 32]) when
// given; `first` = the first window of a sequence (zero flow, nothing valid)
__global__ void out_kernel(const float2* __restrict__ F0, const uint32_t* __restrict__ Ed, int NW, float2* __restrict__ out,
                           uint8_t* __restrict__ valid, int W, int H, int first) {
    IEDS_PIX(W, H)
    int v = first ? 0 : 1;
    if (Ed && v) v = (Ed[(size_t)y * NW + (x >> 5)] >> (x & 31)) & 1u;
    const bool dense = !Ed && !first;
    out[p] = (v || dense) ? F0[p] : make_float2(0.f, 0.f);
    if (valid) valid[p] = (uint8_t)v;
}

inline dim3 pgrid(int W, int H) { return dim3((W + kFT - 1) / kFT, H); }

}  // namespace

struct ieds_flow_handle {
    ieds_flow_config cfg{};
    int dev = 0, L = 0;
    int Ws[kMaxLevels]{}, Hs[kMaxLevels]{};
    size_t off[kMaxLevels]{}, tot = 0;
    float* pyr[2] = {nullptr, nullptr};   // ping-pong pyramids (previous / current)
    float2* P = nullptr;                  // per-level flow (state)
    float2 *init = nullptr, *Pt = nullptr, *w0 = nullptr, *w1 = nullptr;
    float* J1 = nullptr;
    float4* G = nullptr;
    int cur = 0;                          // pyramid buffer that receives the next window
    bool fresh = true;
    cudaStream_t cs = nullptr;            // capture stream
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int64_t coop_blocks = 0;              // sweep CTAs that can be co-resident (0: no cooperative launch)
};

namespace {

struct FlowDevGuard {
    int prev = -1;
    bool ok = true;
    explicit FlowDevGuard(int dev) {
        ok = cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess;
    }
    ~FlowDevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// whether level l runs its sweeps as one cooperative launch: more than one chunk of sweeps, and
// all of its tiles co-resident on the device
bool coop_level(const ieds_flow_handle* h, int l) {
    const dim3 tg = tb_grid(h->Ws[l], h->Hs[l]);
    return h->cfg.iterations[l] > kTbMaxK && (int64_t)tg.x * tg.y <= h->coop_blocks;
}

// every per-level kernel of one non-first step, reading pyr[1-c] as previous, pyr[c] as current
void enqueue_levels(ieds_flow_handle* h, int c, cudaStream_t st) {
    float* cur = h->pyr[c];
    const float* prev = h->pyr[1 - c];
    for (int l = 1; l < h->L; ++l)
        down_kernel<<<pgrid(h->Ws[l], h->Hs[l]), kFT, 0, st>>>(cur + h->off[l - 1], h->Ws[l - 1], cur + h->off[l],
                                                               h->Ws[l], h->Hs[l]);
    for (int l = h->L - 1; l >= 0; --l) {
        const int W = h->Ws[l], H = h->Hs[l];
        float2* Pl = h->P + h->off[l];
        const bool coarsest = l == h->L - 1;
        prep_kernel<<<pgrid(W, H), kFT, 0, st>>>(Pl, coarsest ? nullptr : h->P + h->off[l + 1],
                                                 coarsest ? 0 : h->Ws[l + 1], coarsest ? 0 : h->Hs[l + 1],
                                                 prev + h->off[l], h->Pt, h->init, h->J1, W, H);
        // K sweeps from w^0 = init, kTbMaxK per launch ping-ponging w0 / w1; the last launch
        // writes F_l = (1 - gamma) w + gamma Pt_l into the state
        const int K = h->cfg.iterations[l];
        if (K == 0) {   // no sweeps: F = the filter of init and Pt (w = init)
            const int64_t n = (int64_t)W * H;
            blend_kernel<<<(unsigned)((n + kFT - 1) / kFT), kFT, 0, st>>>(h->init, h->Pt, Pl, n, (float)h->cfg.gamma);
            continue;
        }
        grad_kernel<<<pgrid(W, H), kFT, 0, st>>>(h->J1, cur + h->off[l], h->G, W, H, (float)h->cfg.lambda[l]);
        TbParams q;
        q.win = h->init;
        q.init = h->init;
        q.G = h->G;
        q.Pt = h->Pt;
        q.gamma = (float)h->cfg.gamma;
        q.W = W;
        q.H = H;
        const dim3 tg = tb_grid(W, H);
        if (coop_level(h, l)) {   // every chunk in one launch, grid-wide barriers between them
            int sweeps = K;
            float2 *w0 = h->w0, *w1 = h->w1, *F = Pl;
            void* args[] = {&q, &sweeps, &w0, &w1, &F};
            // an error here is sticky for the capture: ieds_flow_step reports it at the end of capture
            (void)cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_coop_kernel), tg, dim3(kTbThreads), args, 0,
                                              st);
            continue;
        }
        const float2* a = h->init;
        for (int k = 0; k < K; k += kTbMaxK) {
            const bool last = k + kTbMaxK >= K;
            float2* b = last ? Pl : (a == h->w0 ? h->w1 : h->w0);
            q.win = a;
            q.wout = b;
            q.kk = std::min(kTbMaxK, K - k);
            q.blend = last ? 1 : 0;
            jacobi_tb_kernel<<<tg, kTbThreads, 0, st>>>(q);
            a = b;
        }
    }
}

void free_flow(ieds_flow_handle* h) {
    for (int i = 0; i < 2; ++i) {
        if (h->gexec[i]) cudaGraphExecDestroy(h->gexec[i]);
        cudaFree(h->pyr[i]);
    }
    cudaFree(h->P);
    cudaFree(h->init);
    cudaFree(h->Pt);
    cudaFree(h->w0);
    cudaFree(h->w1);
    cudaFree(h->J1);
    cudaFree(h->G);
    if (h->cs) cudaStreamDestroy(h->cs);
}

}  // namespace

extern "C" {

int ieds_flow_create(const ieds_flow_config* cfg, ieds_flow_handle** out) {
    if (!out) return IEDS_EINVAL;
    *out = nullptr;
    if (!cfg || cfg->levels < 1 || cfg->levels > kMaxLevels || cfg->width < 2 || cfg->height < 2 ||
        cfg->width > 65535 || cfg->height > 65535)
        return IEDS_EINVAL;
    if (!(cfg->gamma >= 0.0 && cfg->gamma <= 1.0) || !(cfg->scale > 0.0) || !std::isfinite(cfg->scale)) return IEDS_EINVAL;
    auto h = new ieds_flow_handle();
    h->cfg = *cfg;
    h->L = cfg->levels;
    for (int l = 0; l < h->L; ++l) {
        if (cfg->iterations[l] < 0 || cfg->iterations[l] > 100000 || !(cfg->lambda[l] >= 0.0) ||
            !std::isfinite(cfg->lambda[l])) {
            delete h;
            return IEDS_EINVAL;
        }
        h->Ws[l] = l == 0 ? cfg->width : h->Ws[l - 1] / 2;
        h->Hs[l] = l == 0 ? cfg->height : h->Hs[l - 1] / 2;
        if (h->Ws[l] < 2 || h->Hs[l] < 2) {
            delete h;
            return IEDS_EINVAL;
        }
        h->off[l] = h->tot;
        h->tot += (size_t)h->Ws[l] * h->Hs[l];
    }
    int dev = cfg->device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
        delete h;
        return IEDS_ECUDA;
    }
    h->dev = dev;
    FlowDevGuard g(dev);
    if (!g.ok) {
        delete h;
        return IEDS_ECUDA;
    }
    const size_t n0 = (size_t)cfg->width * cfg->height;
    cudaError_t e = cudaMalloc(&h->pyr[0], sizeof(float) * h->tot);
    if (e == cudaSuccess) e = cudaMalloc(&h->pyr[1], sizeof(float) * h->tot);
    if (e == cudaSuccess) e = cudaMalloc(&h->P, sizeof(float2) * h->tot);
    if (e == cudaSuccess) e = cudaMalloc(&h->init, sizeof(float2) * n0);
    if (e == cudaSuccess) e = cudaMalloc(&h->Pt, sizeof(float2) * n0);
    if (e == cudaSuccess) e = cudaMalloc(&h->w0, sizeof(float2) * n0);
    if (e == cudaSuccess) e = cudaMalloc(&h->w1, sizeof(float2) * n0);
    if (e == cudaSuccess) e = cudaMalloc(&h->J1, sizeof(float) * n0);
    if (e == cudaSuccess) e = cudaMalloc(&h->G, sizeof(float4) * n0);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        int coop = 0, nsm = 0, per_sm = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (coop && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel, kTbThreads, 0) == cudaSuccess)
            h->coop_blocks = (int64_t)per_sm * nsm;
        if (const char* ev = std::getenv("IEDS_FLOW_COOP"))
            if (std::atoi(ev) == 0) h->coop_blocks = 0;
        cudaGetLastError();
    }
    if (e != cudaSuccess) {
        free_flow(h);
        delete h;
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? IEDS_ENOMEM : IEDS_ECUDA;
    }
    *out = h;
    return IEDS_OK;
}

void ieds_flow_destroy(ieds_flow_handle* h) {
    if (!h) return;
    FlowDevGuard g(h->dev);
    cudaDeviceSynchronize();
    free_flow(h);
    delete h;
}

int ieds_flow_reset(ieds_flow_handle* h) {
    if (!h) return IEDS_EINVAL;
    h->fresh = true;
    return IEDS_OK;
}

int ieds_flow_step(ieds_flow_handle* h, const float* surface, const uint32_t* edge_bits, float* flow, uint8_t* valid,
                   void* stream) {
    if (!h || !surface || !flow) return IEDS_EINVAL;
    FlowDevGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int W = h->cfg.width, H = h->cfg.height, NW = (W + 31) / 32;
    const int c = h->cur;
    cudaError_t e = cudaSuccess;
    scale_kernel<<<pgrid(W, H), kFT, 0, st>>>(surface, h->pyr[c], W, H, (float)h->cfg.scale);
    const bool first = h->fresh;
    if (first) {
        float* cur = h->pyr[c];
        for (int l = 1; l < h->L; ++l)
            down_kernel<<<pgrid(h->Ws[l], h->Hs[l]), kFT, 0, st>>>(cur + h->off[l - 1], h->Ws[l - 1], cur + h->off[l],
                                                                   h->Ws[l], h->Hs[l]);
        e = cudaMemsetAsync(h->P, 0, sizeof(float2) * h->tot, st);
    } else {
        if (!h->gexec[c]) {   // capture this parity's step once
            cudaGraph_t graph = nullptr;
            e = cudaStreamBeginCapture(h->cs, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                enqueue_levels(h, c, h->cs);
                e = cudaStreamEndCapture(h->cs, &graph);
            }
            if (e == cudaSuccess) e = cudaGraphInstantiate(&h->gexec[c], graph, 0);
            if (graph) cudaGraphDestroy(graph);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return IEDS_ECUDA;
            }
        }
        e = cudaGraphLaunch(h->gexec[c], st);
    }
    if (e == cudaSuccess) {
        out_kernel<<<pgrid(W, H), kFT, 0, st>>>(h->P, edge_bits, NW, reinterpret_cast<float2*>(flow), valid, W, H,
                                                first ? 1 : 0);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return IEDS_ECUDA;
    h->fresh = false;
    h->cur = 1 - c;
    return IEDS_OK;
}

int64_t ieds_flow_launches_per_step(const ieds_flow_handle* h) {
    if (!h) return 0;
    int64_t n = 2 + (h->L - 1);   // scale, down kernels, output
    for (int l = 0; l < h->L; ++l)   // prep, then grad + the sweeps (the last one blends), or a blend alone
        n += h->cfg.iterations[l] > 0 ? 2 + (coop_level(h, l) ? 1 : (h->cfg.iterations[l] + kTbMaxK - 1) / kTbMaxK) : 2;
    return n;
}

}  // extern "C"

namespace ieds {
// geometry and device of a flow handle, for the pipeline in ieds.cu (not part of the C ABI)
int flow_dims(const ieds_flow_handle* h, int* width, int* height, int* device) {
    if (!h) return IEDS_EINVAL;
    *width = h->cfg.width;
    *height = h->cfg.height;
    *device = h->dev;
    return IEDS_OK;
}
}  // namespace ieds
