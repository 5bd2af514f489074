// Microbenchmark (tools only): the L2 atomic ceiling of row f3's splat pattern.  Per event, the
// FWL splat issues one int32 atomicAdd with return (I_uncomp) and four fp64 atomicAdd with return
// (the bilinear corners of I_comp), into per-window scratch images of 1280x720 (16 windows per
// pass: 177 MB of images, the library's pass size).  Here the same five atomics per event run
// with no warp arithmetic at all, on edge-like synthetic events (75k per window, 90 % on short
// random segments, 10 % uniform noise), so events/s here is what the atomics alone allow.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

__global__ void splat_atomics(const uint32_t* xy, int64_t n_per, int W, int H, size_t stride, double* Ic, int* Iu,
                              double* sink) {
    const int b = blockIdx.y;
    double acc = 0.0;
    long long acci = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_per; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldg(xy + b * n_per + i);
        const int x = (int)(v & 0xFFFFu), y = (int)(v >> 16);
        acci += atomicAdd(Iu + b * stride + (size_t)y * W + x, 1);
        const int ix = min(x, W - 2), iy = min(y, H - 2);   // the warped corner (shifted by a fraction)
        double* c = Ic + b * stride + (size_t)iy * W + ix;
        acc += atomicAdd(c, 0.25) + atomicAdd(c + 1, 0.25) + atomicAdd(c + W, 0.25) + atomicAdd(c + W + 1, 0.25);
    }
    if (acc == -1.0 && acci == -1) sink[0] = acc;
}

int main() {
    const int W = 1280, H = 720, NB = 16, NPER = 75000;
    const size_t stride = (size_t)W * H;
    std::mt19937 rng(7);
    std::vector<uint32_t> h((size_t)NB * NPER);
    for (int b = 0; b < NB; ++b) {
        std::uniform_real_distribution<double> U(0, 1);
        for (int i = 0; i < NPER; ++i) {
            int x, y;
            if (i % 10 == 0) { x = (int)(U(rng) * W); y = (int)(U(rng) * H); }
            else {   // 90 segments of ~150 px per window, ~1 px jitter
                int s = i % 90;
                std::mt19937 r2(b * 1000 + s);
                std::uniform_real_distribution<double> V(0, 1);
                double x0 = V(r2) * W, y0 = V(r2) * H, a = V(r2) * 6.283, L = 30 + V(r2) * 230, t = U(rng) * L;
                x = (int)(x0 + t * cos(a) + (U(rng) - 0.5) * 2); y = (int)(y0 + t * sin(a) + (U(rng) - 0.5) * 2);
                x = ((x % W) + W) % W; y = ((y % H) + H) % H;
            }
            h[(size_t)b * NPER + i] = (uint32_t)x | ((uint32_t)y << 16);
        }
    }
    uint32_t* dxy; double* Ic; int* Iu; double* sink;
    cudaMalloc(&dxy, h.size() * 4);
    cudaMemcpy(dxy, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&Ic, sizeof(double) * stride * NB);
    cudaMalloc(&Iu, sizeof(int) * stride * NB);
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int nsm = 148; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int per_win : {4 * nsm / NB, 8 * nsm / NB, 16 * nsm / NB}) {
        float best = 1e9f;
        for (int it = 0; it < 6; ++it) {
            cudaMemset(Ic, 0, sizeof(double) * stride * NB);
            cudaMemset(Iu, 0, sizeof(int) * stride * NB);
            cudaEventRecord(e0);
            splat_atomics<<<dim3(per_win, NB), 256>>>(dxy, NPER, W, H, stride, Ic, Iu, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        const double ev = (double)NB * NPER / (best / 1e3);
        printf("{\"blocks_per_window\": %d, \"ms_per_pass\": %.4f, \"events_per_s\": %.4e, \"atomics_per_s\": %.4e}\n",
               per_win, best, ev, 5 * ev);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
