// Microbenchmark (tools only): DRAM write throughput of the window kernel's store pattern with
// no compute.  Grid (groups, windows); 8 warps per CTA; warp w of group g writes, for every row
// y of its window, 32 consecutive floats at column 32 * (8g + w) -- a coalesced 128-byte store
// per warp and row, rows W*4 bytes apart, windows H*W*4 apart.  Variants: st.global.cs vs
// st.global, and rows walked per warp (the kernel's order) vs a plain linear fill.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool CS>
__global__ void pattern(float* S, int W, int H, int NW, int rows_per_step) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w = blockIdx.x * 8 + warp;
    if (w >= NW) return;
    const int b = blockIdx.y;
    float* p = S + ((size_t)b * H) * W + 32 * w + lane;
    const float v = 1.0f;
    for (int y = 0; y < H; ++y) {
        if (CS) asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
        else asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
        p += W;
    }
}

__global__ void linear(float4* S, size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        S[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}

int main() {
    const int W = 1280, H = 720, NB = 1000, NW = W / 32;
    const size_t n = (size_t)NB * H * W;
    float* S;
    cudaMalloc(&S, n * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    dim3 g((NW + 7) / 8, NB);
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 3; ++v) {
            float best = 1e9f;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(a);
                if (v == 0) pattern<true><<<g, 256>>>(S, W, H, NW, 1);
                else if (v == 1) pattern<false><<<g, 256>>>(S, W, H, NW, 1);
                else linear<<<148 * 8, 256>>>(reinterpret_cast<float4*>(S), n / 4);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%s: %.4f ms  %.1f GB/s\n", v == 0 ? "pattern st.cs" : v == 1 ? "pattern st" : "linear float4", best,
                   n * 4.0 / (best / 1e3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
