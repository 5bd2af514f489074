// ieds.cu -- C ABI (include/ieds.h) of the batched IEDS build on B200 (sm_100a).
//
// Host side: configuration validation, scratch ownership, the fp64-built Eq. (1) table,
// stream-ordered launches chunk by chunk (launch shapes: row bands for large frames and for
// small batches), the latched device error flag, and the pipelined host-buffer entry point.
// Kernels: frame_kernel.cuh (a1-a3), window_kernel.cuh (a4-a5, default), edt_kernel.cuh
// (a4-a5 exact everywhere), norm_kernel.cuh (row f1 normalised 8-bit), windowing_kernel.cuh
// (row f2), fwl_kernel.cuh (row f3).  Row f4 lives in flow.cu.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/ieds.h"
#include "frame_kernel.cuh"
#include "edt_kernel.cuh"
#include "window_kernel.cuh"
#include "windowing_kernel.cuh"
#include "norm_kernel.cuh"
#include "fwl_kernel.cuh"

#ifndef IEDS_VERSION_STR
#define IEDS_VERSION_STR "ieds-b200 0.1 (sm_100a)"
#endif

namespace {

constexpr int kFrameThreads = 1024;
constexpr int kMaxSmem = 232448;   // 227 KB opt-in per block
constexpr int kLutMax = ieds::kWinLutMax;
// columns per EDT segment (warp), by what the exact kernel writes.  Surfaces only (exact flag):
// 48 / 64 / 80 / 112 / 128 / 144 / 160 measured 99.7 / 99.7 / 99.7 / 86.5 / 106.8 / 101.2 / 97.5 k
// surfaces/s at C3 (1280 = 10 segments of 128).  With D2 written (sqdist, the normalised 8-bit
// view): 80 gives 72.5 k, 128 62.5 k normalised surfaces/s.
constexpr int kSegTarget = 128, kSegTargetD2 = 80;
// row f3: windows per splat pass.  Each window's images are 12 B/px of scratch, hit by the
// splat's atomics and then re-zeroed by a memset; 16 windows at 1280x720 measured best
// (4: 118k, 8: 141k, 16: 146k, 32: 131k windows/s; 64 spills far out of L2: 63k).
// IEDS_FWL_CHUNK overrides it (read once per handle).
constexpr int kFwlChunkDefault = 16;

struct HostPath {
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};    // chunk's copies + kernels finished
    cudaEvent_t kdone[2] = {nullptr, nullptr};   // chunk's kernels finished (scratch free)
    uint32_t* d_xy[2] = {nullptr, nullptr};
    int64_t* d_off[2] = {nullptr, nullptr};
    float* d_S[2] = {nullptr, nullptr};   // (uint8 surfaces use the same buffers)
    int64_t* h_off[2] = {nullptr, nullptr};   // pinned, rebased offsets
    int64_t cap_ev[2] = {0, 0};
};

}  // namespace

struct ProfPool {
    bool on = false;
    std::vector<cudaEvent_t> ev;   // pairs (start, end)
    std::vector<int> kind;         // per pair
    size_t used = 0;               // pairs recorded since last read
};

struct ieds_handle {
    ieds_config cfg;
    int dev;
    int NW, NWP, NR, NS, SEGW;
    int NS_d2, SEGW_d2;        // the exact kernel's segments when it writes D2
    int band_rows, nbands;     // frame kernel: rows per CTA band, bands per window (frame_kernel.cuh)
    int nsm;                   // SMs of the device (small batches spread a window over several)
    int l2_bytes;              // L2 size of the device
    int chunk;        // windows per launch pair of the device path (scratch capacity)
    int host_chunk;   // windows per pipelined copy/compute step of the host path (<= chunk)
    size_t smem_frame, smem_edt, smem_edt_d2;
    int c_sat;                 // ceil(sqrt(K_sat)): rows/columns a near site can be away
    int c_win;                 // window size of the branch-free kernel (>= c_sat)
    bool streaming;            // saturation-aware window kernel usable (K_sat <= 1024)
    bool norm_u8;              // 8-bit view of Id / min / ln normalised by the frame maximum
    bool exact_ok;             // the exact-EDT kernel fits this width (sqdist requests need it)
    bool win_packed = false;   // window kernel CTAs take strips of several windows (narrow frames)
    uint32_t* D2n = nullptr;   // norm_u8: [chunk][H][W] exact D2 scratch
    uint32_t* wmax = nullptr;  // norm_u8: [chunk] per-window max D2
    double* vtab = nullptr;    // norm_u8: [(W-1)^2 + (H-1)^2 + 1] fp64 transfer of every D2
    // row f3 scratch (allocated on the first ieds_fwl_batch): fwl_chunk windows of images
    int fwl_chunk = 0;
    double* fwl_Ic[2] = {nullptr, nullptr};   // two sets of [fwl_chunk][stride] fp64 images, zero when idle
    int* fwl_Iu[2] = {nullptr, nullptr};      // [fwl_chunk][stride] int32
    ieds::FwlPart* fwl_part = nullptr;        // [fwl_chunk][reduce blocks] per-block partial sums
    cudaStream_t fwl_zs = nullptr;            // re-zeroes a set while the other is splatted
    cudaEvent_t fwl_splat[2] = {nullptr, nullptr}, fwl_zero[2] = {nullptr, nullptr};
    int fwl_next = 0;                         // the set the next pass uses
    uint32_t* T = nullptr;     // exact path: [chunk][NR][W] transposed E_df
    uint32_t* Edfs = nullptr;  // streaming path: [chunk][H][NW+2] row-major E_df, zero guards
    // small frames, batches of several chunks: the frame kernel of chunk c + 1 runs on a side
    // stream under the window kernel of chunk c, into a second E_df scratch set
    bool ovl = false;
    uint32_t* Edfs2 = nullptr;
    cudaStream_t ovl_st = nullptr;
    cudaEvent_t ovl_fork = nullptr, ovl_join = nullptr, ovl_frame[2] = {nullptr, nullptr};
    uint32_t* dummy = nullptr; // streaming path: [chunk][32] sink of the lanes beyond W
    unsigned long long* colmask = nullptr;
    int* err = nullptr;
    int* h_err = nullptr;   // pinned
    float* lut = nullptr;
    int K_lut, K_sat;
    float c_exp;
    HostPath hp;
    ProfPool prof;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && dev != prev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

size_t edt_smem_bytes(int W, int NS, int SEGW, int K_lut, bool d2) {
    size_t b = 8ull * W + 4ull * ((K_lut + 3) & ~3) + 2ull * 2 * 32 * NS + 4ull * 32 * 9 * NS;
    if (d2) b += 4ull * 32 * 9 * NS;
    b += (size_t)NS * SEGW * 32;
    return b;
}

// fp32 value of Eq. (1) rounded from fp64, and the first D2 at which it is exactly 1.0f
// Value stored for integer D2 (fp64 arithmetic, then rounded to the output type): the
// transfer of d = sqrt(D2) (Eq. (1) or a §IV-D ablation), 8-bit coded if out_u8.
double transfer_f64(int transfer, double d2, double alpha, double bound) {
    const double d = std::sqrt(d2);
    switch (transfer) {
        case IEDS_TRANSFER_INVEXP: return 1.0 - std::exp(-d / alpha);
        case IEDS_TRANSFER_LINEAR: return d;
        case IEDS_TRANSFER_BOUNDED: return std::min(d, bound);
        default: return std::log(d + 1.0);
    }
}

float table_value(const ieds_config& c, double d2) {
    const double v = transfer_f64(c.transfer, d2, c.alpha, c.bound);
    if (c.out_format == IEDS_OUT_U8) return (float)std::min(255.0, std::max(0.0, std::floor(255.0 * v + 0.5)));
    if (c.out_format == IEDS_OUT_F16) return __half2float(__double2half(v));   // RN-even from fp64
    return (float)v;
}

// value of the limit D2 -> inf (saturation; also the value of an empty frame), or +inf
float limit_value(const ieds_config& c) {
    switch (c.transfer) {
        case IEDS_TRANSFER_INVEXP: return c.out_format == IEDS_OUT_U8 ? 255.0f : 1.0f;
        case IEDS_TRANSFER_BOUNDED:
            return c.out_format == IEDS_OUT_F16 ? __half2float(__double2half(c.bound)) : (float)c.bound;
        default: return INFINITY;
    }
}

// first integer D2 whose stored value equals the limit (values are monotone in D2), or 2^40
int64_t saturation_index(const ieds_config& c) {
    const float lim = limit_value(c);
    if (std::isinf(lim)) return 1ll << 40;
    int64_t lo = 0, hi = 1;
    while (table_value(c, (double)hi) != lim) {
        hi *= 2;
        if (hi > (1ll << 40)) return hi;
    }
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (table_value(c, (double)mid) == lim) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

int cuda_fail(cudaError_t e) { return e == cudaErrorMemoryAllocation ? IEDS_ENOMEM : IEDS_ECUDA; }

void free_host_path(HostPath& hp) {
    for (int i = 0; i < 2; ++i) {
        if (hp.st[i]) cudaStreamDestroy(hp.st[i]);
        if (hp.done[i]) cudaEventDestroy(hp.done[i]);
        if (hp.kdone[i]) cudaEventDestroy(hp.kdone[i]);
        cudaFree(hp.d_xy[i]);
        cudaFree(hp.d_off[i]);
        cudaFree(hp.d_S[i]);
        cudaFreeHost(hp.h_off[i]);
    }
    hp = HostPath{};
}

// returns the event pair to record around the next launch of `kind`, or nulls
void prof_pair(ieds_handle* h, int kind, cudaEvent_t* a, cudaEvent_t* b) {
    *a = *b = nullptr;
    ProfPool& p = h->prof;
    if (!p.on) return;
    if (p.used * 2 + 2 > p.ev.size()) {
        cudaEvent_t e0, e1;
        if (cudaEventCreate(&e0) != cudaSuccess) return;
        if (cudaEventCreate(&e1) != cudaSuccess) { cudaEventDestroy(e0); return; }
        p.ev.push_back(e0);
        p.ev.push_back(e1);
        p.kind.push_back(kind);
    }
    p.kind[p.used] = kind;
    *a = p.ev[2 * p.used];
    *b = p.ev[2 * p.used + 1];
    ++p.used;
}

// window sizes the branch-free kernel is instantiated for (c is rounded up: any C >= c is exact)
constexpr int kWinSizes[] = {4, 6, 8, 10, 12, 14, 16, 19, 22, 25, 28, 31, 34, 37, 40};

int window_size_for(int c) {
    for (int v : kWinSizes)
        if (v >= c) return v;
    return 0;
}


// Sensor-width instantiations (window_kernel.cuh, WIDTH): the row stride is a compile-time
// constant, so every store of a rotation is STG [base + immediate].  The paper's HD camera is
// 1280 pixels wide (Prophesee Gen4); its three saturation windows: Eq. (1) fp32 (C = 19),
// 8-bit (C = 8) and fp16 (C = 10) at d_sat = 6.  Every other width / window runs the generic kernel.
// (A packed 346-wide instantiation for the DAVIS camera, with predicated stores for the
// ragged last strip measured slower: C2 5.90 vs 6.33 M surfaces/s.)
constexpr int kSensorWidth = 1280;
template <int C>
constexpr bool kSensorInst = C == 8 || C == 10 || C == 19;
template <bool PK>
constexpr int kSensorW = kSensorWidth;

template <int C, bool PK>
void launch_window_pk(dim3 grid, cudaStream_t st, const ieds::WinParams& wp, int fmt) {
    const size_t smem = ieds::window_smem_bytes(std::min(wp.H, wp.RB), C, PK);
    if constexpr (!PK && kSensorInst<C>) {
        constexpr int SW = kSensorW<PK>;
        if (wp.W == SW) {
            if (fmt == IEDS_OUT_U8)
                ieds::window_kernel<C, uint8_t, PK, SW><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
            else if (fmt == IEDS_OUT_F16)
                ieds::window_kernel<C, uint16_t, PK, SW><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
            else
                ieds::window_kernel<C, float, PK, SW><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
            return;
        }
    }
    if (fmt == IEDS_OUT_U8) ieds::window_kernel<C, uint8_t, PK><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
    else if (fmt == IEDS_OUT_F16) ieds::window_kernel<C, uint16_t, PK><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
    else ieds::window_kernel<C, float, PK><<<grid, ieds::kWinWarps * 32, smem, st>>>(wp);
}

// packed CTAs (see window_kernel.cuh) exist for the one-word-per-side sizes C <= 31
template <int C>
void launch_window_t(dim3 grid, cudaStream_t st, const ieds::WinParams& wp, int fmt, bool packed) {
    if constexpr (C <= 31) {
        if (packed) return launch_window_pk<C, true>(grid, st, wp, fmt);
    }
    launch_window_pk<C, false>(grid, st, wp, fmt);
}

template <int C, bool PK>
cudaError_t window_attr_pk(int H) {
    const size_t smem = ieds::window_smem_bytes(H, C, PK);
    if constexpr (!PK && kSensorInst<C>) {
        constexpr int SW = kSensorW<PK>;
        cudaError_t e = cudaFuncSetAttribute(ieds::window_kernel<C, float, PK, SW>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ieds::window_kernel<C, uint8_t, PK, SW>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ieds::window_kernel<C, uint16_t, PK, SW>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaFuncSetAttribute(ieds::window_kernel<C, float, PK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ieds::window_kernel<C, uint8_t, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ieds::window_kernel<C, uint16_t, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
    return e;
}

template <int C>
cudaError_t window_attr_t(int H, bool packed) {
    if constexpr (C <= 31) {
        if (packed) return window_attr_pk<C, true>(H);
    }
    return window_attr_pk<C, false>(H);
}

cudaError_t window_attrs(int H, bool packed) {
    cudaError_t e = cudaSuccess;
#define IEDS_WIN_ATTR(c) if (e == cudaSuccess) e = window_attr_t<c>(H, packed);
    IEDS_WIN_ATTR(4) IEDS_WIN_ATTR(6) IEDS_WIN_ATTR(8) IEDS_WIN_ATTR(10) IEDS_WIN_ATTR(12) IEDS_WIN_ATTR(14)
    IEDS_WIN_ATTR(16) IEDS_WIN_ATTR(19) IEDS_WIN_ATTR(22) IEDS_WIN_ATTR(25) IEDS_WIN_ATTR(28) IEDS_WIN_ATTR(31)
    IEDS_WIN_ATTR(34) IEDS_WIN_ATTR(37) IEDS_WIN_ATTR(40)
#undef IEDS_WIN_ATTR
    return e;
}

void launch_window(int C, dim3 grid, cudaStream_t st, const ieds::WinParams& wp, int u8, bool packed) {
    switch (C) {
        case 4: launch_window_t<4>(grid, st, wp, u8, packed); break;
        case 6: launch_window_t<6>(grid, st, wp, u8, packed); break;
        case 8: launch_window_t<8>(grid, st, wp, u8, packed); break;
        case 10: launch_window_t<10>(grid, st, wp, u8, packed); break;
        case 12: launch_window_t<12>(grid, st, wp, u8, packed); break;
        case 14: launch_window_t<14>(grid, st, wp, u8, packed); break;
        case 16: launch_window_t<16>(grid, st, wp, u8, packed); break;
        case 19: launch_window_t<19>(grid, st, wp, u8, packed); break;
        case 22: launch_window_t<22>(grid, st, wp, u8, packed); break;
        case 25: launch_window_t<25>(grid, st, wp, u8, packed); break;
        case 28: launch_window_t<28>(grid, st, wp, u8, packed); break;
        case 31: launch_window_t<31>(grid, st, wp, u8, packed); break;
        case 34: launch_window_t<34>(grid, st, wp, u8, packed); break;
        case 37: launch_window_t<37>(grid, st, wp, u8, packed); break;
        default: launch_window_t<40>(grid, st, wp, u8, packed); break;
    }
}

size_t out_elem_bytes(const ieds_handle* h) {
    return h->cfg.out_format == IEDS_OUT_U8 ? 1 : h->cfg.out_format == IEDS_OUT_F16 ? 2 : 4;
}

// parts (surface path only): 1 = the frame kernel, 2 = the window kernel, 3 = both; edfs = the
// E_df scratch to use (null: the handle's first one)
int launch_chunk(ieds_handle* h, const uint32_t* xy, const int64_t* offsets, int64_t n_events, int nb,
                 void* S, uint32_t* E, uint32_t* Ed, uint32_t* Edf, uint32_t* D2, cudaStream_t st,
                 uint32_t* edfs = nullptr, int parts = 3) {
    ieds::FrameParams fp;
    fp.xy = xy;
    fp.offsets = offsets;
    fp.n_events = n_events;
    fp.W = h->cfg.width;
    fp.H = h->cfg.height;
    fp.NW = h->NW;
    fp.NWP = h->NWP;
    fp.NR = h->NR;
    // Small batches (latency mode, row f2): spread each window's frame over more row bands so
    // that about two waves of CTAs run; bulk batches keep the create-time banding.
    int band_rows = h->band_rows, nbands = h->nbands;
    if (nb < h->nsm && h->cfg.height > 64) {
        const int want = std::min((2 * h->nsm + nb - 1) / nb, (h->cfg.height + 31) / 32);
        const int br = std::min(h->band_rows, ((h->cfg.height + want - 1) / want + 31) / 32 * 32);
        if (br < band_rows) {
            band_rows = br;
            nbands = (h->cfg.height + br - 1) / br;
        }
    }
    fp.band_rows = band_rows;
    fp.nbands = nbands;
    const size_t smem_frame = 4ull * ((4 + (size_t)(band_rows + 6) * h->NWP + 3) & ~3ull) +
                              8ull * std::max(h->cfg.width, h->NWP);
    fp.n_d = h->cfg.n_d;
    fp.n_f = h->cfg.n_f;
    fp.vec_ok = ((reinterpret_cast<uintptr_t>(xy) & 15u) == 0) ? 1 : 0;
    fp.nb = nb;
    // one CTA per SM (large frames): the CTA of window b + nsm starts about a window later.  A
    // wave's prefetches are capped at half the L2 (the first l2 / (2 nsm) bytes of each window):
    // C3 windows (300 KB) are staged whole, C5's 1.2 MB ones partly -- whole ones thrashed the L2
    // (C5 649 k -> 630 k surfaces/s) while C3 gained (frame kernel 0.146 -> 0.134 ms).
    fp.prefetch_ahead = (nbands == 1 && smem_frame > (size_t)kMaxSmem / 2) ? h->nsm : 0;
    fp.prefetch_max = (int64_t)h->l2_bytes / (2 * h->nsm) & ~15ll;
    if (const char* ev = std::getenv("IEDS_FRAME_PREFETCH")) fp.prefetch_ahead = std::atoi(ev) ? fp.prefetch_ahead : 0;
    fp.T = h->T;
    fp.colmask = h->colmask;
    fp.E_out = E;
    fp.Ed_out = Ed;
    fp.Edf_out = Edf;
    fp.Edf_scratch = nullptr;
    fp.err = h->err;
    const bool stream_path = h->streaming && D2 == nullptr;
    if (stream_path) {
        fp.T = nullptr;
        fp.colmask = nullptr;
        fp.Edf_scratch = edfs ? edfs : h->Edfs;
    } else {
        parts = 3;
    }
    cudaEvent_t pa = nullptr, pb = nullptr;
    if (parts & 1) {
    prof_pair(h, 0, &pa, &pb);
    if (pa) cudaEventRecord(pa, st);
    if (!stream_path && nbands > 1 &&   // bands OR their word rows into the column bitmap
        cudaMemsetAsync(h->colmask, 0, sizeof(unsigned long long) * (size_t)nb * h->cfg.width, st) != cudaSuccess)
        return IEDS_ECUDA;
    // Small frames: small CTAs, several per SM, so the scatter and walk phases of different
    // windows overlap and the walk's row bands stay long (346x260, C2: the frame kernel takes
    // 0.053 / 0.038 / 0.032 / 0.030 ms per 1184 windows at 1024 / 512 / 256 / 128 threads).
    // Large frames (one CTA per SM by shared memory) keep 1024 threads (1280x720: 0.145 /
    // 0.143 / 0.151 ms at 1024 / 768 / 512).  The walk needs a thread per word column.
    const size_t fwords = (size_t)band_rows * h->NWP;
    int fthreads = fwords <= 4096 ? 128 : fwords <= 16384 ? 256 : kFrameThreads;
    if (const char* ev = std::getenv("IEDS_FRAME_THREADS")) fthreads = std::max(32, std::min(1024, std::atoi(ev)));
    fthreads = std::max(fthreads, (h->NW + 31) / 32 * 32);
    ieds::frame_kernel<<<dim3(nb, nbands), fthreads, smem_frame, st>>>(fp);
    if (pb) cudaEventRecord(pb, st);
    }   // parts & 1
    if (!(parts & 2)) return cudaGetLastError() == cudaSuccess ? IEDS_OK : IEDS_ECUDA;

    if (stream_path) {
        ieds::WinParams wp;
        wp.Edf = edfs ? edfs : h->Edfs;
        wp.S = S;
        wp.lut = h->lut;
        wp.W = h->cfg.width;
        wp.H = h->cfg.height;
        wp.NW = h->NW;
        wp.K_sat = h->K_sat;
        wp.dummy = h->dummy;
        wp.one = 1u;
        // small batches: row bands (each warming its register window up over C - 1 rows
        // above it) so that about two waves of CTAs run; bulk batches: one band
        // (packed: the launch's nb * NW strips in CTAs of 8, see window_kernel.cuh)
        const int groups = (h->NW + ieds::kWinWarps - 1) / ieds::kWinWarps;
        const int ctas = h->win_packed ? (nb * h->NW + ieds::kWinWarps - 1) / ieds::kWinWarps : groups * nb;
        int nrb = 1;
        if (ctas < 2 * h->nsm) nrb = std::min((2 * h->nsm + ctas - 1) / ctas, std::max(1, h->cfg.height / 32));
        wp.RB = (h->cfg.height + nrb - 1) / nrb;
        nrb = (h->cfg.height + wp.RB - 1) / wp.RB;
        wp.nb = nb;
        dim3 wgrid = h->win_packed ? dim3(ctas, 1, nrb) : dim3(groups, nb, nrb);
        prof_pair(h, 1, &pa, &pb);
        if (pa) cudaEventRecord(pa, st);
        launch_window(h->c_win, wgrid, st, wp, h->cfg.out_format, h->win_packed);
        if (pb) cudaEventRecord(pb, st);
        cudaError_t e2 = cudaGetLastError();
        return e2 == cudaSuccess ? IEDS_OK : IEDS_ECUDA;
    }

    ieds::EdtParams ep;
    ep.T = h->T;
    ep.colmask = h->colmask;
    ep.W = h->cfg.width;
    ep.H = h->cfg.height;
    ep.NR = h->NR;
    uint32_t* D2e = (h->norm_u8 && !D2) ? h->D2n : D2;   // the normalised 8-bit view needs D2
    ep.NS = D2e ? h->NS_d2 : h->NS;
    ep.SEGW = D2e ? h->SEGW_d2 : h->SEGW;
    ep.S = h->norm_u8 ? nullptr : S;
    ep.D2 = D2e;
    ep.lut = h->lut;
    ep.K_lut = h->K_lut;
    ep.K_sat = h->K_sat;
    ep.c_exp = h->c_exp;
    ep.transfer = h->cfg.transfer;
    ep.out_fmt = h->cfg.out_format;
    ep.bound = (float)h->cfg.bound;
    ep.sat_value = limit_value(h->cfg);
    ep.empty_value = limit_value(h->cfg);
    dim3 grid(h->NR, nb);
    prof_pair(h, 1, &pa, &pb);
    if (pa) cudaEventRecord(pa, st);
    ieds::edt_kernel<<<grid, ep.NS * 32, D2e ? h->smem_edt_d2 : h->smem_edt, st>>>(ep);
    if (pb) cudaEventRecord(pb, st);
    if (h->norm_u8) {   // row f1: q = round(255 v(D2) / v(max D2)) per window
        const int64_t npx = (int64_t)ep.W * ep.H;
        const dim3 ngrid((unsigned)std::min<int64_t>(64, (npx + ieds::kNormThreads - 1) / ieds::kNormThreads), nb);
        if (cudaMemsetAsync(h->wmax, 0, sizeof(uint32_t) * nb, st) != cudaSuccess) return IEDS_ECUDA;
        ieds::d2max_kernel<<<ngrid, ieds::kNormThreads, 0, st>>>(D2e, npx, h->wmax);
        ieds::norm_u8_kernel<<<ngrid, ieds::kNormThreads, 0, st>>>(D2e, npx, h->wmax, h->vtab,
                                                                    static_cast<uint8_t*>(S));
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? IEDS_OK : IEDS_ECUDA;
}

}  // namespace

extern "C" {

const char* ieds_version(void) { return IEDS_VERSION_STR; }

const char* ieds_strerror(int code) {
    switch (code) {
        case IEDS_OK: return "ok";
        case IEDS_EINVAL: return "invalid argument";
        case IEDS_ERANGE: return "event outside the frame";
        case IEDS_ECAPACITY: return "capacity exceeded";
        case IEDS_EORDER: return "window offsets not non-decreasing or out of range";
        case IEDS_ECUDA: return "CUDA error";
        case IEDS_ENOMEM: return "out of memory";
        default: return "unknown error";
    }
}

double ieds_alpha_from_dsat(double d_sat) {
    if (!(d_sat > 0.0) || !std::isfinite(d_sat)) return NAN;
    return d_sat / std::log(255.0);   // -d_sat / ln(1/255), Eq. (2)-(3)
}

int ieds_create(const ieds_config* cfg, ieds_handle** out) {
    if (!out) return IEDS_EINVAL;
    *out = nullptr;
    if (!cfg) return IEDS_EINVAL;
    const int W = cfg->width, H = cfg->height;
    if (W < 1 || W > 4096 || H < 1 || H > 2048) return IEDS_EINVAL;
    if (cfg->n_d < 0 || cfg->n_d > 4 || cfg->n_f < 1 || cfg->n_f > 5) return IEDS_EINVAL;
    if (!(cfg->alpha > 0.0) || !std::isfinite(cfg->alpha)) return IEDS_EINVAL;
    if (cfg->chunk_windows < 0 || (cfg->flags & ~(IEDS_FLAG_EXACT_EDT | IEDS_FLAG_TEST_BANDS))) return IEDS_EINVAL;
    if (cfg->transfer < IEDS_TRANSFER_INVEXP || cfg->transfer > IEDS_TRANSFER_LOG) return IEDS_EINVAL;
    if (cfg->transfer == IEDS_TRANSFER_BOUNDED && !(cfg->bound > 0.0 && std::isfinite(cfg->bound)))
        return IEDS_EINVAL;
    if (cfg->out_format < IEDS_OUT_F32 || cfg->out_format > IEDS_OUT_F16) return IEDS_EINVAL;
    if (cfg->out_format == IEDS_OUT_U8 && cfg->transfer == IEDS_TRANSFER_INVEXP &&
        saturation_index(*cfg) > kLutMax)
        return IEDS_EINVAL;

    ieds_handle* h = new ieds_handle();
    h->cfg = *cfg;
    int dev = cfg->device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
        delete h;
        return IEDS_ECUDA;
    }
    h->dev = dev;
    DeviceGuard g(dev);
    if (!g.ok) {
        delete h;
        return IEDS_ECUDA;
    }
    h->NW = (W + 31) / 32;
    h->NWP = (h->NW + 1) | 1;   // odd, with >= 1 zero pad word per row
    h->NR = (H + 31) / 32;
    auto segments = [&](int target, int& NS, int& SEGW) {
        int ns = (W + target - 1) / target;
        ns = std::max(1, std::min(16, ns));
        const int segw = ((W + ns - 1) / ns + 7) & ~7;
        NS = (W + segw - 1) / segw;
        SEGW = segw;
    };
    segments(kSegTarget, h->NS, h->SEGW);
    segments(kSegTargetD2, h->NS_d2, h->SEGW_d2);

    const double alpha = cfg->alpha;
    int64_t ksat = saturation_index(*cfg);
    if (ksat > (1ll << 31)) ksat = (1ll << 31);
    h->K_sat = (int)std::min<int64_t>(ksat, 0x7FFFFFFF);
    h->K_lut = (int)std::min<int64_t>(ksat, kLutMax);
    h->c_exp = (float)(-1.0 / (alpha * std::log(2.0)));
    {
        int64_t cs = (int64_t)std::ceil(std::sqrt((double)ksat));
        while (cs * cs < ksat) ++cs;
        while (cs > 1 && (cs - 1) * (cs - 1) >= ksat) --cs;
        h->c_sat = (int)std::min<int64_t>(cs, 1 << 20);
    }
    h->c_win = window_size_for(std::max(2, h->c_sat));
    h->norm_u8 = cfg->out_format == IEDS_OUT_U8 && cfg->transfer != IEDS_TRANSFER_INVEXP;
    h->streaming = h->c_win > 0 && h->K_sat <= kLutMax && !(cfg->flags & IEDS_FLAG_EXACT_EDT) && !h->norm_u8 &&
                   ieds::window_smem_bytes(H, std::max(2, h->c_win)) <= (size_t)kMaxSmem;

    // 4 zero words + the band's frame rows (band_rows + 6), then the column bitmap of the exact
    // path.  One band holds the whole frame whenever that fits (1280x720: 129 KB); larger
    // frames are split into the fewest bands of a multiple of 32 rows that fit.
    auto frame_bytes = [&](int br) {
        return 4ull * ((4 + (size_t)(br + 6) * h->NWP + 3) & ~3ull) + 8ull * std::max(W, h->NWP);
    };
    h->band_rows = H;
    h->nbands = 1;
    if (frame_bytes(H) > (size_t)kMaxSmem || (cfg->flags & IEDS_FLAG_TEST_BANDS)) {
        int br = (cfg->flags & IEDS_FLAG_TEST_BANDS) ? 64 : ((H + 31) / 32) * 32;
        while (br > 32 && frame_bytes(br) > (size_t)kMaxSmem) br -= 32;
        const int nb = (H + br - 1) / br;
        h->band_rows = ((H + nb - 1) / nb + 31) / 32 * 32;   // balanced, still a multiple of 32
        h->nbands = (H + h->band_rows - 1) / h->band_rows;
    }
    h->smem_frame = frame_bytes(h->band_rows);
    h->smem_edt = edt_smem_bytes(W, h->NS, h->SEGW, h->K_lut, false);
    h->smem_edt_d2 = edt_smem_bytes(W, h->NS_d2, h->SEGW_d2, h->K_lut, true);
    // the exact EDT keeps 1-byte site offsets per segment (<= 255 columns) and its per-row data
    // in shared memory; without it the handle still serves the streaming path (no sqdist)
    h->exact_ok = h->smem_edt_d2 <= (size_t)kMaxSmem && h->smem_edt <= (size_t)kMaxSmem && h->SEGW <= 255 &&
                  h->SEGW_d2 <= 255;
    if (h->smem_frame > (size_t)kMaxSmem || h->NW > kFrameThreads ||   // the D&F walk: a thread per word column
        (!h->exact_ok && (!h->streaming || (cfg->flags & IEDS_FLAG_EXACT_EDT)))) {
        delete h;
        return IEDS_EINVAL;
    }

    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    h->nsm = nsm;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    h->l2_bytes = l2 > 0 ? l2 : (64 << 20);
    // Default: 8 waves of windows per launch pair (~143 MB of scratch at 1280x720), so a
    // 1000-window batch is one frame launch + one window launch with a single partial tail
    // wave instead of four launch pairs whose last one runs a mostly idle wave.  The host
    // path pipelines copies against kernels at a finer 2-wave grain.
    // Windows per launch pair: as many as a 4 GB scratch budget holds (two E_df sets, the exact
    // path's T and column bitmap), a multiple of nsm in [8 nsm, 128 nsm]; the normalised 8-bit
    // view also needs D2 per window: 2 nsm.  Fewer, longer launches pay: 16,000 C3 windows at
    // 1,184 / 2,368 / 4,736 / 9,472 / 16,000 per launch pair took 1.077 / 1.107 / 1.119 / 1.130 /
    // 1.137 M surfaces/s, C2's 10,000 windows 6.38 / 6.57 / 6.73 / 6.83 M (fewer chunk edges,
    // where the window kernel's last wave and the next frame kernel's first idle SMs).
    {
        const double per_window = 4.0 * (2.0 * (h->NW + 2) * H + (double)h->NR * W) + 8.0 * W + 128.0;
        const int64_t fit = (int64_t)(4.0e9 / per_window) / nsm * nsm;
        h->chunk = (int)std::max<int64_t>(8 * nsm, std::min<int64_t>(128 * nsm, fit));
    }
    if (cfg->chunk_windows > 0) h->chunk = cfg->chunk_windows;
    else if (h->norm_u8) h->chunk = 2 * nsm;
    if (const char* ev = std::getenv("IEDS_CHUNK_WINDOWS"))
        if (cfg->chunk_windows == 0 && std::atoi(ev) > 0) h->chunk = std::atoi(ev);
    h->host_chunk = std::min(h->chunk, 2 * nsm);

    cudaError_t e;
    e = cudaFuncSetAttribute(ieds::frame_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem_frame);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ieds::edt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max(h->smem_edt, h->smem_edt_d2));
    if (h->streaming) {
        // Packed window CTAs when more than 1/8 of the strip slots of per-window CTAs would idle
        // (346-wide frames: 11 strips in 16 slots) and the per-warp staging fits.
        const int groups = (h->NW + ieds::kWinWarps - 1) / ieds::kWinWarps;
        h->win_packed = h->c_win <= 31 && 8 * (groups * ieds::kWinWarps - h->NW) > groups * ieds::kWinWarps &&
                        ieds::window_smem_bytes(H, h->c_win, true) <= (size_t)kMaxSmem;
        if (const char* ev = std::getenv("IEDS_WIN_PACKED"))
            h->win_packed = std::atoi(ev) != 0 && h->c_win <= 31 &&
                            ieds::window_smem_bytes(H, h->c_win, true) <= (size_t)kMaxSmem;
    }
    if (e == cudaSuccess && h->streaming) e = window_attrs(H, h->win_packed);
    if (e == cudaSuccess) e = cudaMalloc(&h->T, sizeof(uint32_t) * (size_t)h->chunk * h->NR * W);
    if (e == cudaSuccess) e = cudaMalloc(&h->Edfs, sizeof(uint32_t) * (size_t)h->chunk * (h->NW + 2) * H);
    if (e == cudaSuccess) e = cudaMemset(h->Edfs, 0, sizeof(uint32_t) * (size_t)h->chunk * (h->NW + 2) * H);
    if (e == cudaSuccess) e = cudaMalloc(&h->dummy, sizeof(uint32_t) * 32 * (size_t)h->chunk);
    // chunk overlap (see ieds_build_batch): C2 6.30 -> 6.41 M surfaces/s, C5 677 -> 682 k
    h->ovl = h->streaming;
    if (const char* ev = std::getenv("IEDS_CHUNK_OVERLAP")) h->ovl = h->streaming && std::atoi(ev) != 0;
    if (e == cudaSuccess && h->ovl) {
        int lo = 0, hi = 0;
        e = cudaMalloc(&h->Edfs2, sizeof(uint32_t) * (size_t)h->chunk * (h->NW + 2) * H);
        if (e == cudaSuccess) e = cudaMemset(h->Edfs2, 0, sizeof(uint32_t) * (size_t)h->chunk * (h->NW + 2) * H);
        if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&h->ovl_st, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ovl_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ovl_join, cudaEventDisableTiming);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i)
            e = cudaEventCreateWithFlags(&h->ovl_frame[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess && h->norm_u8) {
        const size_t nv = (size_t)(W - 1) * (W - 1) + (size_t)(H - 1) * (H - 1) + 1;
        e = cudaMalloc(&h->D2n, sizeof(uint32_t) * (size_t)h->chunk * W * H);
        if (e == cudaSuccess) e = cudaMalloc(&h->wmax, sizeof(uint32_t) * (size_t)h->chunk);
        if (e == cudaSuccess) e = cudaMalloc(&h->vtab, sizeof(double) * nv);
        if (e == cudaSuccess) {
            std::vector<double> v(nv);
            for (size_t i = 0; i < nv; ++i) v[i] = transfer_f64(cfg->transfer, (double)i, cfg->alpha, cfg->bound);
            e = cudaMemcpy(h->vtab, v.data(), sizeof(double) * nv, cudaMemcpyHostToDevice);
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&h->colmask, sizeof(unsigned long long) * (size_t)h->chunk * W);
    if (e == cudaSuccess) e = cudaMalloc(&h->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(h->err, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&h->h_err, sizeof(int));
    // table of Eq. (1) over integer D2 < K_lut, plus one saturated entry (1.0f) at K_lut
    if (e == cudaSuccess) e = cudaMalloc(&h->lut, sizeof(float) * (h->K_lut + 1));
    if (e == cudaSuccess) {
        std::vector<float> lut(h->K_lut + 1);
        for (int i = 0; i < h->K_lut; ++i) lut[i] = table_value(*cfg, (double)i);
        lut[h->K_lut] = limit_value(*cfg);
        e = cudaMemcpy(h->lut, lut.data(), sizeof(float) * lut.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        int rc = cuda_fail(e);
        cudaGetLastError();
        ieds_destroy(h);
        return rc;
    }
    *out = h;
    return IEDS_OK;
}

void ieds_destroy(ieds_handle* h) {
    if (!h) return;
    DeviceGuard g(h->dev);
    cudaDeviceSynchronize();
    free_host_path(h->hp);
    for (cudaEvent_t e : h->prof.ev) cudaEventDestroy(e);
    cudaFree(h->T);
    cudaFree(h->Edfs);
    cudaFree(h->Edfs2);
    if (h->ovl_st) cudaStreamDestroy(h->ovl_st);
    for (cudaEvent_t e : {h->ovl_fork, h->ovl_join, h->ovl_frame[0], h->ovl_frame[1]})
        if (e) cudaEventDestroy(e);
    cudaFree(h->dummy);
    cudaFree(h->D2n);
    for (int i = 0; i < 2; ++i) {
        cudaFree(h->fwl_Ic[i]);
        cudaFree(h->fwl_Iu[i]);
        if (h->fwl_splat[i]) cudaEventDestroy(h->fwl_splat[i]);
        if (h->fwl_zero[i]) cudaEventDestroy(h->fwl_zero[i]);
    }
    if (h->fwl_zs) cudaStreamDestroy(h->fwl_zs);
    cudaFree(h->fwl_part);
    cudaFree(h->wmax);
    cudaFree(h->vtab);
    cudaFree(h->colmask);
    cudaFree(h->err);
    cudaFree(h->lut);
    cudaFreeHost(h->h_err);
    delete h;
}

int ieds_profile_enable(ieds_handle* h, int on) {
    if (!h) return IEDS_EINVAL;
    h->prof.on = on != 0;
    return IEDS_OK;
}

int ieds_profile_read(ieds_handle* h, double* frame_ms, int64_t* frame_launches, double* edt_ms,
                      int64_t* edt_launches) {
    if (!h) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    double ms[2] = {0.0, 0.0};
    int64_t n[2] = {0, 0};
    ProfPool& p = h->prof;
    for (size_t i = 0; i < p.used; ++i) {
        if (cudaEventSynchronize(p.ev[2 * i + 1]) != cudaSuccess) return IEDS_ECUDA;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, p.ev[2 * i], p.ev[2 * i + 1]) != cudaSuccess) return IEDS_ECUDA;
        ms[p.kind[i]] += t;
        n[p.kind[i]] += 1;
    }
    p.used = 0;
    if (frame_ms) *frame_ms = ms[0];
    if (frame_launches) *frame_launches = n[0];
    if (edt_ms) *edt_ms = ms[1];
    if (edt_launches) *edt_launches = n[1];
    return IEDS_OK;
}

int64_t ieds_launches_per_batch(const ieds_handle* h, int32_t num_windows) {
    if (!h || num_windows <= 0) return 0;
    return (h->norm_u8 ? 4ll : 2ll) * ((num_windows + h->chunk - 1) / h->chunk);
}

int ieds_build_batch(ieds_handle* h, const uint32_t* events_xy, const int64_t* window_offsets,
                     int64_t n_events, int32_t num_windows, void* surfaces, uint32_t* edge_bits,
                     uint32_t* denoised_bits, uint32_t* filtered_bits, uint32_t* sqdist, void* stream) {
    if (!h || num_windows < 0 || n_events < 0) return IEDS_EINVAL;
    if (num_windows == 0) return IEDS_OK;
    if (!surfaces || !window_offsets || (n_events > 0 && !events_xy)) return IEDS_EINVAL;
    if ((reinterpret_cast<uintptr_t>(events_xy) & 3u) ||
        (reinterpret_cast<uintptr_t>(surfaces) & (out_elem_bytes(h) - 1)))
        return IEDS_EINVAL;
    if (sqdist && !h->exact_ok) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t plane = (size_t)h->cfg.width * h->cfg.height;
    const size_t bplane = (size_t)h->NW * h->cfg.height;
    const int nch = (num_windows + h->chunk - 1) / h->chunk;
    if (h->ovl && nch >= 2 && !sqdist && !edge_bits && !denoised_bits && !filtered_bits) {
        // frame(0) | window(0) || frame(1) | window(1) || frame(2) | ...: the frame kernel of
        // chunk c + 1 (E_df set (c + 1) & 1, high-priority side stream) starts once window(c - 1),
        // the last reader of that set, is done, and window(c + 1) waits for it
        uint32_t* set[2] = {h->Edfs, h->Edfs2};
        auto part = [&](int c, int parts, cudaStream_t s) {
            const int c0 = c * h->chunk, nb = std::min(h->chunk, num_windows - c0);
            return launch_chunk(h, events_xy, window_offsets + c0, n_events, nb,
                                static_cast<char*>(surfaces) + c0 * plane * out_elem_bytes(h),
                                nullptr, nullptr, nullptr, nullptr, s, set[c & 1], parts);
        };
        int rc = part(0, 1, st);
        for (int c = 0; c < nch && rc == IEDS_OK; ++c) {
            if (c + 1 < nch) {
                if (cudaEventRecord(h->ovl_fork, st) != cudaSuccess ||
                    cudaStreamWaitEvent(h->ovl_st, h->ovl_fork, 0) != cudaSuccess)
                    return IEDS_ECUDA;
                rc = part(c + 1, 1, h->ovl_st);
                if (rc != IEDS_OK) break;
                if (cudaEventRecord(h->ovl_frame[(c + 1) & 1], h->ovl_st) != cudaSuccess) return IEDS_ECUDA;
            }
            if (c > 0 && cudaStreamWaitEvent(st, h->ovl_frame[c & 1], 0) != cudaSuccess) return IEDS_ECUDA;
            rc = part(c, 2, st);
        }
        // join: the side stream's last work is a frame(c + 1) that a window waited for; the
        // explicit join keeps capture into a CUDA graph well formed on error paths too
        if (cudaEventRecord(h->ovl_join, h->ovl_st) != cudaSuccess ||
            cudaStreamWaitEvent(st, h->ovl_join, 0) != cudaSuccess)
            return IEDS_ECUDA;
        return rc;
    }
    for (int c0 = 0; c0 < num_windows; c0 += h->chunk) {
        const int nb = std::min(h->chunk, num_windows - c0);
        int rc = launch_chunk(h, events_xy, window_offsets + c0, n_events, nb,
                              static_cast<char*>(surfaces) + c0 * plane * out_elem_bytes(h),
                              edge_bits ? edge_bits + c0 * bplane : nullptr,
                              denoised_bits ? denoised_bits + c0 * bplane : nullptr,
                              filtered_bits ? filtered_bits + c0 * bplane : nullptr,
                              sqdist ? sqdist + c0 * plane : nullptr, st);
        if (rc != IEDS_OK) return rc;
    }
    return IEDS_OK;
}

int ieds_window_offsets(ieds_handle* h, const int64_t* t_us, int64_t n, int64_t t0_us, int64_t dt_us,
                        int32_t num_windows, int64_t* window_offsets, void* stream) {
    if (!h || n < 0 || dt_us <= 0 || num_windows < 0 || !window_offsets || (n > 0 && !t_us)) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t work = std::max<int64_t>(num_windows + 1, n);
    const int blocks = (int)std::min<int64_t>(8 * h->nsm, std::max<int64_t>(1, (work + 255) / 256));
    ieds::window_offsets_kernel<<<blocks, 256, 0, st>>>(t_us, n, t0_us, dt_us, num_windows, window_offsets, h->err);
    return cudaGetLastError() == cudaSuccess ? IEDS_OK : IEDS_ECUDA;
}

int ieds_window_count(ieds_handle* h, const int64_t* t_us, int64_t n, int64_t dt_us, int64_t* t0_us,
                      int32_t* num_windows, void* stream) {
    if (!h || n < 0 || dt_us <= 0 || !t0_us || !num_windows || (n > 0 && !t_us)) return IEDS_EINVAL;
    *t0_us = 0;
    *num_windows = 0;
    if (n == 0) return IEDS_OK;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int64_t* ends = nullptr;   // pinned: t[0], t[n-1]
    cudaError_t e = cudaMallocHost(&ends, 2 * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMemcpyAsync(ends, t_us, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ends + 1, t_us + (n - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeHost(ends);
        return cuda_fail(e);
    }
    const int64_t t0 = ends[0], t1 = ends[1];
    cudaFreeHost(ends);
    *t0_us = t0;
    if (t1 < t0) return IEDS_EORDER;
    const int64_t K = (t1 - t0) / dt_us + 1;   // R16: windows up to the last event's
    if (K > INT32_MAX) return IEDS_ECAPACITY;
    *num_windows = (int32_t)K;
    return IEDS_OK;
}

int ieds_sync(ieds_handle* h, void* stream) {
    if (!h) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(h->h_err, h->err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->err, 0, sizeof(int), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return IEDS_ECUDA;
    const int f = *h->h_err;
    if (f & ieds::kErrOrder) return IEDS_EORDER;
    if (f & ieds::kErrRange) return IEDS_ERANGE;
    return IEDS_OK;
}

// row f3: splat blocks per window (one partial each) when `chunk` windows share a launch:
// about four CTAs per SM of this device in total
static int fwl_splat_blocks(int chunk, int nsm) { return std::max(1, (4 * nsm) / chunk); }

int ieds_fwl_batch(ieds_handle* h, const uint32_t* events_xy, const int64_t* events_t_us, const int8_t* events_p,
                   const int64_t* window_offsets, int64_t n_events, int32_t num_windows, const float* flow,
                   const int64_t* t_ref_us, int64_t dt_us, double* fwl, double* var_comp, double* var_uncomp,
                   double* comp_image, void* stream) {
    if (!h || num_windows < 0 || n_events < 0 || dt_us <= 0) return IEDS_EINVAL;
    if (num_windows == 0) return IEDS_OK;
    if (!window_offsets || !flow || !t_ref_us || !fwl) return IEDS_EINVAL;
    if (n_events > 0 && (!events_xy || !events_t_us || !events_p)) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    const int W = h->cfg.width, H = h->cfg.height;
    const int64_t npx = (int64_t)W * H;
    const int64_t stride = (npx + 3) & ~3ll;   // 16-byte aligned window images in the scratch
    cudaError_t e = cudaSuccess;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!h->fwl_Ic[0]) {
        h->fwl_chunk = kFwlChunkDefault;
        if (const char* env = std::getenv("IEDS_FWL_CHUNK")) h->fwl_chunk = std::max(1, std::min(64, std::atoi(env)));
        const int kFwlChunk = h->fwl_chunk;
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaMalloc(&h->fwl_Ic[i], sizeof(double) * stride * kFwlChunk);
            if (e == cudaSuccess) e = cudaMalloc(&h->fwl_Iu[i], sizeof(int) * stride * kFwlChunk);
            // zeroed on the caller's stream: a blocking cudaMemset runs on the legacy default
            // stream, which a non-blocking caller stream does not wait for
            if (e == cudaSuccess) e = cudaMemsetAsync(h->fwl_Ic[i], 0, sizeof(double) * stride * kFwlChunk, st);
            if (e == cudaSuccess) e = cudaMemsetAsync(h->fwl_Iu[i], 0, sizeof(int) * stride * kFwlChunk, st);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->fwl_splat[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->fwl_zero[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(h->fwl_zero[i], st);
        }
        if (e == cudaSuccess)
            e = cudaMalloc(&h->fwl_part, sizeof(ieds::FwlPart) * fwl_splat_blocks(kFwlChunk, h->nsm) * kFwlChunk);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->fwl_zs, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            for (int i = 0; i < 2; ++i) {
                cudaFree(h->fwl_Ic[i]);
                cudaFree(h->fwl_Iu[i]);
                h->fwl_Ic[i] = nullptr;
                h->fwl_Iu[i] = nullptr;
            }
            cudaFree(h->fwl_part);
            h->fwl_part = nullptr;
            cudaGetLastError();
            return cuda_fail(e);
        }
    }
    // splat grid: enough blocks per window to fill the GPU several times over
    const int kFwlChunk = h->fwl_chunk;
    const int per_win = fwl_splat_blocks(kFwlChunk, h->nsm);
    for (int c0 = 0; c0 < num_windows; c0 += kFwlChunk) {
        const int nb = std::min(kFwlChunk, num_windows - c0);
        const int set = h->fwl_next;
        h->fwl_next ^= 1;
        ieds::FwlParams fp;
        fp.xy = events_xy;
        fp.t = events_t_us;
        fp.p = events_p;
        fp.offsets = window_offsets + c0;
        fp.n_events = n_events;
        fp.flow = reinterpret_cast<const float2*>(flow) + (size_t)c0 * npx;
        fp.t_ref = t_ref_us + c0;
        fp.dt = dt_us;
        fp.W = W;
        fp.H = H;
        fp.stride = stride;
        fp.Ic = h->fwl_Ic[set];
        fp.Iu = h->fwl_Iu[set];
        fp.err = h->err;
        // this set was re-zeroed on the side stream after its last pass
        cudaError_t ce = cudaStreamWaitEvent(st, h->fwl_zero[set], 0);
        if (ce != cudaSuccess) return IEDS_ECUDA;
        ieds::fwl_splat_kernel<<<dim3(per_win, nb), ieds::kFwlThreads, 0, st>>>(fp, h->fwl_part);
        if (comp_image)
            ce = cudaMemcpy2DAsync(comp_image + (size_t)c0 * npx, sizeof(double) * npx, h->fwl_Ic[set],
                                   sizeof(double) * stride, sizeof(double) * npx, nb, cudaMemcpyDeviceToDevice, st);
        // re-zero the set for its next pass on the side stream, overlapped with the next splat
        if (ce == cudaSuccess) ce = cudaEventRecord(h->fwl_splat[set], st);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(h->fwl_zs, h->fwl_splat[set], 0);
        if (ce == cudaSuccess) ce = cudaMemsetAsync(h->fwl_Ic[set], 0, sizeof(double) * stride * nb, h->fwl_zs);
        if (ce == cudaSuccess) ce = cudaMemsetAsync(h->fwl_Iu[set], 0, sizeof(int) * stride * nb, h->fwl_zs);
        if (ce == cudaSuccess) ce = cudaEventRecord(h->fwl_zero[set], h->fwl_zs);
        if (ce != cudaSuccess) return IEDS_ECUDA;
        ieds::fwl_finalize_kernel<<<nb, ieds::kFwlThreads, 0, st>>>(h->fwl_part, per_win, npx, fwl + c0,
                                                                     var_comp ? var_comp + c0 : nullptr,
                                                                     var_uncomp ? var_uncomp + c0 : nullptr);
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? IEDS_OK : IEDS_ECUDA;
}

int ieds_build_batch_host(ieds_handle* h, const uint32_t* events_xy, const int64_t* window_offsets,
                          int32_t num_windows, void* surfaces) {
    if (!h || num_windows < 0) return IEDS_EINVAL;
    if (num_windows == 0) return IEDS_OK;
    if (!window_offsets || !surfaces) return IEDS_EINVAL;
    for (int32_t b = 0; b < num_windows; ++b)
        if (window_offsets[b + 1] < window_offsets[b] || window_offsets[b] < 0) return IEDS_EORDER;
    if (window_offsets[num_windows] > window_offsets[0] && !events_xy) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    // The internal streams reuse the handle's scratch (E_df / T / colmask): wait for every
    // ieds_build_batch still queued on a caller stream (this entry point blocks anyway).
    if (cudaDeviceSynchronize() != cudaSuccess) return IEDS_ECUDA;
    HostPath& hp = h->hp;
    cudaError_t e = cudaSuccess;
    const size_t plane = (size_t)h->cfg.width * h->cfg.height;
    const int chunk = h->host_chunk;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        if (!hp.st[i]) e = cudaStreamCreateWithFlags(&hp.st[i], cudaStreamNonBlocking);
        if (e == cudaSuccess && !hp.done[i]) e = cudaEventCreateWithFlags(&hp.done[i], cudaEventDisableTiming);
        if (e == cudaSuccess && !hp.kdone[i]) e = cudaEventCreateWithFlags(&hp.kdone[i], cudaEventDisableTiming);
        if (e == cudaSuccess && !hp.d_S[i]) e = cudaMalloc(&hp.d_S[i], sizeof(float) * plane * chunk);   // fits u8
        if (e == cudaSuccess && !hp.d_off[i]) e = cudaMalloc(&hp.d_off[i], sizeof(int64_t) * (chunk + 1));
        if (e == cudaSuccess && !hp.h_off[i]) e = cudaMallocHost(&hp.h_off[i], sizeof(int64_t) * (chunk + 1));
    }
    if (e != cudaSuccess) return cuda_fail(e);
    // The two internal streams alternate chunks; the scratch (T, colmask) is shared, so the
    // kernels of consecutive chunks are ordered through events while copies overlap.
    int rc = IEDS_OK;
    int k = 0;
    for (int c0 = 0; c0 < num_windows; c0 += chunk, k ^= 1) {
        const int nb = std::min(chunk, num_windows - c0);
        const int64_t e0 = window_offsets[c0], e1 = window_offsets[c0 + nb];
        const int64_t nev = e1 - e0;
        cudaStream_t st = hp.st[k];
        // buffer k was last used two chunks ago: wait until its copies/kernels finished
        e = cudaEventSynchronize(hp.done[k]);
        if (e == cudaSuccess && nev > hp.cap_ev[k]) {
            cudaFree(hp.d_xy[k]);
            hp.d_xy[k] = nullptr;
            hp.cap_ev[k] = 0;
            e = cudaMalloc(&hp.d_xy[k], sizeof(uint32_t) * (size_t)std::max<int64_t>(nev, 4));
            if (e == cudaSuccess) hp.cap_ev[k] = nev;
        }
        if (e != cudaSuccess) return cuda_fail(e);
        for (int b = 0; b <= nb; ++b) hp.h_off[k][b] = window_offsets[c0 + b] - e0;
        if (nev > 0)
            e = cudaMemcpyAsync(hp.d_xy[k], events_xy + e0, sizeof(uint32_t) * nev, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hp.d_off[k], hp.h_off[k], sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) {
            // order the kernels after the previous chunk's kernels (shared scratch)
            e = cudaStreamWaitEvent(st, hp.kdone[k ^ 1], 0);
        }
        if (e != cudaSuccess) return cuda_fail(e);
        rc = launch_chunk(h, hp.d_xy[k], hp.d_off[k], nev, nb, hp.d_S[k], nullptr, nullptr, nullptr, nullptr, st);
        if (rc != IEDS_OK) return rc;
        e = cudaEventRecord(hp.kdone[k], st);
        if (e != cudaSuccess) return cuda_fail(e);
        e = cudaMemcpyAsync(static_cast<char*>(surfaces) + (size_t)c0 * plane * out_elem_bytes(h), hp.d_S[k],
                            out_elem_bytes(h) * plane * nb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(hp.done[k], st);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    e = cudaStreamSynchronize(hp.st[0]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(hp.st[1]);
    if (e != cudaSuccess) return IEDS_ECUDA;
    return ieds_sync(h, hp.st[0]);
}

}  // extern "C"

// ---- row f2: streaming ingest (include/ieds.h "streaming ingest") ------------------
// Device buffers hold [open window's events (the carry)][this push's events]; the windowing
// kernel finds the boundaries of the windows this push closes (and checks the order of the
// whole span, carry included); the closed windows go through launch_chunk sub-batch by
// sub-batch on two internal streams, each sub-batch's surfaces copied out while the next one
// computes; the new open window's events are moved to the front of the other buffer.
struct ieds_stream {
    ieds_handle* h = nullptr;
    int64_t dt = 0;
    bool started = false;
    int64_t t0 = 0, k_open = 0, last_t = 0;
    int64_t cap = 0;             // device / pinned capacity in events
    int cur = 0;                 // buffer holding the carry
    int64_t n_carry = 0;
    uint32_t* d_xy[2] = {nullptr, nullptr};
    int64_t* d_t[2] = {nullptr, nullptr};
    int64_t cap_off = 0;
    int64_t* d_off = nullptr;    // [cap_off + 2]
    int* d_err = nullptr;        // the stream's own order flag
    uint32_t* p_xy = nullptr;    // pinned staging [cap]
    int64_t* p_t = nullptr;
    int64_t* p_io = nullptr;     // pinned: {err, carry start}
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t kdone[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    void* d_S[2] = {nullptr, nullptr};   // `sub` windows of surfaces each
    int sub = 0;                         // windows per build / copy-out sub-batch
};

namespace {

void stream_free_buffers(ieds_stream* s) {
    for (int i = 0; i < 2; ++i) {
        cudaFree(s->d_xy[i]);
        cudaFree(s->d_t[i]);
        s->d_xy[i] = nullptr;
        s->d_t[i] = nullptr;
    }
    cudaFreeHost(s->p_xy);
    cudaFreeHost(s->p_t);
    s->p_xy = nullptr;
    s->p_t = nullptr;
    s->cap = 0;
}

// capacity for `need` device events (carry preserved) and `chunk` staged host events
cudaError_t stream_reserve(ieds_stream* s, int64_t need) {
    if (need <= s->cap) return cudaSuccess;
    const int64_t cap = std::max<int64_t>(need, 2 * s->cap);
    uint32_t* xy[2] = {nullptr, nullptr};
    int64_t* t[2] = {nullptr, nullptr};
    uint32_t* pxy = nullptr;
    int64_t* pt = nullptr;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaMalloc(&xy[i], sizeof(uint32_t) * cap);
        if (e == cudaSuccess) e = cudaMalloc(&t[i], sizeof(int64_t) * cap);
    }
    if (e == cudaSuccess) e = cudaMallocHost(&pxy, sizeof(uint32_t) * cap);
    if (e == cudaSuccess) e = cudaMallocHost(&pt, sizeof(int64_t) * cap);
    if (e == cudaSuccess && s->n_carry > 0) {   // keep the open window
        e = cudaMemcpyAsync(xy[0], s->d_xy[s->cur], sizeof(uint32_t) * s->n_carry, cudaMemcpyDeviceToDevice, s->st[0]);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(t[0], s->d_t[s->cur], sizeof(int64_t) * s->n_carry, cudaMemcpyDeviceToDevice, s->st[0]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s->st[0]);
    }
    if (e != cudaSuccess) {
        for (int i = 0; i < 2; ++i) {
            cudaFree(xy[i]);
            cudaFree(t[i]);
        }
        cudaFreeHost(pxy);
        cudaFreeHost(pt);
        return e;
    }
    stream_free_buffers(s);
    for (int i = 0; i < 2; ++i) {
        s->d_xy[i] = xy[i];
        s->d_t[i] = t[i];
    }
    s->p_xy = pxy;
    s->p_t = pt;
    s->cap = cap;
    s->cur = 0;
    return cudaSuccess;
}

// surfaces of windows [0, nw) of the CSR (d_xy, d_off) into host `out`, sub-batches of
// host_chunk windows alternating between the two internal streams (kernels ordered through
// events because the handle's scratch is shared; the copies overlap the next kernels)
int stream_build(ieds_stream* s, const uint32_t* d_xy, const int64_t* d_off, int64_t n_ev, int64_t nw, void* out) {
    ieds_handle* h = s->h;
    const size_t plane = (size_t)h->cfg.width * h->cfg.height * out_elem_bytes(h);
    const int chunk = s->sub;
    cudaError_t e = cudaSuccess;
    int k = 0;
    for (int64_t c0 = 0; c0 < nw; c0 += chunk, k ^= 1) {
        const int nb = (int)std::min<int64_t>(chunk, nw - c0);
        cudaStream_t st = s->st[k];
        e = cudaEventSynchronize(s->done[k]);   // buffer k's previous copy finished
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s->kdone[k ^ 1], 0);
        if (e != cudaSuccess) return cuda_fail(e);
        const int rc = launch_chunk(h, d_xy, d_off + c0, n_ev, nb, s->d_S[k], nullptr, nullptr, nullptr, nullptr, st);
        if (rc != IEDS_OK) return rc;
        e = cudaEventRecord(s->kdone[k], st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(static_cast<char*>(out) + (size_t)c0 * plane, s->d_S[k], plane * nb,
                                cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(s->done[k], st);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    e = cudaStreamSynchronize(s->st[0]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->st[1]);
    return e == cudaSuccess ? IEDS_OK : IEDS_ECUDA;
}

}  // namespace

extern "C" {

int ieds_stream_create(ieds_handle* h, int64_t dt_us, ieds_stream** out) {
    if (!out) return IEDS_EINVAL;
    *out = nullptr;
    if (!h || dt_us <= 0) return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    ieds_stream* s = new ieds_stream();
    s->h = h;
    s->dt = dt_us;
    // a push closes a few windows at a time: sub-batches of <= 32 windows (118 MB of fp32
    // surfaces at 1280x720 per buffer) still overlap each copy-out with the next build
    s->sub = std::min(h->host_chunk, 32);
    const size_t plane = (size_t)h->cfg.width * h->cfg.height * out_elem_bytes(h);
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaStreamCreateWithFlags(&s->st[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->kdone[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->done[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaMalloc(&s->d_S[i], plane * s->sub);
    }
    if (e == cudaSuccess) e = cudaMalloc(&s->d_err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(s->d_err, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&s->p_io, 2 * sizeof(int64_t));
    if (e != cudaSuccess) {
        const int rc = cuda_fail(e);
        cudaGetLastError();
        ieds_stream_destroy(s);
        return rc;
    }
    *out = s;
    return IEDS_OK;
}

void ieds_stream_destroy(ieds_stream* s) {
    if (!s) return;
    DeviceGuard g(s->h->dev);
    for (int i = 0; i < 2; ++i) {
        if (s->st[i]) cudaStreamSynchronize(s->st[i]);
    }
    stream_free_buffers(s);
    for (int i = 0; i < 2; ++i) {
        if (s->st[i]) cudaStreamDestroy(s->st[i]);
        if (s->kdone[i]) cudaEventDestroy(s->kdone[i]);
        if (s->done[i]) cudaEventDestroy(s->done[i]);
        cudaFree(s->d_S[i]);
    }
    cudaFree(s->d_off);
    cudaFree(s->d_err);
    cudaFreeHost(s->p_io);
    delete s;
}

int64_t ieds_stream_closing(const ieds_stream* s, int64_t t_first_us, int64_t t_last_us) {
    if (!s) return 0;
    const int64_t t0 = s->started ? s->t0 : t_first_us;
    if (t_last_us < t0) return 0;
    return std::max<int64_t>(0, (t_last_us - t0) / s->dt - (s->started ? s->k_open : 0));
}

}  // extern "C"

namespace {

// A staged push: the chunk appended after the carry on the device, the boundaries of the windows it
// closes in s->d_off (n_closed of them from offsets[0]), the still-open window from `carry0` on.
// Nothing of the stream's state is changed until stream_commit.
struct StreamIngest {
    int64_t t0 = 0, k_last = 0, n_closed = 0, n_tot = 0, carry0 = 0, last_t = 0;
    int cur = 0;
};

int stream_ingest(ieds_stream* s, const int64_t* t_us, const uint32_t* events_xy, int64_t n, int32_t max_out,
                  StreamIngest* ing) {
    ieds_handle* h = s->h;
    // host-checkable order: the chunk continues the stream and its ends are ordered (the
    // device kernel checks every adjacent pair below, before anything is built)
    if ((s->started && t_us[0] < s->last_t) || t_us[n - 1] < t_us[0]) return IEDS_EORDER;
    const int64_t t0 = s->started ? s->t0 : t_us[0];
    const int64_t k_open = s->started ? s->k_open : 0;
    const int64_t k_last = (t_us[n - 1] - t0) / s->dt;
    const int64_t n_closed = k_last - k_open;
    if (n_closed > max_out) return IEDS_ECAPACITY;
    if (cudaDeviceSynchronize() != cudaSuccess) return IEDS_ECUDA;   // scratch shared with queued calls
    cudaError_t e = stream_reserve(s, s->n_carry + n);
    if (e == cudaSuccess && n_closed + 2 > s->cap_off) {
        const int64_t c = std::max<int64_t>(n_closed + 2, 2 * s->cap_off + 64);   // geometric growth
        cudaFree(s->d_off);
        s->d_off = nullptr;
        s->cap_off = 0;
        e = cudaMalloc(&s->d_off, sizeof(int64_t) * c);
        if (e == cudaSuccess) s->cap_off = c;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    const int cur = s->cur;
    const int64_t n_tot = s->n_carry + n;
    cudaStream_t st = s->st[0];
    // the chunk is appended after the carry: straight from the caller's memory when it is
    // page-locked, else through the pinned staging buffers (a host copy)
    auto pinned = [](const void* p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    const int64_t* src_t = t_us;
    const uint32_t* src_xy = events_xy;
    if (!pinned(t_us)) {
        std::memcpy(s->p_t, t_us, sizeof(int64_t) * n);
        src_t = s->p_t;
    }
    if (!pinned(events_xy)) {
        std::memcpy(s->p_xy, events_xy, sizeof(uint32_t) * n);
        src_xy = s->p_xy;
    }
    e = cudaMemcpyAsync(s->d_t[cur] + s->n_carry, src_t, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->d_xy[cur] + s->n_carry, src_xy, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->d_err, 0, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e);
    // boundaries of windows k_open .. k_last over the whole span (offsets[n_closed] = the start
    // of the still-open window k_last) + the order check of every adjacent pair
    const int64_t work = std::max<int64_t>(n_closed + 2, n_tot);
    const int blocks = (int)std::min<int64_t>(8 * h->nsm, std::max<int64_t>(1, (work + 255) / 256));
    ieds::window_offsets_kernel<<<blocks, 256, 0, st>>>(s->d_t[cur], n_tot, t0 + k_open * s->dt, s->dt, n_closed + 1,
                                                         s->d_off, s->d_err);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&s->p_io[0], s->d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&s->p_io[1], s->d_off + n_closed, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return IEDS_ECUDA;
    if (*reinterpret_cast<int*>(&s->p_io[0]) & ieds::kErrOrder) return IEDS_EORDER;   // rejected, stream unchanged
    ing->t0 = t0;
    ing->k_last = k_last;
    ing->n_closed = n_closed;
    ing->n_tot = n_tot;
    ing->carry0 = s->p_io[1];
    ing->last_t = t_us[n - 1];
    ing->cur = cur;
    // the first sub-batch of the closed windows waits for the offsets
    e = cudaEventRecord(s->kdone[1], st);
    return e == cudaSuccess ? IEDS_OK : cuda_fail(e);
}

// the open window k_last (events [carry0, n_tot)) moves to the front of the other buffer, and the
// stream's state advances (enqueued on st[0]; the caller synchronises)
int stream_commit(ieds_stream* s, const StreamIngest& ing) {
    cudaStream_t st = s->st[0];
    const int cur = ing.cur, nxt = cur ^ 1;
    const int64_t nc = ing.n_tot - ing.carry0;
    cudaError_t e =
        cudaMemcpyAsync(s->d_xy[nxt], s->d_xy[cur] + ing.carry0, sizeof(uint32_t) * nc, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->d_t[nxt], s->d_t[cur] + ing.carry0, sizeof(int64_t) * nc, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e);
    s->cur = nxt;
    s->n_carry = nc;
    s->started = true;
    s->t0 = ing.t0;
    s->k_open = ing.k_last;
    s->last_t = ing.last_t;
    return IEDS_OK;
}

// the open window as a one-window CSR in s->d_off (flush)
int stream_last_window(ieds_stream* s) {
    if (s->cap_off < 2) {
        cudaFree(s->d_off);
        s->d_off = nullptr;
        s->cap_off = 0;
        if (cudaMalloc(&s->d_off, sizeof(int64_t) * 64) != cudaSuccess) return IEDS_ENOMEM;
        s->cap_off = 64;
    }
    s->p_io[0] = 0;
    s->p_io[1] = s->n_carry;
    cudaStream_t st = s->st[0];
    cudaError_t e = cudaMemcpyAsync(s->d_off, s->p_io, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(s->kdone[1], st);
    return e == cudaSuccess ? IEDS_OK : cuda_fail(e);
}

}  // namespace

extern "C" {

int ieds_stream_push(ieds_stream* s, const int64_t* t_us, const uint32_t* events_xy, int64_t n, void* surfaces,
                     int32_t max_out, int32_t* num_out) {
    if (!s || !num_out || n < 0 || max_out < 0) return IEDS_EINVAL;
    *num_out = 0;
    if (n == 0) return IEDS_OK;
    if (!t_us || !events_xy) return IEDS_EINVAL;
    ieds_handle* h = s->h;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    if (!surfaces && (t_us[n - 1] - (s->started ? s->t0 : t_us[0])) / s->dt > (s->started ? s->k_open : 0))
        return IEDS_EINVAL;   // windows would close with nowhere to write them
    StreamIngest ing;
    int rc = stream_ingest(s, t_us, events_xy, n, max_out, &ing);
    if (rc != IEDS_OK) return rc;
    if (ing.n_closed > 0) {
        rc = stream_build(s, s->d_xy[ing.cur], s->d_off, ing.n_tot, ing.n_closed, surfaces);
        if (rc != IEDS_OK) return rc;
    }
    rc = stream_commit(s, ing);
    if (rc != IEDS_OK) return rc;
    *num_out = (int32_t)ing.n_closed;
    return ieds_sync(h, s->st[0]);   // waits for the carry move; latched IEDS_ERANGE of the built windows
}

int ieds_stream_flush(ieds_stream* s, void* surfaces, int32_t max_out, int32_t* num_out) {
    if (!s || !num_out || max_out < 0) return IEDS_EINVAL;
    *num_out = 0;
    if (!s->started || s->n_carry == 0) {
        s->started = false;
        return IEDS_OK;
    }
    if (max_out < 1) return IEDS_ECAPACITY;
    if (!surfaces) return IEDS_EINVAL;
    ieds_handle* h = s->h;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    if (cudaDeviceSynchronize() != cudaSuccess) return IEDS_ECUDA;
    int rc = stream_last_window(s);
    if (rc == IEDS_OK) rc = stream_build(s, s->d_xy[s->cur], s->d_off, s->n_carry, 1, surfaces);
    if (rc != IEDS_OK) return rc;
    s->started = false;
    s->n_carry = 0;
    s->k_open = 0;
    *num_out = 1;
    return ieds_sync(h, s->st[0]);
}

}  // extern "C"

// ---- the Fig. 1 pipeline (include/ieds.h "The Fig. 1 pipeline") -----------------
namespace ieds {
int flow_dims(const ieds_flow_handle* h, int* width, int* height, int* device);   // flow.cu
}

struct ieds_pipeline {
    ieds_stream* s = nullptr;                      // owned: windowing, carry, build buffers d_S
    ieds_flow_handle* f = nullptr;                 // borrowed
    uint32_t* d_Ed[2] = {nullptr, nullptr};        // denoised edge bits of a sub-batch [sub][H][NW]
    float* d_flow[2] = {nullptr, nullptr};         // one window's flow [H][W][2], double-buffered
    uint8_t* d_valid[2] = {nullptr, nullptr};      // [H][W]
    cudaStream_t fs = nullptr, cs = nullptr;       // flow stream, copy-out stream
    cudaEvent_t built[2] = {nullptr, nullptr};     // sub-batch buffer k built (and its surfaces copied)
    cudaEvent_t used[2] = {nullptr, nullptr};      // the flow steps are done with buffer k
    cudaEvent_t stepped[2] = {nullptr, nullptr};   // flow buffer q computed
    cudaEvent_t copied[2] = {nullptr, nullptr};    // flow buffer q copied out
};

namespace {

// closed windows [0, nw) of (d_xy, d_off): per sub-batch, surfaces + E_d on the build stream k,
// then the flow of each window in order on fs, each window's flow copied out on cs while the next
// one is computed
int pipeline_build(ieds_pipeline* p, const uint32_t* d_xy, const int64_t* d_off, int64_t n_ev, int64_t nw,
                   float* flow_out, uint8_t* valid_out, void* surf_out) {
    ieds_stream* s = p->s;
    ieds_handle* h = s->h;
    const size_t plane = (size_t)h->cfg.width * h->cfg.height;
    const size_t bplane = (size_t)h->NW * h->cfg.height;
    cudaError_t e = cudaSuccess;
    int k = 0, q = 0;
    for (int64_t c0 = 0; c0 < nw; c0 += s->sub, k ^= 1) {
        const int nb = (int)std::min<int64_t>(s->sub, nw - c0);
        cudaStream_t st = s->st[k];
        e = cudaStreamWaitEvent(st, p->used[k], 0);                    // buffer k free
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s->kdone[k ^ 1], 0);   // shared scratch
        if (e != cudaSuccess) return cuda_fail(e);
        const int rc = launch_chunk(h, d_xy, d_off + c0, n_ev, nb, s->d_S[k], nullptr, p->d_Ed[k], nullptr, nullptr, st);
        if (rc != IEDS_OK) return rc;
        e = cudaEventRecord(s->kdone[k], st);
        if (e == cudaSuccess && surf_out)
            e = cudaMemcpyAsync(static_cast<float*>(surf_out) + c0 * plane, s->d_S[k], sizeof(float) * plane * nb,
                                cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(p->built[k], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->fs, p->built[k], 0);
        if (e != cudaSuccess) return cuda_fail(e);
        for (int i = 0; i < nb; ++i, q ^= 1) {
            e = cudaStreamWaitEvent(p->fs, p->copied[q], 0);           // flow buffer q copied out
            if (e != cudaSuccess) return cuda_fail(e);
            const int rc2 = ieds_flow_step(p->f, static_cast<const float*>(s->d_S[k]) + i * plane,
                                           p->d_Ed[k] + i * bplane, p->d_flow[q], p->d_valid[q], p->fs);
            if (rc2 != IEDS_OK) return rc2;
            e = cudaEventRecord(p->stepped[q], p->fs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(p->cs, p->stepped[q], 0);
            if (e == cudaSuccess && flow_out)
                e = cudaMemcpyAsync(flow_out + (c0 + i) * plane * 2, p->d_flow[q], sizeof(float) * 2 * plane,
                                    cudaMemcpyDeviceToHost, p->cs);
            if (e == cudaSuccess && valid_out)
                e = cudaMemcpyAsync(valid_out + (c0 + i) * plane, p->d_valid[q], plane, cudaMemcpyDeviceToHost, p->cs);
            if (e == cudaSuccess) e = cudaEventRecord(p->copied[q], p->cs);
            if (e != cudaSuccess) return cuda_fail(e);
        }
        e = cudaEventRecord(p->used[k], p->fs);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    for (cudaStream_t x : {s->st[0], s->st[1], p->fs, p->cs}) {
        e = cudaStreamSynchronize(x);
        if (e != cudaSuccess) return IEDS_ECUDA;
    }
    return IEDS_OK;
}

}  // namespace

extern "C" {

int ieds_pipeline_create(ieds_handle* h, ieds_flow_handle* f, int64_t dt_us, ieds_pipeline** out) {
    if (!out) return IEDS_EINVAL;
    *out = nullptr;
    if (!h || !f || dt_us <= 0 || h->cfg.out_format != IEDS_OUT_F32) return IEDS_EINVAL;
    int fw = 0, fh = 0, fd = -1;
    if (ieds::flow_dims(f, &fw, &fh, &fd) != IEDS_OK || fw != h->cfg.width || fh != h->cfg.height || fd != h->dev)
        return IEDS_EINVAL;
    DeviceGuard g(h->dev);
    if (!g.ok) return IEDS_ECUDA;
    ieds_pipeline* p = new ieds_pipeline();
    p->f = f;
    int rc = ieds_stream_create(h, dt_us, &p->s);
    if (rc != IEDS_OK) {
        delete p;
        return rc;
    }
    const size_t plane = (size_t)h->cfg.width * h->cfg.height;
    const size_t bplane = (size_t)h->NW * h->cfg.height;
    cudaError_t e = cudaStreamCreateWithFlags(&p->fs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaMalloc(&p->d_Ed[i], sizeof(uint32_t) * bplane * p->s->sub);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_flow[i], sizeof(float) * 2 * plane);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_valid[i], plane);
        for (cudaEvent_t* ev : {&p->built[i], &p->used[i], &p->stepped[i], &p->copied[i]})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        rc = cuda_fail(e);
        cudaGetLastError();
        ieds_pipeline_destroy(p);
        return rc;
    }
    *out = p;
    return IEDS_OK;
}

void ieds_pipeline_destroy(ieds_pipeline* p) {
    if (!p) return;
    if (p->s) {
        DeviceGuard g(p->s->h->dev);
        for (cudaStream_t x : {p->fs, p->cs})
            if (x) cudaStreamSynchronize(x);
        for (int i = 0; i < 2; ++i) {
            cudaFree(p->d_Ed[i]);
            cudaFree(p->d_flow[i]);
            cudaFree(p->d_valid[i]);
            for (cudaEvent_t ev : {p->built[i], p->used[i], p->stepped[i], p->copied[i]})
                if (ev) cudaEventDestroy(ev);
        }
        for (cudaStream_t x : {p->fs, p->cs})
            if (x) cudaStreamDestroy(x);
        ieds_stream_destroy(p->s);
    }
    delete p;
}

int64_t ieds_pipeline_closing(const ieds_pipeline* p, int64_t t_first_us, int64_t t_last_us) {
    return p ? ieds_stream_closing(p->s, t_first_us, t_last_us) : 0;
}

int ieds_pipeline_push(ieds_pipeline* p, const int64_t* t_us, const uint32_t* events_xy, int64_t n, float* flow,
                       uint8_t* valid, void* surfaces, int32_t max_out, int32_t* num_out) {
    if (!p || !num_out || n < 0 || max_out < 0) return IEDS_EINVAL;
    *num_out = 0;
    if (n == 0) return IEDS_OK;
    if (!t_us || !events_xy) return IEDS_EINVAL;
    ieds_stream* s = p->s;
    DeviceGuard g(s->h->dev);
    if (!g.ok) return IEDS_ECUDA;
    StreamIngest ing;
    int rc = stream_ingest(s, t_us, events_xy, n, max_out, &ing);
    if (rc != IEDS_OK) return rc;
    if (ing.n_closed > 0) {
        rc = pipeline_build(p, s->d_xy[ing.cur], s->d_off, ing.n_tot, ing.n_closed, flow, valid, surfaces);
        if (rc != IEDS_OK) return rc;
    }
    rc = stream_commit(s, ing);
    if (rc != IEDS_OK) return rc;
    *num_out = (int32_t)ing.n_closed;
    return ieds_sync(s->h, s->st[0]);
}

int ieds_pipeline_flush(ieds_pipeline* p, float* flow, uint8_t* valid, void* surfaces, int32_t max_out,
                        int32_t* num_out) {
    if (!p || !num_out || max_out < 0) return IEDS_EINVAL;
    *num_out = 0;
    ieds_stream* s = p->s;
    int rc = IEDS_OK;
    if (s->started && s->n_carry > 0) {
        if (max_out < 1) return IEDS_ECAPACITY;
        DeviceGuard g(s->h->dev);
        if (!g.ok) return IEDS_ECUDA;
        if (cudaDeviceSynchronize() != cudaSuccess) return IEDS_ECUDA;
        rc = stream_last_window(s);
        if (rc == IEDS_OK) rc = pipeline_build(p, s->d_xy[s->cur], s->d_off, s->n_carry, 1, flow, valid, surfaces);
        if (rc != IEDS_OK) return rc;
        *num_out = 1;
        rc = ieds_sync(s->h, s->st[0]);
    }
    s->started = false;
    s->n_carry = 0;
    s->k_open = 0;
    const int rf = ieds_flow_reset(p->f);
    return rc != IEDS_OK ? rc : rf;
}

}  // extern "C"
