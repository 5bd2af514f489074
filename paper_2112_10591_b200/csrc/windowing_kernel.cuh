// windowing_kernel.cuh -- row f2: CSR window offsets of a time-ordered event stream.
//
// §III-A: events are accumulated over windows of length Delta T.  Window k holds
// the events with floor((t - t0) / dt) == k, t in [t0 + k dt, t0 + (k+1) dt) -- reading R16
// (t0 = first timestamp; interior empty windows are emitted).  offsets[k] is the first event
// with t >= t0 + k dt, found by binary search (one thread per window boundary); a second grid
// stride checks that the timestamps are non-decreasing and latches kErrOrder otherwise.
#pragma once
#include <cstdint>

namespace ieds {

__global__ void window_offsets_kernel(const int64_t* __restrict__ t, int64_t n, int64_t t0, int64_t dt,
                                      int64_t K, int64_t* __restrict__ offsets, int* __restrict__ err) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = tid; k <= K; k += nthr) {
        int64_t lo = 0, hi = n;
        if (k == K) {
            lo = n;
        } else {
            const int64_t key = t0 + k * dt;
            while (lo < hi) {   // first index with t >= key
                const int64_t mid = lo + ((hi - lo) >> 1);
                if (__ldg(t + mid) < key) lo = mid + 1;
                else hi = mid;
            }
        }
        offsets[k] = lo;
    }
    // order check, t[i] >= t[i-1] for all i: one HBM pass over the stream (8 B per event).
    // 16-byte loads of timestamp pairs, 4 per lane in flight, each warp on 128 consecutive pairs;
    // the element before a lane's pair is the lane below's second one (lane 0 loads its own).
    bool bad = false;
    if ((reinterpret_cast<uintptr_t>(t) & 15u) == 0) {
        const longlong2* t2 = reinterpret_cast<const longlong2*>(t);
        const int64_t np = n >> 1;
        const int lane = threadIdx.x & 31;
        const int64_t wid = tid >> 5, nw = nthr >> 5;
        for (int64_t base = wid * 128; base < np; base += nw * 128) {
            longlong2 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t m = base + 32 * r + lane;
                v[r] = m < np ? __ldg(t2 + m) : make_longlong2(0, 0);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t m = base + 32 * r + lane;
                long long prev = __shfl_up_sync(0xFFFFFFFFu, v[r].y, 1);
                if (lane == 0) prev = m > 0 && m < np ? __ldg(t + 2 * m - 1) : v[r].x;
                if (m < np) bad |= (v[r].x < prev) | (v[r].y < v[r].x);
            }
        }
        if ((n & 1) && n > 1 && tid == 0) bad |= __ldg(t + n - 1) < __ldg(t + n - 2);   // the unpaired last one
    } else {
        for (int64_t i = tid + 1; i < n; i += nthr) bad |= __ldg(t + i) < __ldg(t + i - 1);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrOrder);
}

}  // namespace ieds
