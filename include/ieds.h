/*
 * ieds.h -- C ABI of the batched inverse-exponential-distance-surface (IEDS) build.
 *
 * Operation (Brebion et al., arXiv 2112.10591; "P:N" = /root/reference/PAPER.md line N):
 * for every time window of events, independently,
 *   a1  edge image E: pixel = 1 iff at least one event of the window fell on it, polarity
 *       ignored (§III-A);
 *   a2  denoising (Algorithm 1): E_d[p] = E[p] and n4_E(p) >= N_d;
 *   a3  filling   (Algorithm 2): E_df[p] = E_d[p] or n4_{E_d}(p) >= N_f,
 *       strictly after a2; out-of-frame neighbours count as non-edge;
 *   a4  exact Euclidean distance transform to the closest E_df pixel (§III-C),
 *       as an exact integer squared distance D2;
 *   a5  surface S = 1 - exp(-sqrt(D2) / alpha) (Eq. (1)), fp32.
 * A window whose E_df is empty has D2 = IEDS_NO_EDGE everywhere and S = 1 (saturated).
 * Row f1 variants (config.transfer / config.out_format): the ablation transfers of §IV-D
 * (Fig. 4) -- Id(d), min(d, bound), ln(d + 1) -- the 8-bit coding of the
 * surface, q = round(255 * S) half away from zero, the 8-bit view of the ablation
 * transfers normalised by their frame maximum, and float16 surfaces.
 * alpha may be derived from the saturation distance with ieds_alpha_from_dsat (Eq. (2)-(3),
 * P:228-233).
 * Further rows: on-device Delta-T windowing (ieds_window_offsets, row f2), the
 * flow-compensated event image and Flow Warping Loss (ieds_fwl_batch, row f3), and
 * a stateful flow consumer with the P:248 edge masking (ieds_flow_*, row f4).
 *
 * Memory model: every array argument of ieds_build_batch is a DEVICE pointer owned by the
 * caller (e.g. a torch tensor); ieds_build_batch_host takes HOST pointers.  The handle owns
 * only its scratch.  Layouts:
 *   events_xy       uint32 [n_events], packed x | (y << 16), x = column, y = row; the
 *                   events of window b are events_xy[window_offsets[b] .. window_offsets[b+1]).
 *   window_offsets  int64 [num_windows + 1], offsets[0] >= 0, non-decreasing,
 *                   offsets[num_windows] <= n_events; empty windows are allowed.
 *   surfaces        float32 [num_windows][height][width], row-major (uint8 with IEDS_OUT_U8,
 *                   float16 with IEDS_OUT_F16).
 *   *_bits          uint32 [num_windows][height][ceil(width/32)]: bit (x % 32) of word x/32
 *                   is pixel x (LSB = lowest x); padding bits beyond width are 0.
 *   sqdist          uint32 [num_windows][height][width]: exact D2, IEDS_NO_EDGE if the
 *                   window's E_df is empty.
 *
 * Errors: functions return IEDS_OK (0) or a negative code.  Argument errors are detected on
 * the host before anything is enqueued.  Data errors found on the device (an event outside
 * the frame -> IEDS_ERANGE, event dropped; bad offsets -> IEDS_EORDER, window left empty)
 * are latched in the handle and returned by the next ieds_sync.
 *
 * Threading: a handle may be used by one host thread at a time; calls on one handle must be
 * issued on streams that are ordered with respect to each other (the scratch is shared).
 * Handles on different devices are independent.
 */
#ifndef IEDS_H
#define IEDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IEDS_NO_EDGE 0xFFFFFFFFu

enum {
    IEDS_OK = 0,
    IEDS_EINVAL = -1,    /* invalid argument / configuration                          */
    IEDS_ERANGE = -2,    /* an event lies outside the width x height frame (device)    */
    IEDS_ECAPACITY = -3, /* batch exceeds a host-API capacity                          */
    IEDS_EORDER = -4,    /* window_offsets not non-decreasing / out of [0, n_events]   */
    IEDS_ECUDA = -5,     /* a CUDA runtime call failed                                  */
    IEDS_ENOMEM = -6     /* device or pinned allocation failed                          */
};

typedef struct ieds_handle ieds_handle; /* opaque */

typedef struct {
    int32_t width;          /* 1 .. 4096 pixels                                         */
    int32_t height;         /* 1 .. 2048 pixels; ceil(width/32)*height words must fit in */
                            /* one CTA's shared memory (ieds_create checks)             */
    int32_t n_d;            /* 0 .. 4, denoising threshold N_d (0 disables)       */
    int32_t n_f;            /* 1 .. 5, filling threshold N_f (5 disables)         */
    double alpha;           /* > 0 and finite, spreading parameter of Eq. (1), pixels    */
    int32_t chunk_windows;  /* windows processed per launch pair (sizes the scratch);    */
                            /* batches of any size are processed chunk by chunk.         */
                            /* 0 = what a 4 GB scratch budget holds (a multiple of the  */
                            /* SM count, 8 to 128 x); the host path pipelines 2 x SMs    */
    int32_t device;         /* CUDA device ordinal; -1 = current device                 */
    int32_t flags;          /* IEDS_FLAG_* bits                                          */
    int32_t transfer;       /* IEDS_TRANSFER_*; 0 = Eq. (1)                             */
    double bound;           /* IEDS_TRANSFER_BOUNDED: upper bound in pixels (> 0) */
    int32_t out_format;     /* IEDS_OUT_F32 (0), IEDS_OUT_U8 (1) or IEDS_OUT_F16 (2)     */
} ieds_config;

/* transfer of the distance d = sqrt(D2) (pixels); an empty frame is the limit d -> inf */
#define IEDS_TRANSFER_INVEXP 0  /* 1 - exp(-d / alpha), Eq. (1); empty -> 1        */
#define IEDS_TRANSFER_LINEAR 1  /* Id(d); empty -> +inf                              */
#define IEDS_TRANSFER_BOUNDED 2 /* min(d, bound); empty -> bound                     */
#define IEDS_TRANSFER_LOG 3     /* ln(d + 1); empty -> +inf                          */
#define IEDS_OUT_F32 0          /* float32 surfaces                                          */
#define IEDS_OUT_U8 1           /* uint8.  Eq. (1): q = round(255 * S), half away from zero  */
                                /* (P:231); q must saturate (255) for some D2 <= 2048.        */
                                /* Id / min(d, bound) / ln(d+1): q = round(255 * v / vmax),   */
                                /* vmax = the frame maximum of v; empty   */
                                /* frame -> 255, vmax = 0 -> 0 (DESIGN reading R17).  This    */
                                /* mode runs the exact EDT, a per-window max and a quantise   */
                                /* pass, with a table of v over every D2 of the frame (fp64). */
#define IEDS_OUT_F16 2          /* float16 (IEEE binary16) surfaces: the fp64 transfer value  */
                                /* rounded to nearest even (beyond the table, for Id and ln,  */
                                /* the fp32 value rounded to nearest even)                    */

/* Always run the uncapped exact-EDT kernel.  By default, when sqdist is not requested and
 * the saturation radius c = ceil(sqrt(K_sat)) is <= 40 pixels, the surface is produced by
 * the saturation-aware streaming kernel, which evaluates D2 exactly wherever D2 < K_sat and
 * gives bit-identical surfaces (K_sat = first D2 whose fp32 Eq. (1) value is 1.0f). */
#define IEDS_FLAG_EXACT_EDT 1

/* Testing aid: split every frame into 64-row bands (one CTA per band, see ieds_create) even
 * when it fits one CTA, so the banded frame kernel can be checked on small frames. */
#define IEDS_FLAG_TEST_BANDS 2

/* Validates cfg, allocates the scratch on cfg->device and builds the Eq. (1) table.
 * On success *out is a new handle; on failure *out is NULL.
 * Frame size: a window's bit frame is held in shared memory by one CTA when
 *   4 * (4 + (height + 6) * NWP) + 8 * max(width, NWP) <= 232448 bytes, NWP = (ceil(width/32) + 1) | 1
 * (1280x720: 129 KB); larger frames (1920x1080 and up to 4096x2048) are split into bands of
 * rows, one CTA each, every band scanning the window's events for its rows plus a 2-row halo.
 * The exact-EDT kernel (sqdist requests, IEDS_FLAG_EXACT_EDT, the non-saturating transfers)
 * needs width <= 3968 (16 column segments of <= 255 columns); wider handles serve surfaces
 * through the streaming kernel and reject sqdist with IEDS_EINVAL. */
int ieds_create(const ieds_config *cfg, ieds_handle **out);

/* NULL-safe.  Synchronises the device before freeing. */
void ieds_destroy(ieds_handle *h);

/* Enqueue the whole path a1..a5 for num_windows windows on `stream` (a cudaStream_t;
 * NULL = legacy default stream).  DEVICE pointers.  surfaces is required; edge_bits,
 * denoised_bits, filtered_bits and sqdist are optional (NULL = not produced).  No host
 * synchronisation and no allocation: the call is CUDA-graph capturable.  num_windows = 0
 * is a no-op.  A batch of more than chunk_windows windows (surfaces only) runs the next
 * chunk's frame kernel on the handle's own side stream, forked from and joined back into
 * `stream` with events inside the call, so all work stays ordered after earlier work on
 * `stream` and before later work on it (also under graph capture). */
int ieds_build_batch(ieds_handle *h, const uint32_t *events_xy, const int64_t *window_offsets,
                     int64_t n_events, int32_t num_windows, void *surfaces, uint32_t *edge_bits,
                     uint32_t *denoised_bits, uint32_t *filtered_bits, uint32_t *sqdist,
                     void *stream);

/* Same operation with HOST pointers (events_xy, window_offsets, surfaces): the library
 * copies events in and surfaces out chunk by chunk, overlapping the copies with the
 * kernels on internal streams, and returns when the surfaces are in host memory.
 * Page-locked host buffers give full PCIe bandwidth.  Grows internal buffers as needed
 * (this entry point may allocate).  Returns data errors directly (no ieds_sync needed).
 * It first synchronises the device, so device-pointer calls on this handle that are still
 * queued on any stream finish before its internal streams reuse the handle's scratch. */
int ieds_build_batch_host(ieds_handle *h, const uint32_t *events_xy,
                          const int64_t *window_offsets, int32_t num_windows, void *surfaces);

/* Row f2 -- windowing of a time-ordered stream (§III-A).  DEVICE pointers.
 * t_us [n] int64 timestamps (non-decreasing; otherwise IEDS_EORDER is latched for ieds_sync),
 * t0_us = the first timestamp, dt_us > 0 the window length Delta T, num_windows =
 * floor((t_last - t0)/dt) + 1.  Writes window_offsets [num_windows + 1]: window k is
 * events [offsets[k], offsets[k+1]) = the events with floor((t - t0)/dt) == k (half-open
 * windows; empty interior windows are emitted).  The events array in the same order is then
 * the events_xy input of ieds_build_batch.  Enqueued on `stream`; no host sync. */
int ieds_window_offsets(ieds_handle *h, const int64_t *t_us, int64_t n, int64_t t0_us, int64_t dt_us,
                        int32_t num_windows, int64_t *window_offsets, void *stream);

/* Row f2 -- the window count of a time-ordered DEVICE stream t_us [n] (reading R16):
 * *t0_us = t_us[0] and *num_windows = floor((t_us[n-1] - t0) / dt_us) + 1 (0 when n = 0), the
 * num_windows that ieds_window_offsets takes.  Reads the two end timestamps (two 8-byte copies
 * on `stream`) and synchronises that stream.  t0_us / num_windows are HOST pointers.
 * IEDS_EORDER if t_us[n-1] < t_us[0]; IEDS_ECAPACITY if the count exceeds INT32_MAX. */
int ieds_window_count(ieds_handle *h, const int64_t *t_us, int64_t n, int64_t dt_us, int64_t *t0_us,
                      int32_t *num_windows, void *stream);

/* ---- Row f2: streaming ingest (Fig. 1 pipeline) -----------------------------
 * The paper's accumulation thread fills a buffer event by event, and a second thread builds
 * the image "when the time window has expired".  An ieds_stream does that for a live
 * stream delivered in host chunks of any size: it windows the events by Delta T on the device
 * (t0 = the first event of the stream, window k = floor((t - t0)/dt) == k, reading R16),
 * carries the still-open window's events on the device from one push to the next, and
 * returns the surface of every window as soon as an event of a later window arrives.
 * Results are bit-identical to ieds_window_offsets + ieds_build_batch over the whole stream,
 * wherever the stream is cut (tests/test_gpu_stream.py).
 * Host buffers: t_us int64 [n] (non-decreasing across the whole stream), events_xy uint32 [n]
 * (x | y << 16); page-locked chunks are copied to the device directly, any other host memory is
 * staged through the stream's pinned buffers (a host copy per push).
 * Surfaces are written to the HOST array `surfaces` ([max_out][H][W] of the handle's output
 * type); page-locked memory gives full PCIe bandwidth.  Calls are synchronous (they return
 * with the surfaces in host memory) and use the handle's scratch: do not interleave them with
 * other calls on the same handle from another thread. */
typedef struct ieds_stream ieds_stream;

/* A stream on handle h (which it borrows: destroy the stream first) with window length dt_us. */
int ieds_stream_create(ieds_handle *h, int64_t dt_us, ieds_stream **out);

/* Number of windows a push of a chunk with first / last timestamps t_first_us / t_last_us
 * would close (the capacity that push needs in `surfaces`; t_first_us sets t0 when it is the
 * stream's first event). */
int64_t ieds_stream_closing(const ieds_stream *s, int64_t t_first_us, int64_t t_last_us);

/* Ingest n events.  Every window that ends before the window of t_us[n-1] is closed: its
 * surface is written to surfaces[*num_out ...] (empty interior windows give the saturated
 * surface).  max_out = capacity of `surfaces` in windows; IEDS_ECAPACITY (nothing consumed)
 * if the push would close more.  IEDS_EORDER (the push is rejected, the stream unchanged) if
 * the chunk starts before the stream's last timestamp or is not non-decreasing; IEDS_ERANGE
 * if an event lies outside the frame (dropped, the push completes). */
int ieds_stream_push(ieds_stream *s, const int64_t *t_us, const uint32_t *events_xy, int64_t n,
                     void *surfaces, int32_t max_out, int32_t *num_out);

/* End of stream: closes the open window (1 surface if any event was pushed since the last
 * flush, else 0) and resets the stream, so the next push starts a new stream with its own t0. */
int ieds_stream_flush(ieds_stream *s, void *surfaces, int32_t max_out, int32_t *num_out);

/* NULL-safe. */
void ieds_stream_destroy(ieds_stream *s);

/* Row f3: flow-compensated event image and Flow Warping Loss of each window (PAPER P:293-297,
 * FWL = var(I_comp) / var(I_uncomp)).  For window b (events
 * window_offsets[b] .. window_offsets[b+1] of the device arrays):
 *   I_uncomp  = signed event image: +1 for events_p > 0, -1 otherwise, at (x, y);
 *   I_comp    = each event's signed unit mass splatted bilinearly at
 *               (x, y) + F_b(x, y) * (t_ref_us[b] - t) / dt_us, evaluated in fp64; an event whose
 *               warped position lies outside [0, W-1] x [0, H-1] is dropped (DESIGN R19);
 *   var       = population variance over all W*H pixels; fwl[b] = var(I_comp) / var(I_uncomp),
 *               NaN when var(I_uncomp) = 0 (no events).
 * Arguments (DEVICE pointers): events_xy uint32 [n_events] (x | y << 16), events_t_us int64
 * [n_events], events_p int8 [n_events], window_offsets int64 [num_windows + 1] (as in
 * ieds_build_batch), flow float32 [num_windows][H][W][2] = (dx, dy) pixels per dt_us (dense,
 * DESIGN R20), t_ref_us int64 [num_windows] (SPEC: the window end), dt_us > 0.
 * Outputs: fwl double [num_windows] (required); var_comp, var_uncomp double [num_windows] and
 * comp_image double [num_windows][H][W] (I_comp) are optional (NULL to skip).
 * Out-of-frame events latch IEDS_ERANGE and are dropped; bad offsets latch IEDS_EORDER (both
 * reported by ieds_sync).  The handle allocates its f3 scratch (two sets of 16 windows of fp64 + int32
 * images, 12 B/px: one set is re-zeroed on an internal stream while the other is used) on the
 * first call.  Enqueued on `stream`; returns IEDS_EINVAL for bad arguments. */
int ieds_fwl_batch(ieds_handle *h, const uint32_t *events_xy, const int64_t *events_t_us,
                   const int8_t *events_p, const int64_t *window_offsets, int64_t n_events,
                   int32_t num_windows, const float *flow, const int64_t *t_ref_us, int64_t dt_us,
                   double *fwl, double *var_comp, double *var_uncomp, double *comp_image,
                   void *stream);

/* ---- Row f4: the flow consumer of the surfaces -------------------------------
 * A stateful, sequential estimator of dense optical flow between consecutive surfaces, then
 * restricted to the denoised edge pixels.  The paper's own flow library is
 * third-party and gives no equations; this is the substitute of DESIGN reading
 * R21: 255-scaled surfaces, 2x2-mean pyramid, the previous flow transported
 * by itself as the prediction, coarse-to-fine incremental Horn-Schunck (Jacobi sweeps on the
 * total flow, weight lambda[l] and iterations[l] per level, level 0 = full resolution), and
 * the temporal filter F = (1 - gamma) F_measured + gamma F_predicted.  fp32 on the device. */
typedef struct ieds_flow_handle ieds_flow_handle;

typedef struct {
    int32_t width, height;     /* 2..65535; level l is (width >> l) x (height >> l), >= 2 x 2  */
    int32_t levels;            /* 1..8 pyramid levels (3)                              */
    int32_t iterations[8];     /* Jacobi sweeps per level, finest first (20 each)      */
    double lambda[8];          /* regularisation weight per level, >= 0 (500 each)     */
    double gamma;              /* temporal filter weight in [0, 1] (0.5)          */
    double scale;              /* surfaces are multiplied by this first (> 0; 255, R21)       */
    int32_t device;            /* CUDA ordinal; -1 = current                                  */
} ieds_flow_config;

/* Validates cfg (IEDS_EINVAL) and allocates the pyramids, state and scratch on the device. */
int ieds_flow_create(const ieds_flow_config *cfg, ieds_flow_handle **out);

/* NULL-safe; waits for the device. */
void ieds_flow_destroy(ieds_flow_handle *h);

/* Starts a new sequence: the next step is a first window. */
int ieds_flow_reset(ieds_flow_handle *h);

/* One window (DEVICE pointers, enqueued on `stream`):
 *   surface    float32 [height][width] (the IEDS surface S of this window);
 *   edge_bits  uint32 [height][ceil(width/32)] denoised edge image E_d (build_batch's
 *              denoised_bits), or NULL for the dense field;
 *   flow       float32 [height][width][2] out: (u, v) pixels per window; 0 off the mask;
 *   valid      uint8 [height][width] out (nullable): E_d (1 everywhere if edge_bits is NULL).
 * The first window of a sequence outputs zero flow with nothing valid.
 * Returns IEDS_EINVAL / IEDS_ECUDA; each step replays one CUDA graph of the per-level kernels. */
int ieds_flow_step(ieds_flow_handle *h, const float *surface, const uint32_t *edge_bits, float *flow,
                   uint8_t *valid, void *stream);

/* Kernel launches of one non-first step (inside and outside its graph). */
int64_t ieds_flow_launches_per_step(const ieds_flow_handle *h);

/* ---- The Fig. 1 pipeline: events in, flow out (rows f2 + a1-a5 + f4) ---------
 * The paper's blocks -- accumulation, denoising and filling, IEDS, flow -- run concurrently, the
 * image of a window being built "when the time window has expired".  An ieds_pipeline
 * takes host chunks of a live stream like ieds_stream_push, builds each closed window's surface
 * and denoised edge bits (handle h), and runs the flow consumer (handle f, same width and height)
 * on them in window order: the surfaces of the next sub-batch of closed windows are built on one
 * internal stream while the flow of the previous ones runs on another, and each window's flow is
 * copied out while the next window's flow is computed.  Results are bit-identical to
 * ieds_stream_push followed by ieds_flow_step per window (tests/test_gpu_pipeline.py).
 * Outputs (HOST, may be NULL): flow float32 [max_out][H][W][2], valid uint8 [max_out][H][W],
 * surfaces [max_out][H][W] of h's output type (which must be IEDS_OUT_F32, the flow's input).
 * The pipeline borrows h and f (destroy it first); flush also resets f (a new sequence). */
typedef struct ieds_pipeline ieds_pipeline;

int ieds_pipeline_create(ieds_handle *h, ieds_flow_handle *f, int64_t dt_us, ieds_pipeline **out);

/* Windows a push of [t_first_us, t_last_us] would close (as ieds_stream_closing). */
int64_t ieds_pipeline_closing(const ieds_pipeline *p, int64_t t_first_us, int64_t t_last_us);

/* As ieds_stream_push; for every closed window writes its flow / valid / surface outputs. */
int ieds_pipeline_push(ieds_pipeline *p, const int64_t *t_us, const uint32_t *events_xy, int64_t n,
                       float *flow, uint8_t *valid, void *surfaces, int32_t max_out, int32_t *num_out);

/* End of stream: the open window's outputs (1 window, or 0), then the stream and f are reset. */
int ieds_pipeline_flush(ieds_pipeline *p, float *flow, uint8_t *valid, void *surfaces, int32_t max_out,
                        int32_t *num_out);

/* NULL-safe. */
void ieds_pipeline_destroy(ieds_pipeline *p);

/* Wait for `stream`, then return (and clear) the latched device error, or IEDS_OK. */
int ieds_sync(ieds_handle *h, void *stream);

/* Number of kernel launches ieds_build_batch issues for num_windows windows (2 per chunk:
 * frame + surface kernel; 4 in the normalised 8-bit mode: + per-window max + quantise). */
int64_t ieds_launches_per_batch(const ieds_handle *h, int32_t num_windows);

/* Per-kernel device timing (tracing).  While enabled, ieds_build_batch records a CUDA event
 * pair around every kernel it launches (on the caller's stream; the event pool grows as
 * needed, so this mode may allocate).  ieds_profile_read waits for the recorded events and
 * returns the summed device time in ms and the launch count of each kernel since the last
 * read, then resets the counters.  kernel 0 = frame (a1-a3), kernel 1 = EDT + surface (a4-a5).
 * Any output pointer may be NULL. */
int ieds_profile_enable(ieds_handle *h, int on);
int ieds_profile_read(ieds_handle *h, double *frame_ms, int64_t *frame_launches, double *edt_ms,
                      int64_t *edt_launches);

/* Static description of an error code. */
const char *ieds_strerror(int code);

/* Eq. (2)-(3): alpha = -d_sat / ln(1/255) = d_sat / ln 255.  NaN if d_sat <= 0
 * or not finite. */
double ieds_alpha_from_dsat(double d_sat);

/* Library / kernel build identification string. */
const char *ieds_version(void);

#ifdef __cplusplus
}
#endif

#endif /* IEDS_H */
