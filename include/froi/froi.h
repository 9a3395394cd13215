/*
 * froi.h — C ABI of the B200-native FlowRoI RoI-extraction stage.
 *
 * This is the drop-in boundary for the reference's stage entry
 *   std::vector<RoiMask> flowroi::extract_roi(const Sequence&, const ExtractParams&,
 *                                             int workers, ExtractInfo*, StageTimes*)
 *   (/root/reference/proj/include/flowroi/roi.hpp:309-364)
 * and for its sub-operators (compute_flow, denoise, estimate_shift, saliency,
 * threshold_mask, morph_cleanup, label_components, temporal_ensemble).  The reference has
 * no FFI of its own: its boundary is the inline C++ API in namespace flowroi.  Each entry
 * below names the reference function it replaces; include/froi/flowroi_gpu.hpp wraps these
 * entries back into the reference's own C++ signatures.
 *
 * Conventions:
 *   - status codes: 0 ok, 1 usage error, 2 data error, 3 internal / CUDA error
 *     (the CLI taxonomy of proj/tools/flowroi.cpp:610-621; usage_error/data_error are
 *     /root/reference/proj/include/flowroi/core.hpp:14-22);
 *   - froi_last_error() returns a thread-local message for the last non-zero status;
 *   - the caller owns every host buffer, the library owns device memory;
 *   - a context is affine to one host thread; distinct contexts may run concurrently;
 *   - no exceptions cross the ABI; there is no CPU fallback: without a usable CUDA device
 *     every compute entry returns 3.
 *
 * Frames are row-major samples of `sample_bytes` = 1 (uint8) or 2 (uint16) bytes.  `depth`
 * (8 or 16) is the reference's Frame::depth (core.hpp:26-58): maxval = 2^depth - 1 is used for
 * normalisation even when the data only occupy 12 bits.  Masks are returned either as the
 * reference's RoiMask bytes (one byte 0/1 per pixel, core.hpp:78-101) or bit-packed in the
 * PBM P4 row layout (MSB first, row stride ceil(W/8) bytes, pgm.hpp:127-138).
 */
#ifndef FROI_H_
#define FROI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FROI_OK 0
#define FROI_ERR_USAGE 1
#define FROI_ERR_DATA 2
#define FROI_ERR_INTERNAL 3

#define FROI_MASK_BYTES 0 /* RoiMask layout: W*H bytes, 0 or 1 */
#define FROI_MASK_PBM 1   /* PBM P4 layout: H rows of ceil(W/8) bytes, MSB first */

#define FROI_GRADIENT_IMAGE 0 /* SaliencyGradient::image (roi.hpp:18) */
#define FROI_GRADIENT_FLOW 1  /* SaliencyGradient::flow  (roi.hpp:18) */

/* ExtractParams{denoise, flow, roi, max_shift} (roi.hpp:263-268), field for field. */
typedef struct froi_params {
    /* DenoiseParams (denoise.hpp:11-24) */
    int denoise_enabled;            /* true */
    int median_radius;              /* 1 -> 3x3 */
    double bilateral_sigma_spatial; /* 2.0 */
    double bilateral_sigma_range;   /* 0.04, on intensities normalised by maxval */
    int bilateral_radius;           /* 2 -> 5x5 */
    /* FlowParams (flow.hpp:12-30) */
    int pyramid_levels;   /* 3 */
    double pyramid_scale; /* 0.5 */
    int window_size;      /* 15 */
    int iterations;       /* 3 */
    int poly_n;           /* 5 */
    double poly_sigma;    /* 1.1 */
    /* RoiParams (roi.hpp:20-38) */
    double roi_threshold; /* 0.2 */
    double flow_weight;   /* 0.7 */
    int adjacent_factor;  /* 0 */
    int min_area;         /* 20 */
    int open_radius;      /* 1 */
    int close_radius;     /* 1 */
    int gradient_source;  /* FROI_GRADIENT_IMAGE */
    /* ExtractParams::max_shift (roi.hpp:267, registration.hpp:20) */
    int max_shift; /* 16 */
} froi_params;

/* Shift (registration.hpp:13-17). */
typedef struct froi_shift {
    int dx;
    int dy;
    double confidence;
} froi_shift;

/* Per-frame diagnostics: ExtractInfo{shifts, raw_fractions} (roi.hpp:271-274) plus counts. */
typedef struct froi_frame_stats {
    int dx;              /* applied shift of frame t relative to t-1 ((0,0) after fallback) */
    int dy;
    double confidence;   /* phase-correlation confidence (kept through the fallback) */
    double raw_fraction; /* mask fraction before temporal ensembling */
    uint32_t mask_count; /* set pixels before temporal ensembling */
    uint32_t components; /* 8-connected components of the cleaned mask (registered frame) */
} froi_frame_stats;

/* StageTimes (roi.hpp:278-283): accumulated device time per stage, nanoseconds. */
typedef struct froi_stage_times {
    uint64_t denoise_ns;
    uint64_t flow_ns; /* registration + flow, as in roi.hpp:331 */
    uint64_t roi_ns;
    uint64_t encode_ns; /* never touched here: encoding stays on the CPU */
} froi_stage_times;

/* Device time per kernel group, accumulated over the batches of the last extract call
 * (CUDA events on the context stream), plus the work counts needed for roofline figures. */
typedef struct froi_kernel_times {
    uint64_t denoise_ns;        /* k_denoise */
    uint64_t fft_forward_ns;    /* k_fft_rows_fwd + k_fft_cols */
    uint64_t expand_ns;         /* pyramid + polynomial expansion of the frame slots */
    uint64_t register_ns;       /* cross-power, inverse FFT, argmax */
    uint64_t expand_shifted_ns; /* pyramid + expansion of registered next frames (s != 0) */
    uint64_t flow_iter_ns;      /* all k_flow_iter launches */
    uint64_t mask_ns;           /* saliency selection, threshold, morphology, CCL, output */
    uint64_t pairs;             /* adjacent pairs processed */
    uint64_t frames;            /* frame slots processed (denoise / FFT / expansion) */
    uint64_t flow_iter_launches;
    uint64_t batches;
} froi_kernel_times;

typedef struct froi_ctx froi_ctx;

/* ---- library / host-only entries (no GPU needed) ---- */
const char* froi_version(void);
const char* froi_last_error(void);
/* Default-constructed ExtractParams{} (roi.hpp:263-268). */
void froi_params_default(froi_params* p);
/* RoiParams::validate + FlowParams::validate + DenoiseParams::validate
 * (roi.hpp:29-37, flow.hpp:20-29, denoise.hpp:18-23). Returns 0 or FROI_ERR_USAGE. */
int froi_params_validate(const froi_params* p);
/* Pyramid geometry the flow will use for a W x H frame (build_pyramid, flow.hpp:287-298). */
int froi_pyramid_levels(const froi_params* p, int width, int height, int* levels_out, int* widths,
                        int* heights);
int froi_device_count(int* count);

/* ---- context ---- */
/* Per-GPU context: device arenas, stream, FFT twiddles.  `max_pairs` bounds the number of
 * adjacent pairs processed per launch batch (0 = choose from free memory). */
int froi_ctx_create(int device, const froi_params* p, int width, int height, int depth,
                    int max_pairs, froi_ctx** out);
void froi_ctx_destroy(froi_ctx* ctx);
int froi_ctx_get_params(const froi_ctx* ctx, froi_params* out);
/* Replace params (same geometry). Validated like froi_params_validate. */
int froi_ctx_set_params(froi_ctx* ctx, const froi_params* p);
/* Device time of the last extract call per stage (sum over batches). */
int froi_ctx_stage_times(const froi_ctx* ctx, froi_stage_times* out);
/* Number of kernels launched by the last extract call. */
int froi_ctx_launch_count(const froi_ctx* ctx, uint64_t* out);
/* Per-kernel-group device times of the last extract call. */
int froi_ctx_kernel_times(const froi_ctx* ctx, froi_kernel_times* out);
/* The context's CUDA stream (cudaStream_t), for callers that time or order work around it.
 * Extract calls end with all their work ordered on this stream (and the host synchronised). */
int froi_ctx_stream(const froi_ctx* ctx, void** stream_out);
/* Execution lanes (1 or 2, default 2 or $FROI_LANES): with 2, the batches of one call alternate
 * between two buffer sets on two streams so their kernels overlap; outputs are identical.
 * Per-stage times (froi_ctx_kernel_times) are exact kernel durations only with 1 lane. */
int froi_ctx_set_lanes(froi_ctx* ctx, int lanes);
/* Intra-batch overlap (1, default, or $FROI_FORK=0 at creation): each batch's frame expansions run
 * on a side branch concurrently with its forward FFT and registration.  0 serialises them, so the
 * per-stage times of froi_ctx_kernel_times bracket each stage's own kernels; outputs are identical. */
int froi_ctx_set_fork(froi_ctx* ctx, int fork);
/* Flow precision (0, default: fp32 flow within the stated tolerance; 1: bit-exact).
 * With 1 the pyramid, polynomial expansion, flow_step with the reference's running-sum box_mean,
 * and the coarse-to-fine prior run in fp64 in the reference's operation order (k_flow64.cu), so
 * flows and masks are byte-identical to the reference's; slower, and allocates its double buffers
 * (about 14 GB per lane at 1024^2 with 64-pair batches) on first use.  Status 3 if they do not fit. */
int froi_ctx_set_flow_exact(froi_ctx* ctx, int exact);
int froi_ctx_get_flow_exact(const froi_ctx* ctx, int* exact_out);

/* ---- stage entry: extract_roi (roi.hpp:309-364) ----
 * Host frames: n_frames frames of width*height samples; frame f starts at
 * frames + f*frame_stride_bytes.  Masks: n_frames masks in `mask_layout`, frame-major.
 * stats (nullable): n_frames entries. */
int froi_extract_roi(froi_ctx* ctx, const void* frames, int sample_bytes,
                     size_t frame_stride_bytes, int n_frames, int mask_layout, uint8_t* masks_out,
                     froi_frame_stats* stats_out);

/* Several independent sequences ("wells") of equal length in one call; wells are
 * independent and are batched together on the device.  frames is
 * well-major: frame f of well w at frames + (w*n_frames + f)*frame_stride_bytes; masks
 * and stats likewise well-major. */
int froi_extract_wells(froi_ctx* ctx, const void* frames, int sample_bytes,
                       size_t frame_stride_bytes, int n_wells, int n_frames, int mask_layout,
                       uint8_t* masks_out, froi_frame_stats* stats_out);

/* Host entries (froi_extract_roi / _wells / _frames, froi_stream_push) stream the frames through
 * bounded rings: frames of any host memory are converted into a pinned staging
 * ring by host threads (pinned frames of the context's sample type are copied directly), copied
 * into a device ring of a few batches' frames just ahead of the batch that needs them, and each
 * batch's masks return while later batches compute.  Device and pinned memory do not grow with
 * the call.  A sample above the depth's maxval (u16 frames of an 8-bit context) is a data error.
 *
 * Per-frame pointers: the reference's Sequence holds separately allocated Frames (core.hpp:61-75)
 * and extract_roi returns separately allocated RoiMasks (roi.hpp:309-311).  frames[t] points at
 * width*height samples of `sample_bytes` (Frame::pixels are uint16: sample_bytes 2), masks[t] at
 * one mask in `mask_layout`; host memory of any kind. */
int froi_extract_frames(froi_ctx* ctx, const void* const* frames, int sample_bytes, int n_frames,
                        int mask_layout, uint8_t* const* masks, froi_frame_stats* stats_out);

/* A mask destination supplied on demand: called (from the library's host threads, concurrently,
 * each (well, frame) once; frame 0 after frame 1) just before mask `frame` of `well` is written;
 * returns where its W*H bytes (or PBM rows) go.  Lets a caller allocate its RoiMasks while the GPU
 * works instead of before the call.  The sink must not unwind (C++ exceptions must not cross
 * it); returning NULL fails the call with FROI_ERR_USAGE. */
typedef uint8_t* (*froi_mask_sink)(void* user, int well, int frame);
int froi_extract_frames_sink(froi_ctx* ctx, const void* const* frames, int sample_bytes, int n_frames,
                             int mask_layout, froi_mask_sink sink, void* user,
                             froi_frame_stats* stats_out);

/* Finished masks handed over instead of written: the library unpacks each mask into a buffer of
 * its own and calls put(user, well, frame, mask) from its host threads (concurrently; each
 * (well, frame) once, frame 0 after frame 1); the caller copies the W*H bytes (or PBM rows) out
 * before returning 0.  This is the drop-in's path: a RoiMask built from the bytes in one pass
 * (std::vector::assign) costs one memory write instead of a zero-fill plus the unpack.  A
 * non-zero return fails the call with FROI_ERR_USAGE; the callback must not unwind. */
typedef int (*froi_mask_put)(void* user, int well, int frame, const uint8_t* mask);
int froi_extract_frames_put(froi_ctx* ctx, const void* const* frames, int sample_bytes, int n_frames,
                            int mask_layout, froi_mask_put put, void* user, froi_frame_stats* stats_out);

/* Device-resident variant used for the device-side throughput figure: d_frames is a device
 * pointer (well-major, as above), d_masks_pbm receives PBM-packed masks on the device.
 * stats_out is a HOST pointer (nullable). Asynchronous work is complete on return. */
int froi_extract_wells_device(froi_ctx* ctx, const void* d_frames, int sample_bytes,
                              size_t frame_stride_bytes, int n_wells, int n_frames,
                              uint8_t* d_masks_pbm, froi_frame_stats* stats_out);

/* ---- streaming ingest (per-well streams) ----
 * froi_stream_reset starts n_wells new sequences.  Each froi_stream_push hands over `chunk`
 * new frames per well (well-major, host or device memory) and returns the masks that became
 * final: on the first push of a well the masks of frames 0..chunk-1, afterwards the masks of
 * the pushed frames (mask of frame 0 = mask of frame 1, roi.hpp:348).  adjacent_factor must be
 * 0 in streaming mode (the ensemble needs look-ahead; use froi_extract_* for k > 0).  The first
 * push of a sequence needs chunk >= 2. */
int froi_stream_reset(froi_ctx* ctx, int n_wells);
int froi_stream_push(froi_ctx* ctx, const void* frames, int frames_on_device, int sample_bytes,
                     size_t frame_stride_bytes, int chunk, int mask_layout, uint8_t* masks_out,
                     int masks_on_device, froi_frame_stats* stats_out);
/* froi_stream_push with one host pointer per frame and per mask (frames[w*chunk + t],
 * masks[w*chunk + t]), for separately allocated Frames / RoiMasks. */
int froi_stream_push_frames(froi_ctx* ctx, const void* const* frames, int sample_bytes, int chunk,
                            int mask_layout, uint8_t* const* masks, froi_frame_stats* stats_out);

/* ---- sub-operators (parity taps; each computes on the GPU with the product kernels) ---- */
/* denoise (denoise.hpp:84-90): median then bilateral, or copy if disabled. */
int froi_denoise(froi_ctx* ctx, const uint16_t* in, uint16_t* out);
/* estimate_shift (registration.hpp:46-97) of `moving` relative to `reference`. */
int froi_estimate_shift(froi_ctx* ctx, const uint16_t* reference, const uint16_t* moving,
                        int max_shift, froi_shift* out);
/* compute_flow (flow.hpp:304-345) with the context's FlowParams. u, v: W*H floats. */
int froi_compute_flow(froi_ctx* ctx, const uint16_t* prev, const uint16_t* next, float* u,
                      float* v);
/* polynomial_expansion (flow.hpp:118-153) of a single-precision image of the context's
 * geometry; planes: 6*W*H floats in the order c, bx, by, a11, a12, a22. */
int froi_polynomial_expansion(froi_ctx* ctx, const float* image, float* planes);
/* saliency (roi.hpp:81-103) of (u, v) against frame (already registered); out: W*H doubles. */
int froi_saliency(froi_ctx* ctx, const float* u, const float* v, const uint16_t* frame,
                  double* out);
/* threshold_mask (roi.hpp:109-138) of a W*H double map; mask: W*H bytes. */
int froi_threshold_mask(froi_ctx* ctx, const double* map, double roi_threshold, uint8_t* mask);
/* morph_cleanup (roi.hpp:237-246), in place on W*H mask bytes. */
int froi_morph_cleanup(froi_ctx* ctx, uint8_t* mask, int open_radius, int close_radius,
                       int min_area);
/* label_components (roi.hpp:184-234): component areas (any order) of a W*H mask.
 * areas_out may be NULL to query the count; *n_components receives the count. */
/* ---- codec side on the GPU ----
 * Reversible 5/3 DWT of one frame of the context geometry (dwt_forward / dwt_inverse,
 * dwt.hpp:113-171): DC-shifted int32 coefficients in the canonical in-place layout, bit-identical.
 * levels < 1 -> usage error; frame smaller than 2^levels -> data error. */
int froi_dwt_forward(froi_ctx* ctx, const uint16_t* frame, int levels, int32_t* coeffs);
int froi_dwt_inverse(froi_ctx* ctx, const int32_t* coeffs, int levels, uint16_t* frame);
/* n device frames (context sample type, packed) -> n device coefficient grids. */
int froi_dwt_forward_device(froi_ctx* ctx, const void* d_frames, int n, int levels, int32_t* d_coeffs);
/* RoI coefficient masks (map_mask_to_subbands, codec.hpp:152-171): level 1..levels masks of
 * ceil-halved extents, concatenated; *out_len receives their total size. */
int froi_map_mask_to_subbands(froi_ctx* ctx, const uint8_t* mask, int levels, uint8_t* out,
                              size_t cap, size_t* out_len);

int froi_component_areas(froi_ctx* ctx, const uint8_t* mask, uint32_t* areas_out,
                         size_t areas_capacity, size_t* n_components);
/* Mask stage of one pair from a given flow (roi.hpp:340-345): saliency against
 * apply_shift(raw, shift), threshold, cleanup, unshift.  Lets parity tests check the mask
 * stage in isolation from the flow's floating-point tolerance. */
int froi_mask_from_flow(froi_ctx* ctx, const float* u, const float* v, const uint16_t* raw_frame,
                        int dx, int dy, uint8_t* mask, froi_frame_stats* stats);
/* Parity tap: mask-stage order statistics of pair slot `pair` from the last call, as doubles
 * {fmag_lo, fmag_hi, grad_lo, grad_hi, boundary, count_greater, need, target, thr_mode}
 * (robust_normalize roi.hpp:47-63 and threshold_mask roi.hpp:109-138). n = entries wanted. */
int froi_debug_pair_stats(froi_ctx* ctx, int pair, double* out, int n);
/* temporal_ensemble (roi.hpp:249-261) over n W*H masks for every t; out: n masks. */
int froi_temporal_ensemble(froi_ctx* ctx, const uint8_t* masks, int n, int k, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* FROI_H_ */
