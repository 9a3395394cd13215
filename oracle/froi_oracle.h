/*
 * froi_oracle.h — CPU restatement of the FlowRoI RoI-extraction path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library, and only as the checker or the timed CPU baseline.  The product path
 * (paper_2511_14419_b200/, libfroi.so) never links or calls it.
 *
 * Every function restates the reference algorithm in plain C, in the same floating-point
 * operation order, so that its outputs are bit-identical to the reference headers compiled in
 * place (oracle/_ref/libfroi_ref.so, see oracle/Makefile); tests/test_oracle_pin.py checks that.
 * Frames are uint16 samples (Frame::pixels, core.hpp:26-58); masks are bytes 0/1.
 */
#ifndef FROI_ORACLE_H_
#define FROI_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/froi/froi.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_threshold_info {
    size_t target;       /* llround(t*n) */
    double boundary;     /* target-th largest value */
    size_t count_greater;/* values strictly above the boundary */
    size_t count_equal;  /* values equal to the boundary */
    size_t ties_admitted;/* equal values admitted in row-major order */
    int degenerate;      /* 1 when boundary <= 0 (mask = values > 0) or target == 0 */
} oracle_threshold_info;

typedef struct oracle_pair_debug {
    double fmag_lo, fmag_hi, grad_lo, grad_hi;
    oracle_threshold_info thr;
} oracle_pair_debug;

/* denoise.hpp */
void oracle_median_filter(const uint16_t* in, int w, int h, int radius, uint16_t* out);
void oracle_bilateral_filter(const uint16_t* in, int w, int h, int depth, int radius,
                             double sigma_spatial, double sigma_range, uint16_t* out);
int oracle_denoise(const uint16_t* in, int w, int h, int depth, const froi_params* p,
                   uint16_t* out);

/* registration.hpp */
int oracle_estimate_shift(const uint16_t* reference, const uint16_t* moving, int w, int h,
                          int max_shift, froi_shift* out);
void oracle_apply_shift(const uint16_t* in, int w, int h, int dx, int dy, uint16_t* out);
void oracle_unshift_mask(const uint8_t* in, int w, int h, int dx, int dy, uint8_t* out);

/* flow.hpp; planes = 6*w*h doubles in the order c, bx, by, a11, a12, a22 */
void oracle_polynomial_expansion(const double* img, int w, int h, int poly_n, double poly_sigma,
                                 double* planes);
void oracle_flow_step(const double* prev_planes, const double* next_planes, int w, int h,
                      const float* prior_u, const float* prior_v, int window_size, float* out_u,
                      float* out_v);
int oracle_compute_flow(const uint16_t* prev, const uint16_t* next, int w, int h, int depth,
                        const froi_params* p, float* u, float* v);

/* roi.hpp */
int oracle_saliency(const float* u, const float* v, const uint16_t* frame, int w, int h,
                    int depth, double flow_weight, int gradient_source, double* out,
                    oracle_pair_debug* dbg);
int oracle_threshold_mask(const double* map, int w, int h, double roi_threshold, uint8_t* mask,
                          oracle_threshold_info* info);
void oracle_morph_open(const uint8_t* in, int w, int h, int radius, uint8_t* out);
void oracle_morph_close(const uint8_t* in, int w, int h, int radius, uint8_t* out);
/* returns the number of components; areas (nullable) receives label-ordered areas */
size_t oracle_label_components(const uint8_t* mask, int w, int h, int* labels, size_t* areas,
                               size_t areas_capacity);
void oracle_morph_cleanup(uint8_t* mask, int w, int h, int open_radius, int close_radius,
                          int min_area);
int oracle_temporal_ensemble(const uint8_t* masks, int n, int w, int h, int t, int k,
                             uint8_t* out);
/* roi.hpp:337-345 for one pair given its flow (registered coordinates) and raw frame t. */
int oracle_mask_from_flow(const float* u, const float* v, const uint16_t* raw_frame, int w,
                          int h, int depth, int dx, int dy, const froi_params* p, uint8_t* mask,
                          oracle_pair_debug* dbg);
/* extract_roi (roi.hpp:309-364).  frames: n*w*h samples; masks: n*w*h bytes;
 * shifts (nullable): n entries; raw_fractions (nullable): n entries. workers <= 1: serial. */
/* Reversible 5/3 DWT (dwt.hpp:113-171) in the canonical in-place layout, DC-shifted int32. */
int oracle_dwt_forward(const uint16_t* frame, int w, int h, int depth, int levels, int32_t* coeffs);
int oracle_dwt_inverse(const int32_t* coeffs, int w, int h, int depth, int levels, uint16_t* frame);
/* map_mask_to_subbands (codec.hpp:152-171): level masks concatenated, level 1 first. */
size_t oracle_map_mask_to_subbands(const uint8_t* mask, int w, int h, int levels, uint8_t* out);

int oracle_extract_roi(const uint16_t* frames, int n, int w, int h, int depth,
                       const froi_params* p, int workers, uint8_t* masks, froi_shift* shifts,
                       double* raw_fractions);

/* glibc-2.39-compatible double hypot restated (used by the GPU kernels; exported for tests) */
double oracle_hypot_restated(double x, double y);

#ifdef __cplusplus
}
#endif
#endif
