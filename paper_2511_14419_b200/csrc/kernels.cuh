// kernels.cuh — device data layout and kernel launchers of the RoI-extraction path.
//
// HBM layout (one context, W x H frames, sample type T = uint8 or uint16):
//   frame slots  f in [0, Fcap): raw T[H*W] (ingest), den T[H*W], spec double2[ph*pw]
//                (full complex spectrum of the windowed denoised frame), pyramid float
//                images of levels >= 1, expansion planes per level: exA float4 {a11,a12,a22,bx}
//                and exB float {by}, concatenated over levels (offset loff[l], lsum total px).
//   pair slots   p in [0, Pcap): PairInfo, inverse-row columns double2[(2M+1)*ph], surface
//                double[(2M+1)^2], shifted-next pyramid/expansions (only when the applied
//                shift is non-zero), flow ping-pong float2[lsum] x 2, mask-stage scratch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace froi {

constexpr int kMaxLevels = 16;
constexpr int kSelBits = 11;  // radix-select digit width
constexpr int kSelBins = 1 << kSelBits;
constexpr int kHistBins = 4096;  // per-query global histogram stride (radix digit or exponent window)
constexpr int kMaxQueries = 4;
constexpr int kSelCap = 16384;  // candidates sorted in shared memory once a radix bin is this small
enum SelMode { SEL_HIST = 0, SEL_COLLECT = 1, SEL_DONE = 2 };

struct Geom {
    int W, H, depth, maxval;
    int sample_bytes;   // 1 or 2
    int L;              // effective pyramid levels
    int lw[kMaxLevels], lh[kMaxLevels];
    long long loff[kMaxLevels];  // pixel offset of level l inside a per-frame pyramid buffer
    long long lsum;              // total pixels over levels
    int pw, ph, log2pw, log2ph;  // FFT grid (next_pow2)
    int WW;                      // 32-bit words per packed mask row
    int SB;                      // bytes per PBM row
    int RMAX;                    // max runs of set pixels per row, (W+1)/2
};

struct PairInfo {
    int est_dx, est_dy;
    double confidence;
    int dx, dy;  // applied (0,0 after the 1.5 fallback)
    int shifted;
    int pad0;
    // mask stage
    double fmag_lo, fmag_hi, grad_lo, grad_hi;
    double fmag_inv, grad_inv;
    int fmag_zero, grad_zero;  // robust_normalize degenerate -> all zeros
    double boundary;
    unsigned long long count_eq;
    unsigned long long target;
    unsigned long long count_gt;
    unsigned long long need;
    int thr_mode;  // 0 all ties admitted (S >= b), 1 empty, 2 positive-only, 3 partial ties
    unsigned int mask_count;
    unsigned int components;
    unsigned int pad1;
    // threshold words already written by phase B's collect pass (all pixels outside the boundary
    // bin); the bin's n_cand candidates are settled by k_thr_fixup
    int bits_ready;
    unsigned int n_cand;
};

struct SelState {
    unsigned long long prefix;
    unsigned long long rank;     // rank within the current prefix group
    unsigned long long k0;       // requested rank (0-based, ascending)
    unsigned long long result;
    unsigned long long mn, mx;   // min / max key of prefix matches in the last pass
    unsigned long long count;    // elements matching the prefix
    unsigned long long count_lt; // on completion: elements below the result
    unsigned long long count_eq; // on completion: elements equal to the result
    int bits_done;
    int mode;                    // SelMode
    int fpw;                     // first pass digit while bits_done == 0: 0 radix, 1 / 2 the
                                 // exponent-window digit of a double / fkey (float) key
};

// Per-batch device tables.
struct BatchTables {
    const void** frame_raw;  // [Fcap] raw frame pointer of each frame slot
    int* pair_prev;          // [Pcap] frame slot of frame t-1
    int* pair_next;          // [Pcap] frame slot of frame t
};

// Device parameter block (constant per context).
struct DevParams {
    // denoise
    int denoise_enabled, median_radius, bilateral_radius;
    // flow
    int window_radius, iterations, poly_radius;
    float poly_moments[7];  // inv_m20, inv_m22, i00, i01, i11, i12, unused
    float g0[16], g1[16], g2[16];  // polynomial-expansion kernels (radius <= 7)
    float blur[7];                 // pyramid Gaussian (sigma 1, radius 3)
    double pyr_scale;
    // roi
    double roi_threshold, flow_weight;
    int min_area, open_radius, close_radius, gradient_source, max_shift;
    // 8-bit frames: normalize_frame's (float)(v * (1.0/maxval)) for v = 0..255 (device, context)
    const float* norm_lut;
    // 8-bit frames: exact |grad I| by table (context constants, nullptr otherwise).  A central
    // difference 0.5*(v[a] - v[b]) of normalised samples takes grad_nv distinct magnitudes
    // (809 for maxval 255); grad_map[a*256 + b] is the index of |0.5*(v[a]-v[b])| among them and
    // grad_tab[i*grad_nv + j] the restated glibc hypot of magnitudes i and j.
    const unsigned short* grad_map;
    const double* grad_tab;
    int grad_nv;
};

// ---------------------------------------------------------------- launchers
// k_denoise.cu
void launch_denoise(const Geom& g, const DevParams& p, const void** d_frame_raw, void* d_den,
                    unsigned long long* d_sums, const double* h_spatial, const double* d_lut,
                    int n_slots, cudaStream_t s);  // h_spatial: host copy of the spatial weights

// k_register.cu
void launch_fft_forward(const Geom& g, const void* d_den, const unsigned long long* d_sums,
                        const double* d_wx, const double* d_wy, const double2* d_tw_row,
                        const double2* d_tw_col, double2* d_spec, int n_slots, cudaStream_t s);
void launch_register_pairs(const Geom& g, const DevParams& p, const double2* d_spec,
                           const int* d_prev, const int* d_next, const double2* d_itw_row,
                           const double2* d_itw_col, double2* d_cols, double* d_surf,
                           PairInfo* d_info, int n_pairs, cudaStream_t s);

// k_dwt.cu (codec side)
void launch_dwt_forward(const void* d_frames, int sample_bytes, int W, int H, int depth, int n,
                        int levels, int32_t* d_coeffs, cudaStream_t s);
void launch_dwt_inverse(int32_t* d_coeffs, int W, int H, int depth, int n, int levels,
                        uint16_t* d_frames, cudaStream_t s);
size_t launch_map_mask_to_subbands(const uint8_t* d_mask, int W, int H, int levels, bool any,
                                   uint8_t* d_out, cudaStream_t s);

// k_flow.cu
struct FlowBuffers {
    const void* den;     // frame-slot denoised frames (T)
    float* pyr_f;        // frame-slot pyramid images, levels >= 1 ([slot][lsum - W*H])
    float4* exA_f;       // frame-slot expansions [slot][lsum]
    float* exB_f;
    float* pyr_p;        // pair-slot shifted pyramids
    float4* exA_p;       // pair-slot shifted expansions
    float* exB_p;
    float2* flow0;       // pair-slot flow ping-pong [pair][lsum]
    float2* flow1;
};
void launch_expand_frames(const Geom& g, const DevParams& p, const FlowBuffers& b, int n_slots,
                          cudaStream_t s);
void launch_expand_shifted(const Geom& g, const DevParams& p, const FlowBuffers& b,
                           const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s);
// Runs all levels and iterations; returns which buffer holds the level-0 flow (0 or 1).
int launch_flow(const Geom& g, const DevParams& p, const FlowBuffers& b, const int* d_prev,
                const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s);
// Debug tap: expansion (6 planes incl. c) of a float image of level-0 geometry.
void launch_expand_image(const Geom& g, const DevParams& p, const float* d_img, float* d_planes,
                         cudaStream_t s);

// k_flow64.cu: the bit-exact fp64 flow (froi_ctx_set_flow_exact)
struct Flow64Const {
    double g0[16], g1[16], g2[16];  // polynomial-expansion kernels w, w t, w t^2 (index t + r)
    double blur[16];                // gaussian_blur3's normalised taps (sigma 1)
    int blur_r, poly_r;
    double inv_m20, inv_m22, i01, i11, i12;  // expansion_moments' inverse (flow.hpp:92-112)
};
struct Flow64Buffers {
    double* img_f;   // frame-slot pyramid images, all levels [slot][lsum]
    double* ex_f;    // frame-slot expansions [slot][5 planes bx, by, a11, a12, a22][lsum]
    double* tmp_f;   // row-blur scratch of the frame slots [slot][W*H]
    double* img_p;   // pair-slot shifted pyramids
    double* ex_p;    // pair-slot shifted expansions
    double* tmp_p;   // row-blur scratch of the pair slots
    double* prod;    // [pair][5][W*H] products, then window means
    double* rowm;    // [pair][5][W*H] row means
    float2* flow0;   // the float2 flow ping-pong shared with the fp32 path
    float2* flow1;
};
int launch_expand_frames64(const Geom& g, const Flow64Const& C, const Flow64Buffers& b, const void* den,
                           int n_slots, cudaStream_t s);
int launch_expand_shifted64(const Geom& g, const Flow64Const& C, const Flow64Buffers& b, const void* den,
                            const int* d_next, const PairInfo* d_info, int n_pairs, cudaStream_t s);
// all levels and iterations; *cur_out = the buffer holding the level-0 flow; returns launches
int launch_flow64(const Geom& g, const DevParams& p, const Flow64Buffers& b, const int* d_prev, const int* d_next,
                  const PairInfo* d_info, int n_pairs, cudaStream_t s, int* cur_out);

// k_mask.cu
struct MaskBuffers {
    const float2* flow;           // [pair][lsum] level-0 flow at offset 0
    long long flow_stride;        // elements between pairs
    const void** raw;             // [pair] raw frame t pointer (T)
    SelState* sel;                // [pair][kMaxQueries]
    unsigned int* hist;           // [pair][kMaxQueries][kHistBins]
    unsigned long long* cand;     // [pair][kMaxQueries][kSelCap]
    unsigned int* cand_count;     // [pair][kMaxQueries]
    unsigned int* cand_idx;       // [pair][kSelCap] pixel index of each phase-B candidate
    float* fm;                    // [pair][H*W] |flow| (FlowField::mag)
    double* gr;                   // [pair][H*W] |grad I|
    unsigned long long* tie_cnt;  // [pair][chunks][2]
    uint32_t* bits_thr;           // [pair][H*WW] thresholded (registered)
    uint32_t* bits_clean;         // [pair][H*WW] after open/close (registered)
    uint32_t* bits_keep;          // [pair][H*WW] pixels of components with area >= min_area
    uint16_t* run_x0;             // [pair][H][RMAX] first x of each run of set pixels
    uint16_t* run_x1;             // [pair][H][RMAX] last x
    int* run_n;                   // [pair][H] runs per row
    int* run_par;                 // [pair][H*RMAX] union-find parent (run ids y*RMAX + k)
    unsigned int* run_area;       // [pair][H*RMAX] component area at the root run
    uint8_t* out_pbm;             // output PBM masks
    const long long* out_index;   // [pair] mask index in out_pbm (frame index)
    PairInfo* info;
};
void launch_mask_stage(const Geom& g, const DevParams& p, const MaskBuffers& b, int n_pairs,
                       cudaStream_t s, uint64_t* launches);
// grad_tab[i*nv + j] = hypot_glibc(mag[i], mag[j]) (context creation)
void launch_grad_table(const double* d_mag, int nv, double* d_tab, cudaStream_t s);
// Debug taps on the same kernels.
void launch_saliency_map(const Geom& g, const DevParams& p, const MaskBuffers& b, double* d_out,
                         cudaStream_t s);
void launch_threshold_from_map(const Geom& g, const DevParams& p, const MaskBuffers& b,
                               const double* d_map, double threshold, cudaStream_t s);
void launch_cleanup_only(const Geom& g, const DevParams& p, const MaskBuffers& b,
                         int open_radius, int close_radius, int min_area, cudaStream_t s);
void launch_unpack_pbm(const Geom& g, const uint8_t* d_pbm, uint8_t* d_bytes, int n_masks,
                       cudaStream_t s);
void launch_pack_bytes_to_words(const Geom& g, const uint8_t* d_bytes, uint32_t* d_words,
                                cudaStream_t s);
void launch_ensemble(const Geom& g, const uint8_t* d_in, uint8_t* d_out, int n, int k,
                     cudaStream_t s);

}  // namespace froi
