// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference headers, compiled in place.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile builds this file against
// $(FLOWROI_REF_INCLUDE) (default /root/reference/proj/include) into oracle/_ref/libfroi_ref.so
// with the reference's Release flags (-O3 -DNDEBUG, gnu++20, no -march).  No reference source
// is copied into this repository; this file only calls the reference's public functions so that
// Python tests and bench.py (--impl reference, cpu_baseline) can drive the real reference code.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "flowroi/codec.hpp"
#include "flowroi/denoise.hpp"
#include "flowroi/dwt.hpp"
#include "flowroi/flow.hpp"
#include "flowroi/registration.hpp"
#include "flowroi/roi.hpp"
#include "flowroi/rng.hpp"
#include "flowroi/synthetic.hpp"

#include "../include/froi/froi.h"

using namespace flowroi;

namespace {

int status_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const usage_error&) {
        return 1;
    } catch (const data_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

#define SHIM_TRY try {
#define SHIM_CATCH                                  \
    }                                               \
    catch (...) {                                   \
        return status_of(std::current_exception()); \
    }                                               \
    return 0;

Frame make_frame(const uint16_t* px, int w, int h, int depth) {
    Frame f(w, h, depth);
    std::memcpy(f.pixels.data(), px, sizeof(uint16_t) * f.size());
    return f;
}

ExtractParams to_params(const froi_params* p) {
    ExtractParams e;
    e.denoise.enabled = p->denoise_enabled != 0;
    e.denoise.median_radius = p->median_radius;
    e.denoise.bilateral_sigma_spatial = p->bilateral_sigma_spatial;
    e.denoise.bilateral_sigma_range = p->bilateral_sigma_range;
    e.denoise.bilateral_radius = p->bilateral_radius;
    e.flow.pyramid_levels = p->pyramid_levels;
    e.flow.pyramid_scale = p->pyramid_scale;
    e.flow.window_size = p->window_size;
    e.flow.iterations = p->iterations;
    e.flow.poly_n = p->poly_n;
    e.flow.poly_sigma = p->poly_sigma;
    e.roi.roi_threshold = p->roi_threshold;
    e.roi.flow_weight = p->flow_weight;
    e.roi.adjacent_factor = p->adjacent_factor;
    e.roi.min_area = p->min_area;
    e.roi.open_radius = p->open_radius;
    e.roi.close_radius = p->close_radius;
    e.roi.gradient_source =
        p->gradient_source == FROI_GRADIENT_FLOW ? SaliencyGradient::flow : SaliencyGradient::image;
    e.max_shift = p->max_shift;
    return e;
}

}  // namespace

extern "C" {

int ref_denoise(const uint16_t* in, int w, int h, int depth, const froi_params* p, uint16_t* out) {
    SHIM_TRY
    const Frame d = denoise(make_frame(in, w, h, depth), to_params(p).denoise);
    std::memcpy(out, d.pixels.data(), sizeof(uint16_t) * d.size());
    SHIM_CATCH
}

int ref_estimate_shift(const uint16_t* a, const uint16_t* b, int w, int h, int depth, int max_shift,
                       froi_shift* out) {
    SHIM_TRY
    const Shift s = estimate_shift(make_frame(a, w, h, depth), make_frame(b, w, h, depth), max_shift);
    out->dx = s.dx;
    out->dy = s.dy;
    out->confidence = s.confidence;
    SHIM_CATCH
}

int ref_compute_flow(const uint16_t* a, const uint16_t* b, int w, int h, int depth,
                     const froi_params* p, float* u, float* v) {
    SHIM_TRY
    const FlowField f =
        compute_flow(make_frame(a, w, h, depth), make_frame(b, w, h, depth), to_params(p).flow);
    std::memcpy(u, f.u.data(), sizeof(float) * f.size());
    std::memcpy(v, f.v.data(), sizeof(float) * f.size());
    SHIM_CATCH
}

// planes: c, bx, by, a11, a12, a22
int ref_polynomial_expansion(const double* img, int w, int h, int poly_n, double sigma,
                             double* planes) {
    SHIM_TRY
    ImageF im(w, h);
    std::memcpy(im.values.data(), img, sizeof(double) * im.size());
    const PolyExpansion e = polynomial_expansion(im, poly_n, sigma);
    const std::size_t n = im.size();
    std::memcpy(planes + 0 * n, e.c.data(), sizeof(double) * n);
    std::memcpy(planes + 1 * n, e.bx.data(), sizeof(double) * n);
    std::memcpy(planes + 2 * n, e.by.data(), sizeof(double) * n);
    std::memcpy(planes + 3 * n, e.a11.data(), sizeof(double) * n);
    std::memcpy(planes + 4 * n, e.a12.data(), sizeof(double) * n);
    std::memcpy(planes + 5 * n, e.a22.data(), sizeof(double) * n);
    SHIM_CATCH
}

int ref_saliency(const float* u, const float* v, const uint16_t* frame, int w, int h, int depth,
                 double flow_weight, int gradient_source, double* out) {
    SHIM_TRY
    FlowField f(w, h);
    std::memcpy(f.u.data(), u, sizeof(float) * f.size());
    std::memcpy(f.v.data(), v, sizeof(float) * f.size());
    const SaliencyMap s =
        saliency(f, make_frame(frame, w, h, depth), flow_weight,
                 gradient_source == FROI_GRADIENT_FLOW ? SaliencyGradient::flow : SaliencyGradient::image);
    std::memcpy(out, s.values.data(), sizeof(double) * s.size());
    SHIM_CATCH
}

int ref_threshold_mask(const double* map, int w, int h, double t, uint8_t* mask) {
    SHIM_TRY
    SaliencyMap m(w, h);
    std::memcpy(m.values.data(), map, sizeof(double) * m.size());
    const RoiMask r = threshold_mask(m, t);
    std::memcpy(mask, r.bits.data(), r.size());
    SHIM_CATCH
}

int ref_morph_cleanup(uint8_t* mask, int w, int h, int ro, int rc, int min_area) {
    SHIM_TRY
    RoiMask m(w, h);
    std::memcpy(m.bits.data(), mask, m.size());
    const RoiMask r = morph_cleanup(m, ro, rc, min_area);
    std::memcpy(mask, r.bits.data(), r.size());
    SHIM_CATCH
}

// dwt_forward / dwt_inverse (dwt.hpp:113-171), map_mask_to_subbands (codec.hpp:152-171)
int ref_dwt_forward(const uint16_t* px, int w, int h, int depth, int levels, int32_t* out) {
    try {
        Frame f(w, h, depth);
        std::memcpy(f.pixels.data(), px, sizeof(uint16_t) * f.size());
        const SubbandGrid g = dwt_forward(f, levels);
        std::memcpy(out, g.coeffs.data(), sizeof(int32_t) * g.coeffs.size());
        return 0;
    } catch (const usage_error&) {
        return 1;
    } catch (const data_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

int ref_dwt_inverse(const int32_t* coeffs, int w, int h, int depth, int levels, uint16_t* out) {
    try {
        SubbandGrid g;
        g.width = w;
        g.height = h;
        g.levels = levels;
        g.depth = depth;
        g.coeffs.assign(coeffs, coeffs + std::size_t(w) * h);
        const Frame f = dwt_inverse(g);
        std::memcpy(out, f.pixels.data(), sizeof(uint16_t) * f.size());
        return 0;
    } catch (...) {
        return 3;
    }
}

long ref_map_mask_to_subbands(const uint8_t* mask, int w, int h, int levels, uint8_t* out) {
    try {
        RoiMask m(w, h);
        std::memcpy(m.bits.data(), mask, m.size());
        const auto lv = map_mask_to_subbands(m, levels);
        long off = 0;
        for (const auto& r : lv) {
            std::memcpy(out + off, r.bits.data(), r.size());
            off += long(r.size());
        }
        return off;
    } catch (...) {
        return -1;
    }
}

long ref_label_components(const uint8_t* mask, int w, int h, uint32_t* areas, long cap) {
    try {
        RoiMask m(w, h);
        std::memcpy(m.bits.data(), mask, m.size());
        std::vector<std::size_t> a;
        label_components(m, a);
        const long n = long(a.size()) - 1;
        for (long i = 0; i < n && i < cap; ++i) areas[i] = uint32_t(a[std::size_t(i) + 1]);
        return n;
    } catch (...) {
        return -1;
    }
}

int ref_extract_roi(const uint16_t* frames, int n, int w, int h, int depth, const froi_params* p,
                    int workers, uint8_t* masks, froi_shift* shifts, double* raw_fractions,
                    uint64_t* stage_ns) {
    SHIM_TRY
    Sequence seq;
    const std::size_t px = std::size_t(w) * h;
    for (int i = 0; i < n; ++i) seq.push(make_frame(frames + px * std::size_t(i), w, h, depth));
    ExtractInfo info;
    StageTimes times;
    const auto out = extract_roi(seq, to_params(p), workers, &info, &times);
    for (int i = 0; i < n; ++i) std::memcpy(masks + px * std::size_t(i), out[std::size_t(i)].bits.data(), px);
    if (shifts)
        for (int i = 0; i < n; ++i) {
            shifts[i].dx = info.shifts[std::size_t(i)].dx;
            shifts[i].dy = info.shifts[std::size_t(i)].dy;
            shifts[i].confidence = info.shifts[std::size_t(i)].confidence;
        }
    if (raw_fractions)
        for (int i = 0; i < n; ++i) raw_fractions[i] = info.raw_fractions[std::size_t(i)];
    if (stage_ns) {
        stage_ns[0] = times.denoise_ns.load();
        stage_ns[1] = times.flow_ns.load();
        stage_ns[2] = times.roi_ns.load();
        stage_ns[3] = times.encode_ns.load();
    }
    SHIM_CATCH
}

// generate_synthetic (synthetic.hpp:135-290) with the fields the reference tests set.
int ref_generate_synthetic(int n_cells, int n_frames, int w, int h, int depth, double speed_min,
                           double speed_max, double contrast_min, double contrast_max,
                           double low_contrast_fraction, double temporal_noise_sigma,
                           uint64_t seed, uint16_t* frames, uint8_t* truth_masks,
                           double* track_xy, double* radii) {
    SHIM_TRY
    SyntheticSpec s;
    s.n_cells = n_cells;
    s.n_frames = n_frames;
    s.width = w;
    s.height = h;
    s.depth = depth;
    s.speed_min = speed_min;
    s.speed_max = speed_max;
    s.contrast_min = contrast_min;
    s.contrast_max = contrast_max;
    s.low_contrast_fraction = low_contrast_fraction;
    s.temporal_noise_sigma = temporal_noise_sigma;
    s.seed = seed;
    auto [seq, truth] = generate_synthetic(s);
    const std::size_t px = std::size_t(w) * h;
    for (int i = 0; i < n_frames; ++i) {
        std::memcpy(frames + px * std::size_t(i), seq[std::size_t(i)].pixels.data(), sizeof(uint16_t) * px);
        if (truth_masks)
            std::memcpy(truth_masks + px * std::size_t(i), truth.masks[std::size_t(i)].bits.data(), px);
    }
    // track_xy: [cell][frame][x, y]; radii: [cell]
    for (std::size_t c = 0; c < truth.tracks.size(); ++c) {
        if (radii) radii[c] = truth.tracks[c].radius;
        if (track_xy)
            for (int i = 0; i < n_frames; ++i) {
                track_xy[(c * std::size_t(n_frames) + std::size_t(i)) * 2 + 0] = truth.tracks[c].centers[std::size_t(i)].x;
                track_xy[(c * std::size_t(n_frames) + std::size_t(i)) * 2 + 1] = truth.tracks[c].centers[std::size_t(i)].y;
            }
    }
    SHIM_CATCH
}

// flowroi::Rng (rng.hpp:11-62) streams, to pin the Python fixture restatement.
void ref_rng_stream(uint64_t seed, int n, uint64_t* u64_out, double* normal_out) {
    Rng a(seed), b(seed);
    for (int i = 0; i < n; ++i) u64_out[i] = a.next_u64();
    for (int i = 0; i < n; ++i) normal_out[i] = b.normal(0.0, 1.0);
}

}  // extern "C"
