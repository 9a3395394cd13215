// flowroi_gpu.hpp — drop-in C++ replacement for the reference's RoI stage entry points.
//
// Same signatures and error behaviour as
//   flowroi::extract_roi   (/root/reference/proj/include/flowroi/roi.hpp:309-364)
//   flowroi::compute_flow  (flow.hpp:304-345)
// over the reference's own value types (Sequence, Frame, RoiMask, FlowField, ExtractParams,
// ExtractInfo, StageTimes from flowroi/core.hpp and flowroi/roi.hpp), implemented on the B200 through
// the C ABI in froi.h (libfroi.so).  Swapping `extract_roi(` for `flowroi_gpu::extract_roi(` at
// pipeline.hpp:142 is the whole integration; the encoder consumes the returned RoiMask unchanged.
//
// Build: -I<reference>/proj/include -I<repo>/include, link -lfroi (paper_2511_14419_b200/_lib).
// Contexts (device arenas) are cached per thread, keyed by device, geometry and parameters.
#pragma once

#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "flowroi/roi.hpp"
#include "froi/froi.h"

namespace flowroi_gpu {

using flowroi::data_error;
using flowroi::usage_error;

inline void check(int status, const char* what) {
    if (status == FROI_OK) return;
    const std::string msg = std::string(what) + ": " + froi_last_error();
    if (status == FROI_ERR_USAGE) throw usage_error(msg);
    if (status == FROI_ERR_DATA) throw data_error(msg);
    throw std::runtime_error(msg);  // internal / CUDA: exit code 3 in the CLI taxonomy
}

inline froi_params to_c(const flowroi::ExtractParams& e) {
    froi_params p;
    p.denoise_enabled = e.denoise.enabled ? 1 : 0;
    p.median_radius = e.denoise.median_radius;
    p.bilateral_sigma_spatial = e.denoise.bilateral_sigma_spatial;
    p.bilateral_sigma_range = e.denoise.bilateral_sigma_range;
    p.bilateral_radius = e.denoise.bilateral_radius;
    p.pyramid_levels = e.flow.pyramid_levels;
    p.pyramid_scale = e.flow.pyramid_scale;
    p.window_size = e.flow.window_size;
    p.iterations = e.flow.iterations;
    p.poly_n = e.flow.poly_n;
    p.poly_sigma = e.flow.poly_sigma;
    p.roi_threshold = e.roi.roi_threshold;
    p.flow_weight = e.roi.flow_weight;
    p.adjacent_factor = e.roi.adjacent_factor;
    p.min_area = e.roi.min_area;
    p.open_radius = e.roi.open_radius;
    p.close_radius = e.roi.close_radius;
    p.gradient_source = e.roi.gradient_source == flowroi::SaliencyGradient::flow ? FROI_GRADIENT_FLOW
                                                                                 : FROI_GRADIENT_IMAGE;
    p.max_shift = e.max_shift;
    return p;
}

namespace detail {

struct CtxDeleter {
    void operator()(froi_ctx* c) const { froi_ctx_destroy(c); }
};

inline bool& exact_flag() {
    thread_local bool on = false;
    return on;
}

// Thread-affine context cache (froi contexts are not internally locked).
inline froi_ctx* context(int device, const froi_params& p, int w, int h, int depth) {
    thread_local std::map<std::string, std::unique_ptr<froi_ctx, CtxDeleter>> cache;
    const bool exact = exact_flag();
    std::string key(reinterpret_cast<const char*>(&p), sizeof(p));
    key += std::to_string(device) + ":" + std::to_string(w) + "x" + std::to_string(h) + ":" +
           std::to_string(depth) + (exact ? ":exact" : "");
    auto it = cache.find(key);
    if (it != cache.end()) return it->second.get();
    froi_ctx* c = nullptr;
    check(froi_ctx_create(device, &p, w, h, depth, 0, &c), "froi_ctx_create");
    std::unique_ptr<froi_ctx, CtxDeleter> owned(c);
    if (exact) check(froi_ctx_set_flow_exact(c, 1), "froi_ctx_set_flow_exact");
    cache.emplace(key, std::move(owned));
    return c;
}

// n empty-initialised masks, constructed by several threads: a RoiMask zero-fills W*H fresh bytes
// (core.hpp:84-85), which single-threaded costs about as much as the GPU work of a pair.
inline std::vector<flowroi::RoiMask> make_masks(std::size_t n, int w, int h) {
    std::vector<flowroi::RoiMask> m(n);
    const unsigned hw = std::thread::hardware_concurrency();
    const std::size_t T = std::max<std::size_t>(1, std::min<std::size_t>({8, hw ? hw : 1, n}));
    std::vector<std::thread> th;
    for (std::size_t k = 1; k < T; ++k)
        th.emplace_back([&m, k, T, w, h] {
            for (std::size_t t = k; t < m.size(); t += T) m[t] = flowroi::RoiMask(w, h);
        });
    for (std::size_t t = 0; t < m.size(); t += T) m[t] = flowroi::RoiMask(w, h);
    for (auto& x : th) x.join();
    return m;
}

}  // namespace detail

// Opt in (for calls made from this thread) to the bit-exact fp64 flow (froi_ctx_set_flow_exact):
// flows and masks byte-identical to the reference's instead of within the fp32 flow tolerance,
// at about a third of the throughput.  Off by default.
inline void set_exact_flow(bool on) { detail::exact_flag() = on; }

// flowroi::extract_roi on the GPU.  `workers` keeps the reference signature: outputs never
// depend on it (parallel.hpp:17-19); a single sequence runs on one device (device 0).
inline std::vector<flowroi::RoiMask> extract_roi(const flowroi::Sequence& seq,
                                                 const flowroi::ExtractParams& params,
                                                 int workers = 1,
                                                 flowroi::ExtractInfo* info = nullptr,
                                                 flowroi::StageTimes* timers = nullptr) {
    (void)workers;
    params.roi.validate();
    params.flow.validate();
    const std::size_t n = seq.size();
    if (n < 2) throw data_error("extract_roi: sequence needs at least 2 frames");
    params.denoise.validate();
    const froi_params cp = to_c(params);
    const flowroi::Frame& f0 = seq[0];
    froi_ctx* ctx = detail::context(0, cp, f0.width, f0.height, f0.depth);
    // the Frames and RoiMasks go to the library as they are: one pointer each, uint16 samples
    // (narrowed to bytes for 8-bit frames by the library's host threads on the way into its
    // pinned staging ring), masks unpacked from the returned PBM rows straight into RoiMask::bits
    std::vector<const void*> fp(n);
    for (std::size_t t = 0; t < n; ++t) {
        if (!seq[t].same_shape(f0)) throw data_error("sequence frames must share dimensions and depth");
        fp[t] = seq[t].pixels.data();
    }
    // each RoiMask is built by the library's host threads from its finished bytes in one pass
    // (std::vector::assign: no zero-fill, core.hpp:84-85), while the GPU works on later pairs
    std::vector<flowroi::RoiMask> masks(n);
    struct Put {
        std::vector<flowroi::RoiMask>* m;
        int w, h;
        // called from the library's host threads: must not throw across the C ABI
        static int at(void* u, int, int t, const uint8_t* bytes) noexcept {
            Put* p = static_cast<Put*>(u);
            try {
                flowroi::RoiMask& r = (*p->m)[static_cast<std::size_t>(t)];
                r.width = p->w;
                r.height = p->h;
                r.bits.assign(bytes, bytes + static_cast<std::size_t>(p->w) * p->h);
                return 0;
            } catch (...) {
                return 1;
            }
        }
    } put{&masks, f0.width, f0.height};
    std::vector<froi_frame_stats> stats(n);
    check(froi_extract_frames_put(ctx, fp.data(), 2, static_cast<int>(n), FROI_MASK_BYTES, &Put::at, &put,
                                  stats.data()),
          "extract_roi");
    if (info) {
        info->shifts.resize(n);
        info->raw_fractions.resize(n);
        for (std::size_t t = 0; t < n; ++t) {
            info->shifts[t] = flowroi::Shift{stats[t].dx, stats[t].dy, stats[t].confidence};
            info->raw_fractions[t] = stats[t].raw_fraction;
        }
    }
    if (timers) {
        froi_stage_times st;
        check(froi_ctx_stage_times(ctx, &st), "stage_times");
        timers->denoise_ns += st.denoise_ns;
        timers->flow_ns += st.flow_ns;
        timers->roi_ns += st.roi_ns;
    }
    return masks;
}

// flowroi::compute_flow on the GPU (fp32 flow; see DESIGN.md for the tolerance).
inline flowroi::FlowField compute_flow(const flowroi::Frame& prev, const flowroi::Frame& next,
                                       const flowroi::FlowParams& fp) {
    fp.validate();
    if (!prev.same_shape(next)) throw data_error("compute_flow: frames must share dimensions");
    flowroi::ExtractParams e;
    e.flow = fp;
    e.max_shift = std::max(1, std::min(e.max_shift, std::min(prev.width, prev.height) / 4 - 1));
    froi_ctx* ctx = detail::context(0, to_c(e), prev.width, prev.height, prev.depth);
    flowroi::FlowField out(prev.width, prev.height);
    check(froi_compute_flow(ctx, prev.pixels.data(), next.pixels.data(), out.u.data(), out.v.data()),
          "compute_flow");
    return out;
}

}  // namespace flowroi_gpu
