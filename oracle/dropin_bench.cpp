// dropin_bench.cpp — times the reference-type drop-in (BENCH TOOL, built like dropin_test.cpp).
//
// flowroi_gpu::extract_roi (include/froi/flowroi_gpu.hpp) over the reference's own value types:
// a Sequence of separately allocated uint16 Frames in, a std::vector<RoiMask> of byte masks out —
// the call compress_sequence makes (pipeline.hpp:142) — on one C3 well whose u8 samples bench.py
// writes to a raw file.  Timed on the host clock: the call is synchronous, and everything it
// does (mask construction, u16 -> u8 narrowing, H2D, GPU work, D2H, PBM -> byte unpacking) is the
// cost a reference user pays.  Prints one JSON line.
//
//   dropin_bench RAW W H FRAMES STEPS WARMUP
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "flowroi/roi.hpp"
#include "froi/flowroi_gpu.hpp"

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: %s RAW W H FRAMES STEPS WARMUP\n", argv[0]);
        return 2;
    }
    const int W = std::atoi(argv[2]), H = std::atoi(argv[3]), F = std::atoi(argv[4]);
    const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
    std::FILE* f = std::fopen(argv[1], "rb");
    if (!f) {
        std::perror(argv[1]);
        return 2;
    }
    const std::size_t px = (std::size_t)W * H;
    std::vector<std::uint8_t> raw(px * F);
    if (std::fread(raw.data(), 1, raw.size(), f) != raw.size()) {
        std::fprintf(stderr, "short read\n");
        return 2;
    }
    std::fclose(f);
    flowroi::Sequence seq;
    for (int t = 0; t < F; ++t) {
        flowroi::Frame fr(W, H, 8);
        for (std::size_t i = 0; i < px; ++i) fr.pixels[i] = raw[px * t + i];
        seq.push(std::move(fr));
    }
    flowroi::ExtractParams params;
    std::size_t set = 0;
    double secs = 0.0;
    try {
        for (int i = 0; i < warmup + steps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            flowroi::ExtractInfo info;
            const std::vector<flowroi::RoiMask> masks = flowroi_gpu::extract_roi(seq, params, 1, &info);
            const auto t1 = std::chrono::steady_clock::now();
            if (i >= warmup) secs += std::chrono::duration<double>(t1 - t0).count();
            set = 0;
            for (const auto& m : masks) set += m.count();  // after the clock: a consumer's read
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_bench: %s\n", e.what());
        return 3;
    }
    std::printf("{\"dropin_frames_per_s\": %.3f, \"ms_per_step\": %.3f, \"frames\": %d, \"steps\": %d, "
                "\"mask_pixels\": %zu}\n",
                double(F) * steps / secs, 1e3 * secs / steps, F, steps, set);
    return 0;
}
