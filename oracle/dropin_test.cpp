// dropin_test.cpp — the reference's own stage next to the drop-in (TEST INFRASTRUCTURE).
//
// Built by `make -C oracle dropin` against the UNMODIFIED reference headers (compiled in place)
// and include/froi/flowroi_gpu.hpp, linked to libfroi.so.  For each case it runs
//   flowroi::extract_roi      (the reference, CPU)
//   flowroi_gpu::extract_roi  (the drop-in, B200)
// on the same Sequence, then feeds both mask sets to the reference encoder
// (flowroi::encode, codec.hpp:227) exactly as compress_sequence does (pipeline.hpp:142-147), and
// prints one JSON object per case: mask mismatch, shift agreement, encoded-bytes agreement.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "flowroi/codec.hpp"
#include "flowroi/roi.hpp"
#include "flowroi/synthetic.hpp"
#include "froi/flowroi_gpu.hpp"
#ifdef FROI_HAVE_JSON
#include "froi/flowroi_gpu_pipeline.hpp"
#endif

using namespace flowroi;

static int run_case(const char* name, int cells, int frames, int size, int depth, std::uint64_t seed,
                    const ExtractParams& params, bool exact = false) {
    flowroi_gpu::set_exact_flow(exact);
    SyntheticSpec spec;
    spec.n_cells = cells;
    spec.n_frames = frames;
    spec.width = spec.height = size;
    spec.depth = depth;
    spec.seed = seed;
    auto [seq, truth] = generate_synthetic(spec);
    ExtractInfo ic, ig;
    StageTimes tc, tg;
    const auto cpu = flowroi::extract_roi(seq, params, 0, &ic, &tc);
    const auto gpu = flowroi_gpu::extract_roi(seq, params, 1, &ig, &tg);
    std::size_t mism = 0, total = 0, frames_equal = 0, bytes_equal = 0, shifts_equal = 0;
    std::size_t enc_bytes = 0;
    for (std::size_t t = 0; t < seq.size(); ++t) {
        std::size_t m = 0;
        for (std::size_t i = 0; i < cpu[t].size(); ++i) m += cpu[t].bits[i] != gpu[t].bits[i];
        mism += m;
        total += cpu[t].size();
        frames_equal += m == 0;
        shifts_equal += ic.shifts[t].dx == ig.shifts[t].dx && ic.shifts[t].dy == ig.shifts[t].dy &&
                        ic.shifts[t].confidence == ig.shifts[t].confidence;
        // the encoder consumes the masks unchanged (pipeline.hpp:144-147)
        const auto ec = encode(seq[t], cpu[t], CodecParams{});
        const auto eg = encode(seq[t], gpu[t], CodecParams{});
        bytes_equal += ec == eg;
        enc_bytes += eg.size();
    }
    std::printf("{\"case\": \"%s\", \"frames\": %zu, \"size\": %d, \"depth\": %d, \"mask_mismatch\": %.3e, "
                "\"frames_identical\": %zu, \"shifts_identical\": %zu, \"encoded_identical\": %zu, "
                "\"encoded_bytes\": %zu, \"gpu_flow_ns\": %llu, \"cpu_flow_ns\": %llu}\n",
                name, seq.size(), size, depth, double(mism) / double(total), frames_equal, shifts_equal,
                bytes_equal, enc_bytes, (unsigned long long)tg.flow_ns.load(),
                (unsigned long long)tc.flow_ns.load());
    flowroi_gpu::set_exact_flow(false);
    // the bit-exact flow mode must reproduce the reference byte for byte, encoder output included
    if (exact) return (mism == 0 && shifts_equal == seq.size() && bytes_equal == seq.size()) ? 0 : 1;
    return (shifts_equal == seq.size() && double(mism) / double(total) <= 1e-4) ? 0 : 1;
}

#ifdef FROI_HAVE_JSON
// compress_sequence (pipeline.hpp:137-153) with the CPU stage vs the pipelined GPU stage: one
// .froi file per frame, identical wherever the masks are identical; shifts identical.
static int run_pipeline_case(const char* name, int cells, int frames, int size, std::uint64_t seed,
                             int adjacent, int chunk) {
    SyntheticSpec spec;
    spec.n_cells = cells;
    spec.n_frames = frames;
    spec.width = spec.height = size;
    spec.seed = seed;
    auto [seq, truth] = generate_synthetic(spec);
    PipelineConfig cfg;
    cfg.workers = 4;
    cfg.roi.adjacent_factor = adjacent;
    const CompressResult cpu = compress_sequence(seq, cfg);
    const CompressResult gpu = flowroi_gpu::compress_sequence(seq, cfg, chunk);
    std::size_t frames_equal = 0, files_equal = 0, shifts_equal = 0, mism = 0, total = 0;
    for (std::size_t t = 0; t < seq.size(); ++t) {
        std::size_t m = 0;
        for (std::size_t i = 0; i < cpu.masks[t].size(); ++i) m += cpu.masks[t].bits[i] != gpu.masks[t].bits[i];
        mism += m;
        total += cpu.masks[t].size();
        frames_equal += m == 0;
        files_equal += cpu.files[t] == gpu.files[t];
        shifts_equal += cpu.info.shifts[t].dx == gpu.info.shifts[t].dx &&
                        cpu.info.shifts[t].dy == gpu.info.shifts[t].dy &&
                        cpu.info.shifts[t].confidence == gpu.info.shifts[t].confidence;
    }
    std::printf("{\"pipeline_case\": \"%s\", \"frames\": %zu, \"chunk\": %d, \"mask_mismatch\": %.3e, "
                "\"frames_identical\": %zu, \"files_identical\": %zu, \"shifts_identical\": %zu, "
                "\"gpu_wall_s\": %.3f, \"cpu_wall_s\": %.3f, \"gpu_encode_ns\": %llu}\n",
                name, seq.size(), chunk, double(mism) / double(total), frames_equal, files_equal, shifts_equal,
                gpu.wall_seconds, cpu.wall_seconds, (unsigned long long)gpu.stages.encode_ns);
    return (shifts_equal == seq.size() && files_equal >= frames_equal && double(mism) / double(total) <= 1e-4) ? 0 : 1;
}
#endif

int main() {
    int bad = 0;
#ifdef FROI_HAVE_JSON
    bad += run_pipeline_case("pipeline-160-chunk4", 5, 11, 160, 31, 0, 4);
    bad += run_pipeline_case("pipeline-128-ensemble", 4, 6, 128, 32, 1, 4);
#endif
    ExtractParams p;
    bad += run_case("synthetic-160", 5, 6, 160, 8, 77, p);
    bad += run_case("synthetic-256-16bit", 8, 4, 256, 16, 12, p);
    ExtractParams q = p;
    q.roi.adjacent_factor = 1;
    q.roi.roi_threshold = 0.1;
    bad += run_case("ensemble-k1", 4, 5, 128, 8, 5, q);
    // the same cases through the bit-exact flow mode (flowroi_gpu::set_exact_flow)
    bad += run_case("exact-synthetic-160", 5, 6, 160, 8, 77, p, true);
    bad += run_case("exact-synthetic-256-16bit", 8, 4, 256, 16, 12, p, true);
    bad += run_case("exact-ensemble-k1", 4, 5, 128, 8, 5, q, true);
    // error taxonomy: usage_error / data_error cross the boundary as the same exception types
    int errors_ok = 0;
    try {
        Sequence one;
        one.push(Frame(64, 64, 8));
        flowroi_gpu::extract_roi(one, p);
    } catch (const data_error&) {
        ++errors_ok;
    }
    try {
        ExtractParams bp;
        bp.roi.roi_threshold = 1.5;
        SyntheticSpec s;
        s.n_frames = 2;
        s.width = s.height = 96;
        auto [seq, truth] = generate_synthetic(s);
        flowroi_gpu::extract_roi(seq, bp);
    } catch (const usage_error&) {
        ++errors_ok;
    }
    std::printf("{\"errors_mapped\": %d}\n", errors_ok);
    return bad + (errors_ok == 2 ? 0 : 1);
}
