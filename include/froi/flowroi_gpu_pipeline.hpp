// flowroi_gpu_pipeline.hpp — the reference's compression run with the B200 RoI stage.
//
// flowroi_gpu::compress_sequence has the contract of flowroi::compress_sequence
// (/root/reference/proj/include/flowroi/pipeline.hpp:137-153): same CompressResult (one .froi
// file per frame from the reference encoder, flowroi::encode, codec.hpp:227; the masks;
// ExtractInfo; per-stage nanoseconds), same validation and exceptions, and files byte-identical
// to the CPU run wherever the masks are identical.  The masks come from the B200 in chunks through
// the streaming ABI (froi_stream_push) while CPU worker threads encode the frames of the chunks
// already returned, so mask production and encoding overlap.  With the
// temporal ensemble on (adjacent_factor > 0) the masks need look-ahead: the whole sequence is
// extracted first, then encoded in parallel, as the reference does.
//
// Build: -I<reference>/proj/include -I<json.hpp dir> -I<repo>/include, link -lfroi.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "flowroi/pipeline.hpp"
#include "froi/flowroi_gpu.hpp"

namespace flowroi_gpu {

namespace detail {

// Frame indices handed to `workers` encoder threads as the GPU returns them.
class EncodePool {
public:
    EncodePool(int workers, const flowroi::Sequence& seq, flowroi::CompressResult& res,
               const flowroi::CodecParams& codec)
        : seq_(seq), res_(res), codec_(codec) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { run(); });
    }
    ~EncodePool() { finish(); }
    void submit(std::size_t first, std::size_t count) {
        {
            std::lock_guard<std::mutex> lk(m_);
            for (std::size_t i = first; i < first + count; ++i) q_.push_back(i);
        }
        cv_.notify_all();
    }
    // Waits for every submitted frame; rethrows the first encoder exception.
    void finish() {
        {
            std::lock_guard<std::mutex> lk(m_);
            closed_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_)
            if (t.joinable()) t.join();
        threads_.clear();
        if (error_) {
            auto e = error_;
            error_ = nullptr;
            std::rethrow_exception(e);
        }
    }
    std::uint64_t encode_ns() const { return encode_ns_.load(); }

private:
    void run() {
        for (;;) {
            std::size_t i;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [this] { return closed_ || !q_.empty(); });
                if (q_.empty()) return;
                i = q_.front();
                q_.pop_front();
            }
            try {
                const auto t0 = std::chrono::steady_clock::now();
                res_.files[i] = flowroi::encode(seq_[i], res_.masks[i], codec_);
                encode_ns_ += (std::uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - t0)
                                  .count();
            } catch (...) {
                std::lock_guard<std::mutex> lk(m_);
                if (!error_) error_ = std::current_exception();
            }
        }
    }
    const flowroi::Sequence& seq_;
    flowroi::CompressResult& res_;
    const flowroi::CodecParams& codec_;
    std::vector<std::thread> threads_;
    std::deque<std::size_t> q_;
    std::mutex m_;
    std::condition_variable cv_;
    bool closed_ = false;
    std::exception_ptr error_;
    std::atomic<std::uint64_t> encode_ns_{0};
};

inline int encode_workers(int workers) {
    if (workers > 0) return workers;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? (int)hw : 1;
}

}  // namespace detail

inline flowroi::CompressResult compress_sequence(const flowroi::Sequence& seq,
                                                 const flowroi::PipelineConfig& config,
                                                 int chunk = 32) {
    config.validate();
    const auto t0 = std::chrono::steady_clock::now();
    flowroi::CompressResult res;
    const flowroi::ExtractParams params = config.extract_params();
    params.roi.validate();
    params.flow.validate();
    const std::size_t n = seq.size();
    if (n < 2) throw data_error("extract_roi: sequence needs at least 2 frames");
    params.denoise.validate();
    res.files.resize(n);
    std::uint64_t denoise_ns = 0, flow_ns = 0, roi_ns = 0;
    if (params.roi.adjacent_factor != 0) {
        flowroi::StageTimes timers;
        res.masks = flowroi_gpu::extract_roi(seq, params, config.workers, &res.info, &timers);
        detail::EncodePool pool(detail::encode_workers(config.workers), seq, res, config.codec);
        pool.submit(0, n);
        pool.finish();
        res.stages = {timers.denoise_ns.load(), timers.flow_ns.load(), timers.roi_ns.load(),
                      pool.encode_ns()};
    } else {
        const flowroi::Frame& f0 = seq[0];
        froi_ctx* ctx = detail::context(0, to_c(params), f0.width, f0.height, f0.depth);
        chunk = std::max(2, chunk);
        res.masks = detail::make_masks(n, f0.width, f0.height);
        res.info.shifts.resize(n);
        res.info.raw_fractions.resize(n);
        // Frames and RoiMasks are handed over by pointer (no packing or copying here)
        std::vector<const void*> fp(n);
        std::vector<uint8_t*> mp(n);
        for (std::size_t t = 0; t < n; ++t) {
            if (!seq[t].same_shape(f0)) throw data_error("sequence frames must share dimensions and depth");
            fp[t] = seq[t].pixels.data();
            mp[t] = res.masks[t].bits.data();
        }
        std::vector<froi_frame_stats> stats((std::size_t)chunk);
        detail::EncodePool pool(detail::encode_workers(config.workers), seq, res, config.codec);
        check(froi_stream_reset(ctx, 1), "compress_sequence");
        for (std::size_t a = 0; a < n; a += (std::size_t)chunk) {
            const int k = (int)std::min<std::size_t>((std::size_t)chunk, n - a);
            check(froi_stream_push_frames(ctx, fp.data() + a, 2, k, FROI_MASK_BYTES, mp.data() + a, stats.data()),
                  "compress_sequence");
            for (int t = 0; t < k; ++t) {
                res.info.shifts[a + t] = flowroi::Shift{stats[t].dx, stats[t].dy, stats[t].confidence};
                res.info.raw_fractions[a + t] = stats[t].raw_fraction;
            }
            froi_stage_times st;
            check(froi_ctx_stage_times(ctx, &st), "stage_times");
            denoise_ns += st.denoise_ns;
            flow_ns += st.flow_ns;
            roi_ns += st.roi_ns;
            pool.submit(a, (std::size_t)k);  // encoded while the GPU works on the next chunk
        }
        pool.finish();
        res.stages = {denoise_ns, flow_ns, roi_ns, pool.encode_ns()};
    }
    res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return res;
}

}  // namespace flowroi_gpu
