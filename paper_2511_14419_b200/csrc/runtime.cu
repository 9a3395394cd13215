// runtime.cu — per-GPU context, batch scheduler and the C ABI (include/froi/froi.h).
//
// A context owns one CUDA stream and fixed device arenas sized for `Pcap` adjacent pairs per
// batch (frame slots: raw, denoised, spectrum, pyramid + expansions; pair slots: registration
// scratch, shifted expansions, flow ping-pong, mask-stage scratch).  extract_* calls split the
// work into batches of pairs (pairs of one well are independent once their frames are denoised,
// roi.hpp:325), launch every stage for the whole batch at once (grid.z = slot), and gather
// packed masks + per-pair stats.  Host tables are double-buffered in pinned memory.
//
// Host-side constants that must match the reference bit for bit (bilateral LUT and spatial
// weights, Hann windows, FFT twiddle recurrence) are computed here with the same libm calls and
// expression order as the reference; this file is compiled with -ffp-contract=off.
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>
#include <array>
#include <vector>

#include <chrono>
#include <map>
#include <memory>
#include <thread>
#include <tuple>

#include "../../include/froi/froi.h"
#include "host_pool.hpp"
#include "kernels.cuh"

using namespace froi;

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

#define ABI_TRY try {
#define ABI_CATCH                                   \
    }                                               \
    catch (const froi::Error& e) {                  \
        return fail(e.status, e.what());            \
    }                                               \
    catch (const std::bad_alloc&) {                 \
        return fail(3, "host allocation failed");   \
    }                                               \
    catch (const std::exception& e) {               \
        return fail(3, e.what());                   \
    }                                               \
    return 0;

constexpr double kPi = 3.14159265358979323846;

int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}
int ilog2(int n) {
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}

std::string validate(const froi_params* p) {
    if (!p) return "params must not be null";
    // RoiParams::validate (roi.hpp:29-37)
    if (!(p->roi_threshold > 0.0 && p->roi_threshold < 1.0)) return "roi: roi_threshold must be in (0,1)";
    if (p->flow_weight < 0.0 || p->flow_weight > 1.0) return "roi: flow_weight must be in [0,1]";
    if (p->adjacent_factor < 0) return "roi: adjacent_factor must be >= 0";
    if (p->min_area < 0) return "roi: min_area must be >= 0";
    if (p->open_radius < 0 || p->close_radius < 0) return "roi: radii must be >= 0";
    // FlowParams::validate (flow.hpp:20-29)
    if (p->pyramid_levels < 1) return "flow: pyramid_levels must be >= 1";
    if (!(p->pyramid_scale > 0.0 && p->pyramid_scale < 1.0)) return "flow: pyramid_scale must be in (0,1)";
    if (p->window_size < 3 || p->window_size % 2 == 0) return "flow: window_size must be odd and >= 3";
    if (p->poly_n < 3 || p->poly_n % 2 == 0) return "flow: poly_n must be odd and >= 3";
    if (p->iterations < 1) return "flow: iterations must be >= 1";
    if (p->poly_sigma <= 0.0) return "flow: poly_sigma must be > 0";
    // DenoiseParams::validate (denoise.hpp:18-23)
    if (p->median_radius < 1 || p->bilateral_radius < 1) return "denoise: radii must be >= 1";
    if (p->bilateral_sigma_spatial <= 0 || p->bilateral_sigma_range <= 0) return "denoise: sigmas must be > 0";
    if (p->gradient_source != FROI_GRADIENT_IMAGE && p->gradient_source != FROI_GRADIENT_FLOW)
        return "roi: unknown gradient_source";
    // limits of this implementation's shared-memory tiles
    if (p->poly_n > 15) return "flow: poly_n > 15 is not supported by the GPU kernels";
    if (p->window_size > 15) return "flow: window_size > 15 is not supported by the GPU kernels";
    if (p->median_radius > 3) return "denoise: median_radius > 3 is not supported by the GPU kernels";
    if (p->bilateral_radius > 7) return "denoise: bilateral_radius > 7 is not supported by the GPU kernels";
    if (p->open_radius > 31 || p->close_radius > 31) return "roi: radii > 31 are not supported by the GPU kernels";
    return "";
}

// Levels build_pyramid (flow.hpp:289-298) would make, without this implementation's cap.
int pyramid_levels_uncapped(const froi_params& p, int W, int H) {
    int L = 1;
    for (int l = 1, w = W, h = H; l < p.pyramid_levels; ++l) {
        const int tw = int(w * p.pyramid_scale), th = int(h * p.pyramid_scale);
        if (tw < 32 || th < 32) break;
        w = tw;
        h = th;
        L = l + 1;
    }
    return L;
}

// "" or the usage error for a geometry the GPU tables cannot hold (never a silent cap)
std::string check_geometry(const froi_params& p, int W, int H) {
    if (pyramid_levels_uncapped(p, W, H) > kMaxLevels)
        return "flow: this pyramid_levels / pyramid_scale would build more than " +
               std::to_string(kMaxLevels) + " levels, which the GPU kernels do not support";
    return "";
}

Geom make_geom(const froi_params& p, int W, int H, int depth) {
    Geom g{};
    g.W = W;
    g.H = H;
    g.depth = depth;
    g.maxval = (1 << depth) - 1;
    g.sample_bytes = depth == 8 ? 1 : 2;
    // build_pyramid (flow.hpp:289-298)
    g.lw[0] = W;
    g.lh[0] = H;
    g.L = 1;
    for (int l = 1; l < p.pyramid_levels && l < kMaxLevels; ++l) {
        const int tw = int(g.lw[l - 1] * p.pyramid_scale), th = int(g.lh[l - 1] * p.pyramid_scale);
        if (tw < 32 || th < 32) break;
        g.lw[l] = tw;
        g.lh[l] = th;
        g.L = l + 1;
    }
    long long off = 0;
    for (int l = 0; l < g.L; ++l) {
        g.loff[l] = off;
        off += (long long)g.lw[l] * g.lh[l];
        off = (off + 3) & ~3LL;  // keep float4 rows of the next level 16-byte aligned
    }
    if (g.L == 1) g.loff[1] = off;
    else for (int l = g.L; l < kMaxLevels; ++l) g.loff[l] = off;
    g.lsum = off;
    g.pw = next_pow2(W);
    g.ph = next_pow2(H);
    g.log2pw = ilog2(g.pw);
    g.log2ph = ilog2(g.ph);
    g.WW = (W + 31) / 32;
    g.SB = (W + 7) / 8;
    g.RMAX = (W + 1) / 2;
    return g;
}

DevParams make_dev_params(const froi_params& p) {
    DevParams d{};
    d.denoise_enabled = p.denoise_enabled ? 1 : 0;
    d.median_radius = p.median_radius;
    d.bilateral_radius = p.bilateral_radius;
    d.window_radius = (p.window_size - 1) / 2;
    d.iterations = p.iterations;
    d.poly_radius = (p.poly_n - 1) / 2;
    // polynomial_expansion kernels and expansion_moments (flow.hpp:92-127), fp64 then float
    const int r = d.poly_radius;
    std::vector<double> g0(p.poly_n), g1(p.poly_n), g2(p.poly_n);
    for (int t = -r; t <= r; ++t) {
        const double w = std::exp(-double(t) * t / (2.0 * p.poly_sigma * p.poly_sigma));
        g0[t + r] = w;
        g1[t + r] = w * t;
        g2[t + r] = w * t * t;
    }
    double s0 = 0, s2 = 0, s4 = 0;
    for (int t = -r; t <= r; ++t) {
        const double w = g0[t + r];
        s0 += w;
        s2 += w * t * t;
        s4 += w * t * t * t * t;
    }
    const double m00 = s0 * s0, m20 = s2 * s0, m40 = s4 * s0, m22 = s2 * s2;
    const double det = m00 * (m40 * m40 - m22 * m22) - m20 * (m20 * m40 - m22 * m20) +
                       m20 * (m20 * m22 - m40 * m20);
    d.poly_moments[0] = float(1.0 / m20);
    d.poly_moments[1] = float(1.0 / m22);
    d.poly_moments[2] = float((m40 * m40 - m22 * m22) / det);
    d.poly_moments[3] = float((m20 * m22 - m20 * m40) / det);
    d.poly_moments[4] = float((m00 * m40 - m20 * m20) / det);
    d.poly_moments[5] = float((m20 * m20 - m00 * m22) / det);
    for (int i = 0; i < p.poly_n; ++i) {
        d.g0[i] = float(g0[i]);
        d.g1[i] = float(g1[i]);
        d.g2[i] = float(g2[i]);
    }
    // gaussian_blur3(., 1.0) (flow.hpp:259-272): radius max(1, ceil(2.5)) = 3
    double k[7], sum = 0.0;
    for (int t = -3; t <= 3; ++t) {
        k[t + 3] = std::exp(-double(t) * t / (2.0 * 1.0 * 1.0));
        sum += k[t + 3];
    }
    for (int i = 0; i < 7; ++i) d.blur[i] = float(k[i] / sum);
    d.pyr_scale = p.pyramid_scale;
    d.roi_threshold = p.roi_threshold;
    d.flow_weight = p.flow_weight;
    d.min_area = p.min_area;
    d.open_radius = p.open_radius;
    d.close_radius = p.close_radius;
    d.gradient_source = p.gradient_source;
    d.max_shift = p.max_shift;
    return d;
}

// The bit-exact flow's constants (k_flow64.cu): the same host expressions as make_dev_params,
// kept in double (polynomial_expansion flow.hpp:118-127, expansion_moments :92-112,
// gaussian_blur3 :259-266).
Flow64Const make_flow64_const(const froi_params& p) {
    Flow64Const c{};
    const int r = (p.poly_n - 1) / 2;
    c.poly_r = r;
    for (int t = -r; t <= r; ++t) {
        const double w = std::exp(-double(t) * t / (2.0 * p.poly_sigma * p.poly_sigma));
        c.g0[t + r] = w;
        c.g1[t + r] = w * t;
        c.g2[t + r] = w * t * t;
    }
    double s0 = 0, s2 = 0, s4 = 0;
    for (int t = -r; t <= r; ++t) {
        const double w = c.g0[t + r];
        s0 += w;
        s2 += w * t * t;
        s4 += w * t * t * t * t;
    }
    const double m00 = s0 * s0, m20 = s2 * s0, m40 = s4 * s0, m22 = s2 * s2;
    const double det = m00 * (m40 * m40 - m22 * m22) - m20 * (m20 * m40 - m22 * m20) +
                       m20 * (m20 * m22 - m40 * m20);
    c.inv_m20 = 1.0 / m20;
    c.inv_m22 = 1.0 / m22;
    c.i01 = (m20 * m22 - m20 * m40) / det;
    c.i11 = (m00 * m40 - m20 * m20) / det;
    c.i12 = (m20 * m20 - m00 * m22) / det;
    const double sigma = 1.0;
    const int br = std::max(1, int(std::ceil(2.5 * sigma)));
    c.blur_r = br;
    double sum = 0.0;
    for (int t = -br; t <= br; ++t) {
        c.blur[t + br] = std::exp(-double(t) * t / (2.0 * sigma * sigma));
        sum += c.blur[t + br];
    }
    for (int i = 0; i < 2 * br + 1; ++i) c.blur[i] /= sum;
    return c;
}

// fft_inplace twiddle sequence (fft.hpp:27-37): stage len = 2h stores w_0..w_{h-1} at [h-1, 2h-2]
std::vector<double2> twiddles(int n, bool inverse) {
    std::vector<double2> tw(n > 1 ? n - 1 : 1);
    for (int len = 2; len <= n; len <<= 1) {
        const double ang = (inverse ? 2.0 : -2.0) * kPi / len;
        const double wr = std::cos(ang), wi = std::sin(ang);
        double cr = 1.0, ci = 0.0;
        for (int k = 0; k < len / 2; ++k) {
            tw[len / 2 - 1 + k] = make_double2(cr, ci);
            const double nr = cr * wr - ci * wi;  // std::complex product without FMA
            const double ni = cr * wi + ci * wr;
            cr = nr;
            ci = ni;
        }
    }
    return tw;
}

template <typename T>
T* dalloc(size_t count, size_t* total) {
    void* p = nullptr;
    const size_t bytes = count * sizeof(T);
    FROI_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    *total += bytes;
    return (T*)p;
}

}  // namespace

#ifndef FROI_PCAP_MAX
#define FROI_PCAP_MAX 64
#endif

static bool default_fork() {
    const char* e = getenv("FROI_FORK");
    return !(e && atoi(e) == 0);
}

static bool default_graphs() {
    const char* e = getenv("FROI_GRAPHS");
    return !(e && atoi(e) == 0);
}

static int default_lanes() {
    const char* e = getenv("FROI_LANES");
    return (e && atoi(e) == 1) ? 1 : 2;
}

struct froi_ctx {
    int device = 0;
    froi_params params{};
    Geom g{};
    DevParams dp{};
    cudaStream_t stream = nullptr;
    int Pcap = 0, Fcap = 0;
    size_t frame_bytes = 0;  // W*H*sample_bytes
    size_t device_bytes = 0;
    // constants
    double *d_spatial = nullptr, *d_lut = nullptr, *d_wx = nullptr, *d_wy = nullptr;
    float* d_norm_lut = nullptr;
    unsigned short* d_grad_map = nullptr;  // 8-bit frames: |grad I| table (DevParams::grad_*)
    double* d_grad_tab = nullptr;
    int grad_nv = 0;
    std::vector<double> h_spatial;
    double2 *d_tw_row = nullptr, *d_tw_col = nullptr, *d_itw_row = nullptr, *d_itw_col = nullptr;
    // frame slots
    uint8_t* d_raw = nullptr;
    uint8_t* d_den = nullptr;
    unsigned long long* d_sums = nullptr;
    double2* d_spec = nullptr;
    float* d_pyr_f = nullptr;
    float4* d_exA_f = nullptr;
    float* d_exB_f = nullptr;
    // pair slots
    PairInfo* d_info = nullptr;
    double2* d_cols = nullptr;
    double* d_surf = nullptr;
    float* d_pyr_p = nullptr;
    float4* d_exA_p = nullptr;
    float* d_exB_p = nullptr;
    float2* d_flow0 = nullptr;
    float2* d_flow1 = nullptr;
    SelState* d_sel = nullptr;
    unsigned int* d_hist = nullptr;
    unsigned long long* d_cand = nullptr;
    unsigned int* d_cand_count = nullptr;
    unsigned int* d_cand_idx = nullptr;
    float* d_fm = nullptr;
    double* d_gr = nullptr;
    unsigned long long* d_tie = nullptr;
    uint32_t *d_bits_thr = nullptr, *d_bits_clean = nullptr, *d_bits_keep = nullptr;
    uint16_t *d_run_x0 = nullptr, *d_run_x1 = nullptr;
    int *d_run_n = nullptr, *d_run_par = nullptr;
    unsigned int* d_run_area = nullptr;
    uint8_t* d_out_batch = nullptr;  // [Pcap] PBM masks for taps
    // tables (device + pinned host, double-buffered)
    const void** d_frame_raw[2] = {nullptr, nullptr};
    int* d_prev[2] = {nullptr, nullptr};
    int* d_next[2] = {nullptr, nullptr};
    const void** d_pair_raw[2] = {nullptr, nullptr};
    long long* d_out_index[2] = {nullptr, nullptr};
    void* h_tables[2] = {nullptr, nullptr};
    size_t tables_bytes = 0;
    cudaEvent_t tables_free[2] = {nullptr, nullptr};
    int tb = 0;
    // second execution lane (own buffers and stream, same constants): batches of one call
    // alternate between the lanes so one lane's kernels fill the other's tails and small launches
    froi_ctx* lane = nullptr;
    int lanes = default_lanes();
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    PairInfo* h_info = nullptr;  // pinned, one entry per pair of the current call
    size_t h_info_cap = 0;
    std::vector<std::array<cudaEvent_t, 8>> bev;  // stage events of each batch of a call
    // sequence-level output buffer (PBM) for host outputs
    uint8_t* d_seq_out = nullptr;
    size_t seq_out_cap = 0;
    uint8_t* d_seq_tmp = nullptr;
    size_t seq_tmp_cap = 0;
    // streaming state
    int stream_wells = 0;
    std::vector<long long> stream_next_t;  // next frame index per well
    uint8_t* d_carry[2] = {nullptr, nullptr};  // last raw frame per well (current / next push)
    int carry_cur = 0;
    size_t carry_cap = 0;
    // timing
    cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    froi_stage_times times{};
    froi_kernel_times ktimes{};
    // host ingest / egress pipeline (run_host_call): bounded rings, whatever the call size
    std::unique_ptr<HostPool> pool;      // frame conversion into staging, mask unpacking
    std::unique_ptr<HostPool> courier;   // one thread: waits for each batch, then delivers it
    std::unique_ptr<HostPool> dpool;     // mask delivery threads (unpacking), apart from conversion
    uint8_t* d_ring = nullptr;           // ingest ring: ring_frames device frame slots
    int ring_chunk = 0, ring_frames = 0; // upload chunk (frames) and ring size (frames)
    uint8_t* h_stage = nullptr;          // pinned staging ring: kStageChunks chunks
    std::vector<cudaEvent_t> stage_free; // staging chunk i may be refilled
    uint8_t* d_outring = nullptr;        // egress ring: kOutBatches x Pcap PBM masks
    uint8_t* h_outring = nullptr;        // pinned twin of d_outring (general destinations)
    std::vector<cudaEvent_t> delivered;  // per batch of a call: its masks are in host memory
    cudaStream_t copy_stream = nullptr;
    // intra-batch fork: the frame expansions (HBM-bound) run on `side` while the forward FFT and
    // registration (fp64-bound) run on the batch's stream; both branches live in the batch graph
    cudaStream_t side = nullptr;
    cudaEvent_t ev_den = nullptr, ev_exp = nullptr;
    bool fork = default_fork();
    cudaStream_t d2h_stream = nullptr;       // per-batch mask read-back (host PBM), off the lanes
    std::vector<cudaEvent_t> d2h_ev;         // batch b's masks are final
    cudaEvent_t d2h_done = nullptr;
    std::vector<cudaEvent_t> chunk_ready;  // per upload chunk of a call
    uint64_t launches = 0;
    // CUDA graphs of a batch's kernel sequence, one per (table buffer, pairs, frame slots, output):
    // captured on first use, replayed with this batch's stage events swapped into its 8 event nodes
    struct BatchGraph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t ev_node[8] = {};
        uint64_t launches = 0;
    };
    std::map<std::tuple<int, int, int, const void*>, BatchGraph> graphs;
    bool use_graphs = default_graphs();

    // bit-exact fp64 flow (froi_ctx_set_flow_exact): its constants and buffers, allocated on first use
    bool flow_exact = false;
    Flow64Const f64c{};
    double *d64_img_f = nullptr, *d64_ex_f = nullptr, *d64_img_p = nullptr, *d64_ex_p = nullptr;
    double *d64_prod = nullptr, *d64_rowm = nullptr;

    Flow64Buffers flow64_buffers() const {
        Flow64Buffers b;
        b.img_f = d64_img_f;
        b.ex_f = d64_ex_f;
        b.tmp_f = d64_prod;  // the frame expansions' row blur runs before the flow needs prod
        b.img_p = d64_img_p;
        b.ex_p = d64_ex_p;
        b.tmp_p = d64_rowm;  // (the shifted expansions may overlap them on the other branch)
        b.prod = d64_prod;
        b.rowm = d64_rowm;
        b.flow0 = d_flow0;
        b.flow1 = d_flow1;
        return b;
    }
    MaskBuffers mask_buffers(int tb_) const {
        MaskBuffers b;
        b.flow = nullptr;
        b.flow_stride = g.lsum;
        b.raw = d_pair_raw[tb_];
        b.sel = d_sel;
        b.hist = d_hist;
        b.cand = d_cand;
        b.cand_count = d_cand_count;
        b.cand_idx = d_cand_idx;
        b.fm = d_fm;
        b.gr = d_gr;
        b.tie_cnt = d_tie;
        b.bits_thr = d_bits_thr;
        b.bits_clean = d_bits_clean;
        b.bits_keep = d_bits_keep;
        b.run_x0 = d_run_x0;
        b.run_x1 = d_run_x1;
        b.run_n = d_run_n;
        b.run_par = d_run_par;
        b.run_area = d_run_area;
        b.out_pbm = d_out_batch;
        b.out_index = d_out_index[tb_];
        b.info = d_info;
        return b;
    }
    FlowBuffers flow_buffers() const {
        FlowBuffers b;
        b.den = d_den;
        b.pyr_f = d_pyr_f;
        b.exA_f = d_exA_f;
        b.exB_f = d_exB_f;
        b.pyr_p = d_pyr_p;
        b.exA_p = d_exA_p;
        b.exB_p = d_exB_p;
        b.flow0 = d_flow0;
        b.flow1 = d_flow1;
        return b;
    }
};

namespace {

// the |grad I| table only serves the image-gradient saliency (gradient_source 0)
void set_grad_params(froi_ctx* c) {
    static const bool off = [] {  // FROI_NO_GRAD_TABLE=1: compute every hypot (A/B runs)
        const char* e = getenv("FROI_NO_GRAD_TABLE");
        return e && atoi(e) != 0;
    }();
    const bool on = c->d_grad_tab && c->params.gradient_source == 0 && !off;
    c->dp.grad_map = on ? c->d_grad_map : nullptr;
    c->dp.grad_tab = on ? c->d_grad_tab : nullptr;
    c->dp.grad_nv = on ? c->grad_nv : 0;
}

void ctx_alloc(froi_ctx* c) {
    const Geom& g = c->g;
    const size_t px = (size_t)g.W * g.H;
    const int P = c->Pcap, F = c->Fcap;
    size_t& t = c->device_bytes;
    c->frame_bytes = px * g.sample_bytes;
    // constants
    const froi_params& p = c->params;
    {
        const int br = p.bilateral_radius, side = 2 * br + 1;
        std::vector<double> spatial((size_t)side * side);
        for (int dy = -br; dy <= br; ++dy)
            for (int dx = -br; dx <= br; ++dx)
                spatial[(dy + br) * side + (dx + br)] =
                    std::exp(-(dx * dx + dy * dy) / (2.0 * p.bilateral_sigma_spatial * p.bilateral_sigma_spatial));
        std::vector<double> lut((size_t)g.maxval + 1);
        for (int d = 0; d <= g.maxval; ++d) {
            const double tt = double(d) / g.maxval;
            lut[d] = std::exp(-tt * tt / (2.0 * p.bilateral_sigma_range * p.bilateral_sigma_range));
        }
        std::vector<double> wx(g.pw), wy(g.ph);
        for (int x = 0; x < g.pw; ++x) wx[x] = 0.5 - 0.5 * std::cos(2.0 * kPi * x / g.pw);
        for (int y = 0; y < g.ph; ++y) wy[y] = 0.5 - 0.5 * std::cos(2.0 * kPi * y / g.ph);
        c->h_spatial = spatial;
        {
            std::vector<float> nl(256, 0.f);
            const double inv = 1.0 / g.maxval;
            for (int v = 0; v < 256 && v <= g.maxval; ++v) nl[v] = (float)((double)v * inv);
            c->d_norm_lut = dalloc<float>(256, &t);
            FROI_CUDA(cudaMemcpy(c->d_norm_lut, nl.data(), 256 * sizeof(float), cudaMemcpyHostToDevice));
            c->dp.norm_lut = c->d_norm_lut;
        }
        if (g.sample_bytes == 1) {
            // gradient_magnitude (roi.hpp:65-74) of 8-bit frames: every central difference
            // 0.5*(v[a]*inv - v[b]*inv) is one of a few hundred magnitudes, so hypot of a pixel's
            // two differences is a table entry (the same restated glibc hypot, evaluated once)
            const double inv = 1.0 / g.maxval;
            std::vector<double> lv(256), mags;
            for (int v = 0; v < 256; ++v) lv[v] = (double)v * inv;
            mags.reserve(65536);
            for (int a = 0; a < 256; ++a)
                for (int b = 0; b < 256; ++b) mags.push_back(std::fabs(0.5 * (lv[a] - lv[b])));
            std::vector<double> u(mags);
            std::sort(u.begin(), u.end());
            u.erase(std::unique(u.begin(), u.end()), u.end());
            std::vector<unsigned short> map(65536);
            for (int i = 0; i < 65536; ++i)
                map[i] = (unsigned short)(std::lower_bound(u.begin(), u.end(), mags[i]) - u.begin());
            c->grad_nv = (int)u.size();
            c->d_grad_map = dalloc<unsigned short>(65536, &t);
            FROI_CUDA(cudaMemcpy(c->d_grad_map, map.data(), 65536 * sizeof(unsigned short), cudaMemcpyHostToDevice));
            double* d_mag = nullptr;
            FROI_CUDA(cudaMalloc(&d_mag, u.size() * sizeof(double)));
            FROI_CUDA(cudaMemcpyAsync(d_mag, u.data(), u.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            c->d_grad_tab = dalloc<double>(u.size() * u.size(), &t);
            launch_grad_table(d_mag, c->grad_nv, c->d_grad_tab, c->stream);
            FROI_CUDA(cudaStreamSynchronize(c->stream));
            FROI_CUDA(cudaFree(d_mag));
        }
        set_grad_params(c);
        c->d_spatial = dalloc<double>(spatial.size(), &t);
        c->d_lut = dalloc<double>(lut.size(), &t);
        c->d_wx = dalloc<double>(wx.size(), &t);
        c->d_wy = dalloc<double>(wy.size(), &t);
        FROI_CUDA(cudaMemcpy(c->d_spatial, spatial.data(), spatial.size() * 8, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_lut, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_wx, wx.data(), wx.size() * 8, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_wy, wy.data(), wy.size() * 8, cudaMemcpyHostToDevice));
        const auto twr = twiddles(g.pw, false), twc = twiddles(g.ph, false);
        const auto itwr = twiddles(g.pw, true), itwc = twiddles(g.ph, true);
        c->d_tw_row = dalloc<double2>(twr.size(), &t);
        c->d_tw_col = dalloc<double2>(twc.size(), &t);
        c->d_itw_row = dalloc<double2>(itwr.size(), &t);
        c->d_itw_col = dalloc<double2>(itwc.size(), &t);
        FROI_CUDA(cudaMemcpy(c->d_tw_row, twr.data(), twr.size() * 16, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_tw_col, twc.data(), twc.size() * 16, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_itw_row, itwr.data(), itwr.size() * 16, cudaMemcpyHostToDevice));
        FROI_CUDA(cudaMemcpy(c->d_itw_col, itwc.data(), itwc.size() * 16, cudaMemcpyHostToDevice));
    }
    const size_t pyr_px = (size_t)(g.lsum - g.loff[1]);
    c->d_raw = dalloc<uint8_t>(c->frame_bytes * F, &t);
    c->d_den = dalloc<uint8_t>(c->frame_bytes * F, &t);
    c->d_sums = dalloc<unsigned long long>(F, &t);
    c->d_spec = dalloc<double2>((size_t)g.pw * g.ph * F, &t);
    c->d_pyr_f = dalloc<float>(pyr_px * F, &t);
    c->d_exA_f = dalloc<float4>((size_t)g.lsum * F, &t);
    c->d_exB_f = dalloc<float>((size_t)g.lsum * F, &t);
    const int M = p.max_shift, nc = 2 * M + 1;
    c->d_info = dalloc<PairInfo>(P, &t);
    c->d_cols = dalloc<double2>((size_t)nc * g.ph * P, &t);
    c->d_surf = dalloc<double>((size_t)nc * nc * P, &t);
    c->d_pyr_p = dalloc<float>(pyr_px * P, &t);
    c->d_exA_p = dalloc<float4>((size_t)g.lsum * P, &t);
    c->d_exB_p = dalloc<float>((size_t)g.lsum * P, &t);
    c->d_flow0 = dalloc<float2>((size_t)g.lsum * P, &t);
    c->d_flow1 = dalloc<float2>((size_t)g.lsum * P, &t);
    c->d_sel = dalloc<SelState>((size_t)kMaxQueries * P, &t);
    c->d_hist = dalloc<unsigned int>((size_t)kMaxQueries * kHistBins * P, &t);
    FROI_CUDA(cudaMemset(c->d_hist, 0, sizeof(unsigned int) * (size_t)kMaxQueries * kHistBins * P));
    c->d_cand = dalloc<unsigned long long>((size_t)kMaxQueries * kSelCap * P, &t);
    c->d_cand_count = dalloc<unsigned int>((size_t)kMaxQueries * P, &t);
    c->d_cand_idx = dalloc<unsigned int>((size_t)kSelCap * P, &t);
    FROI_CUDA(cudaMemset(c->d_cand_count, 0, sizeof(unsigned int) * (size_t)kMaxQueries * P));
    c->d_fm = dalloc<float>(px * P, &t);
    c->d_gr = dalloc<double>(px * P, &t);
    const int nch = (g.H + 3) / 4;
    c->d_tie = dalloc<unsigned long long>((size_t)nch * 2 * P, &t);
    const size_t words = (size_t)g.H * g.WW;
    c->d_bits_thr = dalloc<uint32_t>(words * P, &t);
    c->d_bits_clean = dalloc<uint32_t>(words * P, &t);
    c->d_bits_keep = dalloc<uint32_t>(words * P, &t);
    const size_t runs = (size_t)g.H * g.RMAX * P;
    c->d_run_x0 = dalloc<uint16_t>(runs, &t);
    c->d_run_x1 = dalloc<uint16_t>(runs, &t);
    c->d_run_n = dalloc<int>((size_t)g.H * P, &t);
    c->d_run_par = dalloc<int>(runs, &t);
    c->d_run_area = dalloc<unsigned int>(runs, &t);
    c->d_out_batch = dalloc<uint8_t>((size_t)g.H * g.SB * P, &t);
    // tables
    c->tables_bytes = sizeof(void*) * F + sizeof(int) * 2 * P + sizeof(void*) * P + sizeof(long long) * P;
    for (int i = 0; i < 2; ++i) {
        c->d_frame_raw[i] = (const void**)dalloc<void*>(F, &t);
        c->d_prev[i] = dalloc<int>(P, &t);
        c->d_next[i] = dalloc<int>(P, &t);
        c->d_pair_raw[i] = (const void**)dalloc<void*>(P, &t);
        c->d_out_index[i] = dalloc<long long>(P, &t);
        FROI_CUDA(cudaMallocHost(&c->h_tables[i], c->tables_bytes));
        FROI_CUDA(cudaEventCreateWithFlags(&c->tables_free[i], cudaEventDisableTiming));
    }
    FROI_CUDA(cudaMallocHost((void**)&c->h_info, sizeof(PairInfo) * P));
    c->h_info_cap = P;
    for (int i = 0; i < 8; ++i) FROI_CUDA(cudaEventCreate(&c->ev[i]));
    FROI_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    FROI_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    FROI_CUDA(cudaEventCreateWithFlags(&c->ev_den, cudaEventDisableTiming));
    FROI_CUDA(cudaEventCreateWithFlags(&c->ev_exp, cudaEventDisableTiming));
    FROI_CUDA(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
    FROI_CUDA(cudaEventCreateWithFlags(&c->d2h_done, cudaEventDisableTiming));
    // the constant tables above went through pageable cudaMemcpy on the legacy stream, which may
    // return before the DMA lands and does not order the non-blocking streams: finish them here
    FROI_CUDA(cudaDeviceSynchronize());
}

// Buffers of the bit-exact flow (double images and expansions per slot, two [pair][5][W*H]
// scratch planes sets), allocated when the mode is first switched on.
void ensure_flow64(froi_ctx* c) {
    if (c->d64_ex_f) return;
    const Geom& g = c->g;
    const size_t px = (size_t)g.W * g.H, ls = (size_t)g.lsum;
    size_t& t = c->device_bytes;
    c->d64_img_f = dalloc<double>(ls * c->Fcap, &t);
    c->d64_ex_f = dalloc<double>(5 * ls * c->Fcap, &t);
    c->d64_img_p = dalloc<double>(ls * c->Pcap, &t);
    c->d64_ex_p = dalloc<double>(5 * ls * c->Pcap, &t);
    // prod doubles as the frame slots' blur scratch (Fcap <= 5 Pcap), rowm as the pair slots'
    c->d64_prod = dalloc<double>(5 * px * std::max<size_t>(c->Pcap, (c->Fcap + 4) / 5), &t);
    c->d64_rowm = dalloc<double>(5 * px * c->Pcap, &t);
}

void drop_graphs(froi_ctx* c) {
    for (auto& kv : c->graphs) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
    }
    c->graphs.clear();
}

void ctx_free(froi_ctx* c) {
    cudaSetDevice(c->device);
    drop_graphs(c);
    if (c->lane) {
        ctx_free(c->lane);
        delete c->lane;
        c->lane = nullptr;
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->stream) cudaStreamSynchronize(c->stream);
    void* ptrs[] = {c->d_norm_lut, c->d_grad_map, c->d_grad_tab, c->d_spatial, c->d_lut, c->d_wx, c->d_wy, c->d_tw_row, c->d_tw_col, c->d_itw_row,
                    c->d_itw_col, c->d_raw, c->d_den, c->d_sums, c->d_spec, c->d_pyr_f, c->d_exA_f,
                    c->d_exB_f, c->d_info, c->d_cols, c->d_surf, c->d_pyr_p, c->d_exA_p, c->d_exB_p,
                    c->d_flow0, c->d_flow1, c->d_sel, c->d_hist, c->d_cand, c->d_cand_count, c->d_cand_idx, c->d_fm, c->d_gr, c->d_tie, c->d_bits_thr,
                    c->d_bits_clean, c->d_bits_keep, c->d_run_x0, c->d_run_x1, c->d_run_n, c->d_run_par, c->d_run_area,
                    c->d_out_batch, c->d_seq_out, c->d_seq_tmp, c->d_carry[0], c->d_carry[1],
                    c->d_ring, c->d_outring, c->d64_img_f, c->d64_ex_f, c->d64_img_p, c->d64_ex_p,
                    c->d64_prod, c->d64_rowm};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        if (c->d_frame_raw[i]) cudaFree((void*)c->d_frame_raw[i]);
        if (c->d_prev[i]) cudaFree(c->d_prev[i]);
        if (c->d_next[i]) cudaFree(c->d_next[i]);
        if (c->d_pair_raw[i]) cudaFree((void*)c->d_pair_raw[i]);
        if (c->d_out_index[i]) cudaFree(c->d_out_index[i]);
        if (c->h_tables[i]) cudaFreeHost(c->h_tables[i]);
        if (c->tables_free[i]) cudaEventDestroy(c->tables_free[i]);
    }
    if (c->h_info) cudaFreeHost(c->h_info);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& a : c->bev)
        for (auto e : a) cudaEventDestroy(e);
    c->courier.reset();  // joins its thread (idle between calls)
    c->dpool.reset();
    c->pool.reset();
    for (auto e : c->chunk_ready) cudaEventDestroy(e);
    for (auto e : c->stage_free) cudaEventDestroy(e);
    for (auto e : c->delivered) cudaEventDestroy(e);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_outring) cudaFreeHost(c->h_outring);
    for (auto e : c->d2h_ev) cudaEventDestroy(e);
    if (c->d2h_done) cudaEventDestroy(c->d2h_done);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_den) cudaEventDestroy(c->ev_den);
    if (c->ev_exp) cudaEventDestroy(c->ev_exp);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
}

void ensure_seq_out(froi_ctx* c, size_t bytes) {
    if (c->seq_out_cap >= bytes) return;
    if (c->d_seq_out) FROI_CUDA(cudaFree(c->d_seq_out));
    c->d_seq_out = nullptr;
    FROI_CUDA(cudaMalloc(&c->d_seq_out, bytes));
    c->seq_out_cap = bytes;
}
void ensure_seq_tmp(froi_ctx* c, size_t bytes) {
    if (c->seq_tmp_cap >= bytes) return;
    if (c->d_seq_tmp) FROI_CUDA(cudaFree(c->d_seq_tmp));
    c->d_seq_tmp = nullptr;
    FROI_CUDA(cudaMalloc(&c->d_seq_tmp, bytes));
    c->seq_tmp_cap = bytes;
}

// One adjacent pair (frame a -> frame b) of some well.
struct PairJob {
    const void* raw_prev;  // device pointers to the raw frames
    const void* raw_next;
    long long out_index;   // mask index in the output PBM buffer
    long long stats_index; // index into the caller's stats array (or -1)
    cudaEvent_t ready = nullptr;  // ingest of this pair's frames complete (copy stream)
};

// Runs one batch of pairs.  frames given on device; output PBM masks written at out_index of
// out_pbm (device).  h_stats_pairs receives the PairInfo of each pair (host, after sync).
// One batch of pairs, enqueued without a host synchronisation: its PairInfo rows are copied to
// h_info[info_off ..] and its stage events are batch event set `bi` (read by finish_batches).
void run_batch(froi_ctx* c, froi_ctx* owner, const std::vector<PairJob>& jobs, size_t j0, size_t j1,
               uint8_t* out_pbm, size_t bi, size_t info_off) {
    const Geom& g = c->g;
    const int n_pairs = int(j1 - j0);
    cudaStream_t s = c->stream;
    const int tb = c->tb;
    c->tb ^= 1;
    FROI_CUDA(cudaEventSynchronize(c->tables_free[tb]));
    // frame slots: unique raw pointers in order
    uint8_t* h = (uint8_t*)c->h_tables[tb];
    const void** h_frame_raw = (const void**)h;
    int* h_prev = (int*)(h + sizeof(void*) * c->Fcap);
    int* h_next = h_prev + c->Pcap;
    const void** h_pair_raw = (const void**)(h_next + c->Pcap);
    long long* h_out = (long long*)(h_pair_raw + c->Pcap);
    int nf = 0;
    const void* last = nullptr;
    std::vector<cudaEvent_t> slot_ready;  // ingest event each frame slot waits for
    for (size_t j = j0; j < j1; ++j) {
        const PairJob& J = jobs[j];
        int sp, sn;
        if (nf > 0 && last == J.raw_prev) sp = nf - 1;
        else {
            h_frame_raw[nf] = J.raw_prev;
            slot_ready.push_back(J.ready);
            sp = nf++;
        }
        h_frame_raw[nf] = J.raw_next;
        slot_ready.push_back(J.ready);
        sn = nf++;
        last = J.raw_next;
        const int p = int(j - j0);
        h_prev[p] = sp;
        h_next[p] = sn;
        h_pair_raw[p] = J.raw_next;
        h_out[p] = J.out_index;
    }
    FROI_CUDA(cudaMemcpyAsync(c->d_frame_raw[tb], h_frame_raw, sizeof(void*) * nf, cudaMemcpyHostToDevice, s));
    FROI_CUDA(cudaMemcpyAsync(c->d_prev[tb], h_prev, sizeof(int) * n_pairs, cudaMemcpyHostToDevice, s));
    FROI_CUDA(cudaMemcpyAsync(c->d_next[tb], h_next, sizeof(int) * n_pairs, cudaMemcpyHostToDevice, s));
    FROI_CUDA(cudaMemcpyAsync(c->d_pair_raw[tb], h_pair_raw, sizeof(void*) * n_pairs, cudaMemcpyHostToDevice, s));
    FROI_CUDA(cudaMemcpyAsync(c->d_out_index[tb], h_out, sizeof(long long) * n_pairs, cudaMemcpyHostToDevice, s));
    FROI_CUDA(cudaEventRecord(c->tables_free[tb], s));

    cudaEvent_t* ev = owner->bev[bi].data();
    // runs of frame slots that share an ingest event
    std::vector<std::pair<int, int>> runs;
    for (int s0 = 0; s0 < nf;) {
        int s1 = s0 + 1;
        while (s1 < nf && slot_ready[s1] == slot_ready[s0]) ++s1;
        runs.emplace_back(s0, s1);
        s0 = s1;
    }
    // the stage sequence; `rec` records stage event i (a plain record, or an external event node
    // inside a capture), `first_wait` orders each denoise run after its ingest event
    bool fork_now = false;  // set for graph captures when the context forks (below)
    auto enqueue = [&](auto rec, bool per_run) {
        rec(0);
        FROI_CUDA(cudaMemsetAsync(c->d_sums, 0, sizeof(unsigned long long) * nf, s));
        // denoise each run of frame slots as soon as the ingest chunk holding it has landed (the
        // first batch of a host call starts after its first sub-chunk instead of the whole batch)
        if (per_run) {
            for (auto& r : runs) {
                if (slot_ready[r.first]) FROI_CUDA(cudaStreamWaitEvent(s, slot_ready[r.first], 0));
                launch_denoise(g, c->dp, c->d_frame_raw[tb] + r.first, c->d_den + c->frame_bytes * r.first,
                               c->d_sums + r.first, c->h_spatial.data(), c->d_lut, r.second - r.first, s);
            }
        } else {
            launch_denoise(g, c->dp, c->d_frame_raw[tb], c->d_den, c->d_sums, c->h_spatial.data(), c->d_lut, nf, s);
        }
        rec(1);
        FlowBuffers fb = c->flow_buffers();
        Flow64Buffers fb64 = c->flow64_buffers();
        // the flow's expansions: fp32 (k_flow.cu) or the bit-exact fp64 mode (k_flow64.cu)
        auto expand_frames = [&](cudaStream_t st) {
            if (c->flow_exact) launch_expand_frames64(g, c->f64c, fb64, c->d_den, nf, st);
            else launch_expand_frames(g, c->dp, fb, nf, st);
        };
        auto expand_shifted = [&](cudaStream_t st) {
            if (c->flow_exact) launch_expand_shifted64(g, c->f64c, fb64, c->d_den, c->d_next[tb], c->d_info, n_pairs, st);
            else launch_expand_shifted(g, c->dp, fb, c->d_next[tb], c->d_info, n_pairs, st);
        };
        if (fork_now) {
            // expansions of the frame slots on the side branch, FFT + registration on this one
            FROI_CUDA(cudaEventRecord(c->ev_den, s));
            FROI_CUDA(cudaStreamWaitEvent(c->side, c->ev_den, 0));
            expand_frames(c->side);
            FROI_CUDA(cudaEventRecord(c->ev_exp, c->side));
            launch_fft_forward(g, c->d_den, c->d_sums, c->d_wx, c->d_wy, c->d_tw_row, c->d_tw_col, c->d_spec, nf, s);
            rec(2);
            rec(3);
            launch_register_pairs(g, c->dp, c->d_spec, c->d_prev[tb], c->d_next[tb], c->d_itw_row, c->d_itw_col,
                                  c->d_cols, c->d_surf, c->d_info, n_pairs, s);
            rec(4);
            expand_shifted(s);
            FROI_CUDA(cudaStreamWaitEvent(s, c->ev_exp, 0));
            rec(5);
        } else {
            launch_fft_forward(g, c->d_den, c->d_sums, c->d_wx, c->d_wy, c->d_tw_row, c->d_tw_col, c->d_spec, nf, s);
            rec(2);
            expand_frames(s);
            rec(3);
            launch_register_pairs(g, c->dp, c->d_spec, c->d_prev[tb], c->d_next[tb], c->d_itw_row, c->d_itw_col,
                                  c->d_cols, c->d_surf, c->d_info, n_pairs, s);
            rec(4);
            expand_shifted(s);
            rec(5);
        }
        int cur = 0;
        if (c->flow_exact) launch_flow64(g, c->dp, fb64, c->d_prev[tb], c->d_next[tb], c->d_info, n_pairs, s, &cur);
        else cur = launch_flow(g, c->dp, fb, c->d_prev[tb], c->d_next[tb], c->d_info, n_pairs, s);
        rec(6);
        MaskBuffers mb = c->mask_buffers(tb);
        mb.flow = cur ? c->d_flow1 : c->d_flow0;
        mb.out_pbm = out_pbm;
        uint64_t ml = 0;
        launch_mask_stage(g, c->dp, mb, n_pairs, s, &ml);
        rec(7);
        return ml;
    };
    // a CUDA graph per batch shape; the first batch of a host call, whose frames arrive in
    // sub-chunks, keeps one denoise launch per sub-chunk (it starts before its frames are all in)
    const bool graph = c->use_graphs && runs.size() <= 2;
    int n_denoise = graph ? 1 : (int)runs.size();
    if (graph) {
        for (auto& r : runs)
            if (slot_ready[r.first]) FROI_CUDA(cudaStreamWaitEvent(s, slot_ready[r.first], 0));
        const auto key = std::make_tuple(tb, n_pairs, nf, (const void*)out_pbm);
        auto it = c->graphs.find(key);
        if (it == c->graphs.end()) {
            froi_ctx::BatchGraph bg;
            FROI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            fork_now = c->fork;
            try {
                bg.launches = enqueue([&](int i) { FROI_CUDA(cudaEventRecordWithFlags(ev[i], s, cudaEventRecordExternal)); },
                                      false);
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            FROI_CUDA(cudaStreamEndCapture(s, &bg.graph));
            size_t nn = 0;
            FROI_CUDA(cudaGraphGetNodes(bg.graph, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            FROI_CUDA(cudaGraphGetNodes(bg.graph, nodes.data(), &nn));
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType ty;
                FROI_CUDA(cudaGraphNodeGetType(nd, &ty));
                if (ty != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t e;
                FROI_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &e));
                for (int i = 0; i < 8; ++i)
                    if (e == ev[i]) bg.ev_node[i] = nd;
            }
            for (int i = 0; i < 8; ++i)
                if (!bg.ev_node[i]) throw Error(3, "batch graph: stage event node missing");
            FROI_CUDA(cudaGraphInstantiate(&bg.exec, bg.graph, 0));
            it = c->graphs.emplace(key, bg).first;
        }
        froi_ctx::BatchGraph& bg = it->second;
        for (int i = 0; i < 8; ++i) FROI_CUDA(cudaGraphExecEventRecordNodeSetEvent(bg.exec, bg.ev_node[i], ev[i]));
        FROI_CUDA(cudaGraphLaunch(bg.exec, s));
        owner->launches += bg.launches;
    } else {
        owner->launches += enqueue([&](int i) { FROI_CUDA(cudaEventRecord(ev[i], s)); }, true);
    }
    FROI_CUDA(cudaMemcpyAsync(owner->h_info + info_off, c->d_info, sizeof(PairInfo) * n_pairs,
                              cudaMemcpyDeviceToHost, s));
    froi_kernel_times& K = owner->ktimes;
    K.pairs += n_pairs;
    K.frames += nf;
    K.flow_iter_launches += (uint64_t)g.L * c->dp.iterations;
    K.batches += 1;
    // launches: denoise (one per ingest run), fft 2, expand (1 + 2(L-1)) x2, register 3,
    // flow L*iters + (L-1) upsamplings (+ the mask stage's own count)
    // (bit-exact flow: expand (1 + 2(L-1) + L) x2, flow 3 L iters + (L-1))
    if (c->flow_exact)
        owner->launches += n_denoise + 2 + 2 * (1 + 2 * (g.L - 1) + g.L) + 3 + 3 * (uint64_t)g.L * c->dp.iterations +
                           (g.L - 1);
    else
        owner->launches += n_denoise + 2 + 2 * (1 + 2 * (g.L - 1)) + 3 + (uint64_t)g.L * c->dp.iterations + (g.L - 1);
}

// The second lane, created on first use with the owner's device, parameters and capacity.
// One lane (froi_ctx_set_lanes or FROI_LANES=1) keeps every batch on the owner's stream.
froi_ctx* lane_of(froi_ctx* c) {
    if (c->lanes < 2) return nullptr;
    if (!c->lane) {
        froi_ctx* l = new froi_ctx();
        try {
            l->device = c->device;
            l->params = c->params;
            l->g = c->g;
            l->dp = c->dp;
            l->Pcap = c->Pcap;
            l->Fcap = c->Fcap;
            FROI_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
            ctx_alloc(l);
        } catch (...) {
            ctx_free(l);
            delete l;
            throw;
        }
        c->lane = l;
        FROI_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        FROI_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    c->lane->fork = c->fork;
    c->lane->dp = c->dp;  // set_params may have changed the run-time parameters
    c->lane->params = c->params;
    c->lane->f64c = c->f64c;
    if (c->flow_exact) ensure_flow64(c->lane);
    if (c->lane->flow_exact != c->flow_exact) drop_graphs(c->lane);
    c->lane->flow_exact = c->flow_exact;
    return c->lane;
}

void accumulate_batch_times(froi_ctx* c, size_t nb);

// Batch boundaries over n pairs: a first batch of `first` (<= cap) pairs, then batches of cap.  A
// short tail (< cap / 2) is evened out with the batch before it: the two run on different
// execution lanes, so both lanes finish together instead of one lane trailing a full batch while
// the other has (nearly) nothing left.  $FROI_TAIL=0 keeps the plain split.
std::vector<size_t> batch_bounds(size_t n, size_t cap, size_t first) {
    static const bool tail = [] {
        const char* e = getenv("FROI_TAIL");
        return !(e && atoi(e) == 0);
    }();
    std::vector<size_t> b{0};
    for (size_t pos = 0; pos < n;) {
        pos = std::min(n, pos + (b.size() == 1 ? std::min(first, cap) : cap));
        b.push_back(pos);
    }
    const size_t nbat = b.size() - 1;
    if (tail && nbat >= 2 && n - b[nbat - 1] < cap / 2) b[nbat - 1] = b[nbat - 2] + (n - b[nbat - 2] + 1) / 2;
    return b;
}

// Device-resident frames and masks: enqueue every batch of `jobs`, then synchronise once; stage
// times from each batch's events, PairInfo rows in job order.
void run_batches(froi_ctx* c, const std::vector<PairJob>& jobs, uint8_t* out_pbm,
                 std::vector<PairInfo>& infos) {
    const std::vector<size_t> bb = batch_bounds(jobs.size(), (size_t)c->Pcap, (size_t)c->Pcap);
    const size_t nb = bb.size() - 1;
    if (c->h_info_cap < jobs.size()) {
        FROI_CUDA(cudaStreamSynchronize(c->stream));
        FROI_CUDA(cudaFreeHost(c->h_info));
        c->h_info = nullptr;
        c->h_info_cap = 0;
        FROI_CUDA(cudaMallocHost((void**)&c->h_info, sizeof(PairInfo) * jobs.size()));
        c->h_info_cap = jobs.size();
    }
    while (c->bev.size() < nb) {
        std::array<cudaEvent_t, 8> a;
        for (auto& e : a) FROI_CUDA(cudaEventCreate(&e));
        c->bev.push_back(a);
    }
    froi_ctx* lane = nb >= 2 ? lane_of(c) : nullptr;
    if (lane) {
        // the lane starts after everything already ordered on the owner's stream
        FROI_CUDA(cudaEventRecord(c->ev_fork, c->stream));
        FROI_CUDA(cudaStreamWaitEvent(lane->stream, c->ev_fork, 0));
    }
    for (size_t b = 0; b < nb; ++b) {
        const size_t j0 = bb[b], j1 = bb[b + 1];
        froi_ctx* x = (lane && (b & 1)) ? lane : c;
        run_batch(x, c, jobs, j0, j1, out_pbm, b, j0);
    }
    if (lane) {
        // later work on the owner's stream (frame-0 copies, ensemble, delivery) follows both lanes
        FROI_CUDA(cudaEventRecord(c->ev_join, lane->stream));
        FROI_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    accumulate_batch_times(c, nb);
    infos.insert(infos.end(), c->h_info, c->h_info + jobs.size());
}

// Stage times of the nb batches of the last call from their events (after the host sync).
void accumulate_batch_times(froi_ctx* c, size_t nb) {
    auto ns = [](float m) { return (uint64_t)((double)m * 1e6); };
    froi_kernel_times& K = c->ktimes;
    for (size_t b = 0; b < nb; ++b) {
        float ms[7];
        for (int i = 0; i < 7; ++i) FROI_CUDA(cudaEventElapsedTime(&ms[i], c->bev[b][i], c->bev[b][i + 1]));
        c->times.denoise_ns += ns(ms[0]);
        c->times.flow_ns += ns(ms[1] + ms[2] + ms[3] + ms[4] + ms[5]);
        c->times.roi_ns += ns(ms[6]);
        K.denoise_ns += ns(ms[0]);
        K.fft_forward_ns += ns(ms[1]);
        K.expand_ns += ns(ms[2]);
        K.register_ns += ns(ms[3]);
        K.expand_shifted_ns += ns(ms[4]);
        K.flow_iter_ns += ns(ms[5]);
        K.mask_ns += ns(ms[6]);
    }
}

// One frame of host samples into the context's sample type: Frame::pixels are uint16 whatever
// the depth (core.hpp:30), so 8-bit frames are narrowed here, with the Frame invariant
// (core.hpp:24-25, every sample < 2^depth) checked on the way.
void convert_frame(const uint8_t* src, int src_bytes, uint8_t* dst, int dst_bytes, size_t px) {
    if (src_bytes == dst_bytes) {
        std::memcpy(dst, src, px * src_bytes);
        return;
    }
    if (src_bytes == 2) {
        const uint16_t* s16 = (const uint16_t*)src;
        uint16_t hi = 0;
        for (size_t i = 0; i < px; ++i) {
            hi |= s16[i];
            dst[i] = (uint8_t)s16[i];
        }
        if (hi > 255) throw Error(2, "frame sample exceeds the 8-bit depth");
        return;
    }
    uint16_t* d16 = (uint16_t*)dst;
    for (size_t i = 0; i < px; ++i) d16[i] = src[i];
}

void fill_stats(const Geom& g, const PairInfo& I, froi_frame_stats* st) {
    st->dx = I.dx;
    st->dy = I.dy;
    st->confidence = I.confidence;
    st->mask_count = I.mask_count;
    st->raw_fraction = double(I.mask_count) / double((long long)g.W * g.H);
    st->components = I.components;
}

// Ingest host frames (any sample width) into a device buffer of the context's sample type, on
// the context stream (used by the single-frame parity taps; the throughput entries go through
// run_host_call).  The conversion buffer is kept alive until its copy has completed.
void upload_frames(froi_ctx* c, const void* frames, int sample_bytes, size_t stride, long long n,
                   uint8_t* dst) {
    const Geom& g = c->g;
    const size_t px = (size_t)g.W * g.H;
    if (sample_bytes == g.sample_bytes && stride == c->frame_bytes) {
        FROI_CUDA(cudaMemcpyAsync(dst, frames, c->frame_bytes * n, cudaMemcpyHostToDevice, c->stream));
        return;
    }
    if (sample_bytes == g.sample_bytes) {
        FROI_CUDA(cudaMemcpy2DAsync(dst, c->frame_bytes, frames, stride, c->frame_bytes, n,
                                    cudaMemcpyHostToDevice, c->stream));
        return;
    }
    std::vector<uint8_t> tmp(c->frame_bytes);
    for (long long f = 0; f < n; ++f) {
        convert_frame((const uint8_t*)frames + stride * f, sample_bytes, tmp.data(), g.sample_bytes, px);
        FROI_CUDA(cudaMemcpyAsync(dst + c->frame_bytes * f, tmp.data(), c->frame_bytes, cudaMemcpyHostToDevice,
                                  c->stream));
        FROI_CUDA(cudaStreamSynchronize(c->stream));  // tmp is reused by the next frame
    }
}

// Whole wells: frames on device (well-major, contiguous in ctx sample type).
void extract_wells_dev(froi_ctx* c, const uint8_t* d_frames, size_t stride, int n_wells, int n_frames,
                       uint8_t* d_out, std::vector<PairInfo>& infos) {
    const Geom& g = c->g;
    std::vector<PairJob> jobs;
    jobs.reserve((size_t)n_wells * (n_frames - 1));
    for (int w = 0; w < n_wells; ++w)
        for (int t = 1; t < n_frames; ++t) {
            PairJob J;
            J.raw_prev = d_frames + stride * ((size_t)w * n_frames + t - 1);
            J.raw_next = d_frames + stride * ((size_t)w * n_frames + t);
            J.out_index = (long long)w * n_frames + t;
            J.stats_index = J.out_index;
            jobs.push_back(J);
        }
    c->times = froi_stage_times{};
    c->ktimes = froi_kernel_times{};
    c->launches = 0;
    run_batches(c, jobs, d_out, infos);
    // frame 0 borrows frame 1's mask (roi.hpp:348)
    const size_t mb = (size_t)g.H * g.SB;
    for (int w = 0; w < n_wells; ++w)
        FROI_CUDA(cudaMemcpyAsync(d_out + mb * ((size_t)w * n_frames), d_out + mb * ((size_t)w * n_frames + 1),
                                  mb, cudaMemcpyDeviceToDevice, c->stream));
    // temporal ensemble on the pre-ensemble masks (roi.hpp:356-362)
    if (c->params.adjacent_factor > 0) {
        ensure_seq_tmp(c, mb * n_frames);
        for (int w = 0; w < n_wells; ++w) {
            uint8_t* base = d_out + mb * ((size_t)w * n_frames);
            launch_ensemble(g, base, c->d_seq_tmp, n_frames, c->params.adjacent_factor, c->stream);
            FROI_CUDA(cudaMemcpyAsync(base, c->d_seq_tmp, mb * n_frames, cudaMemcpyDeviceToDevice, c->stream));
            ++c->launches;
        }
    }
}

void stats_for_wells(froi_ctx* c, const std::vector<PairInfo>& infos, int n_wells, int n_frames,
                     froi_frame_stats* stats) {
    if (!stats) return;
    size_t k = 0;
    for (int w = 0; w < n_wells; ++w) {
        froi_frame_stats* s = stats + (size_t)w * n_frames;
        for (int t = 1; t < n_frames; ++t) fill_stats(c->g, infos[k++], &s[t]);
        s[0] = s[1];
        s[0].dx = 0;
        s[0].dy = 0;
        s[0].confidence = 1.0;
    }
}

int check_layout(int layout) {
    return layout == FROI_MASK_BYTES || layout == FROI_MASK_PBM;
}

// ------------------------------------------------------------------ host ingest / egress pipeline
//
// One host call (froi_extract_wells / froi_extract_frames / froi_stream_push) streams its frames
// through bounded rings, so device and pinned host memory do not grow with the call:
//
//   host frames --(pool: copy or u16<->u8 conversion)--> pinned staging ring (kStageChunks
//   chunks) --copy stream--> device ingest ring (kRingChunks chunks of ring_chunk frames)
//   --batches on the execution lanes--> device egress ring (kOutBatches batches of PBM masks)
//   --d2h stream--> caller's pinned PBM buffers directly, or the pinned egress twin from which
//   the courier thread unpacks each batch into the caller's RoiMask bytes (or copies PBM rows).
//
// Frames are uploaded in (well, frame) order just ahead of the batch that first needs them;
// each upload chunk records an event the batch's denoise waits on.  Pinned sources of the
// context's sample type skip the staging ring.  A ring slot is rewritten only after the last
// batch reading it has finished (stream-ordered waits, no host sync), a staging chunk only after
// its previous copy has completed, an egress slot only after its masks reached the host.
// Temporal ensembling (k > 0) needs every mask of a well before any output: those calls keep
// the masks on the device until the end (full egress buffer) and deliver them afterwards.
constexpr int kRingChunks = 6;
constexpr int kStageChunks = 3;
constexpr int kOutBatches = 4;

struct HostCall {
    int n_wells = 0, n_frames = 0;        // frames per well in this call
    int t_begin = 1;                      // next frame of each well's first pair (0: prev = carry)
    int src_bytes = 1;                    // sample bytes of the host frames
    std::vector<const uint8_t*> host;     // [w*n + t] host frame (nullptr: dev[] has it)
    std::vector<const uint8_t*> dev;      // [w*n + t] device-resident frame (context sample type)
    std::vector<const uint8_t*> carry;    // [w] device frame t = -1 when t_begin == 0
    uint8_t* new_carry = nullptr;         // device [w] frames: receives each well's last frame
    int layout = FROI_MASK_PBM;
    std::vector<uint8_t*> mask;           // [w*n + t] host destination (layout)
    froi_mask_sink sink = nullptr;        // or: destination asked for just before it is written
    froi_mask_put put = nullptr;          // or: finished mask handed over (caller copies it)
    void* sink_user = nullptr;
    uint8_t* dev_masks = nullptr;         // device PBM destination [w*n + t] instead of mask[]
    bool frame0_rule = true;              // mask (w, 0) := mask (w, 1) (roi.hpp:348)
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess;
    cudaGetLastError();  // an unregistered pointer may leave an error behind on older drivers
    return ok && (a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged);
}

// Pinned-ness of n buffers of `bytes` each: a run of back-to-back buffers is one allocation when
// its first and last byte are both pinned (two queries per run instead of one per buffer).
std::vector<char> pinned_flags(const std::vector<const uint8_t*>& p, size_t bytes) {
    std::vector<char> f(p.size(), 0);
    for (size_t i = 0; i < p.size();) {
        if (!p[i]) {
            ++i;
            continue;
        }
        size_t e = i + 1;
        while (e < p.size() && p[e] && p[e] == p[e - 1] + bytes) ++e;
        const bool pin = is_pinned(p[i]) && is_pinned(p[e - 1] + bytes - 1);
        for (size_t k = i; k < e; ++k) f[k] = pin;
        i = e;
    }
    return f;
}

void ensure_pipeline(froi_ctx* c) {
    if (!c->pool) {
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        const int dev = c->device;
        // host threads: all but two hardware threads (the caller's and the courier), at most 16
        // ($FROI_HOST_THREADS overrides), split between frame conversion (the caller's pool) and
        // mask delivery (the courier's), so a batch's delivery never queues behind the next
        // batches' conversions
        int nt = std::max(2, std::min(16, hw - 2));
        if (const char* e = getenv("FROI_HOST_THREADS")) nt = std::max(2, atoi(e));
        auto init = [dev] { cudaSetDevice(dev); };
        c->pool.reset(new HostPool(nt - nt / 2, init));
        c->dpool.reset(new HostPool(nt / 2, init));
        c->courier.reset(new HostPool(1, init));
    }
    if (!c->d_ring) {
        c->ring_chunk = std::max(8, c->Pcap);
        c->ring_frames = kRingChunks * c->ring_chunk;
        FROI_CUDA(cudaMalloc(&c->d_ring, c->frame_bytes * c->ring_frames));
        const size_t mb = (size_t)c->g.H * c->g.SB;
        FROI_CUDA(cudaMalloc(&c->d_outring, mb * c->Pcap * kOutBatches));
    }
}

void ensure_staging(froi_ctx* c) {
    if (c->h_stage) return;
    FROI_CUDA(cudaMallocHost((void**)&c->h_stage, c->frame_bytes * c->ring_chunk * kStageChunks));
    for (int i = 0; i < kStageChunks; ++i) {
        cudaEvent_t e;
        FROI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->stage_free.push_back(e);
    }
}

void ensure_host_outring(froi_ctx* c) {
    if (c->h_outring) return;
    const size_t mb = (size_t)c->g.H * c->g.SB;
    FROI_CUDA(cudaMallocHost((void**)&c->h_outring, mb * c->Pcap * kOutBatches));
}

cudaEvent_t event_at(std::vector<cudaEvent_t>& v, size_t i) {
    while (v.size() <= i) {
        cudaEvent_t e;
        FROI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        v.push_back(e);
    }
    return v[i];
}

// $FROI_TRACE=1: host-side phase times of each host call on stderr (diagnostics)
static bool trace_on() {
    static const bool on = [] {
        const char* e = getenv("FROI_TRACE");
        return e && atoi(e) == 1;
    }();
    return on;
}
static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// One PBM mask (H rows of SB bytes, MSB first) into the caller's layout.
void put_mask(const Geom& g, const uint8_t* pbm, int layout, uint8_t* dst) {
    const size_t mb = (size_t)g.H * g.SB;
    if (layout == FROI_MASK_PBM) {
        std::memcpy(dst, pbm, mb);
        return;
    }
    // RoiMask bytes (core.hpp:78-101): 8 pixels per PBM byte through a 256-entry table
    static const auto table = [] {
        std::array<uint64_t, 256> t{};
        for (int v = 0; v < 256; ++v) {
            uint64_t x = 0;
            for (int b = 0; b < 8; ++b) x |= (uint64_t)((v >> (7 - b)) & 1) << (8 * b);  // little endian
            t[v] = x;
        }
        return t;
    }();
    const int full = g.W / 8, rem = g.W % 8;
    for (int y = 0; y < g.H; ++y) {
        const uint8_t* r = pbm + (size_t)y * g.SB;
        uint8_t* o = dst + (size_t)y * g.W;
        for (int i = 0; i < full; ++i) std::memcpy(o + 8 * i, &table[r[i]], 8);
        if (rem) std::memcpy(o + 8 * full, &table[r[full]], rem);
    }
}

// Runs one host call end to end (see the comment block above).  Throws froi::Error; on any error
// every queued copy, kernel and host task has finished before the exception leaves.
void run_host_call(froi_ctx* c, const HostCall& io, std::vector<PairInfo>& infos) {
    double t_convert = 0.0, t_stage_wait = 0.0, t_tail_tasks = 0.0;
    const double t_call0 = trace_on() ? now_ms() : 0.0;
    const Geom& g = c->g;
    const size_t fb = c->frame_bytes, mb = (size_t)g.H * g.SB;
    const int n = io.n_frames, nw = io.n_wells;
    const size_t nk = (size_t)nw * n;
    const bool ring_out = !io.dev_masks && c->params.adjacent_factor == 0;
    ensure_pipeline(c);
    // pairs in (well, frame) order; frame (w, t) of the call has upload index k = w*n + t
    std::vector<PairJob> jobs;
    std::vector<std::pair<int, int>> wt;
    jobs.reserve(nk);
    for (int w = 0; w < nw; ++w)
        for (int t = io.t_begin; t < n; ++t) {
            jobs.push_back(PairJob{});
            wt.emplace_back(w, t);
        }
    // which frames go through the pinned staging ring (pageable, or another sample width)
    // (frames of another sample width are staged whatever their memory: no pinned-ness queries)
    const std::vector<char> src_pinned = io.src_bytes == g.sample_bytes
                                             ? pinned_flags(io.host, (size_t)g.W * g.H * io.src_bytes)
                                             : std::vector<char>(nk, 0);
    bool any_staged = false;
    for (size_t k = 0; k < nk; ++k) any_staged |= io.host[k] && (io.src_bytes != g.sample_bytes || !src_pinned[k]);
    // batches: Pcap pairs, except a first batch of Pcap / 4 when the frames need host conversion,
    // so the GPU starts after a quarter of the first batch's frames are converted, not all of them
    const size_t P = (size_t)c->Pcap;
    const std::vector<size_t> bb = batch_bounds(jobs.size(), P, any_staged ? std::max<size_t>(1, P / 4) : P);
    auto bstart = [&](size_t b) { return bb[b]; };
    const size_t nb = bb.size() - 1;
    if (c->h_info_cap < jobs.size()) {
        FROI_CUDA(cudaStreamSynchronize(c->stream));
        FROI_CUDA(cudaFreeHost(c->h_info));
        c->h_info = nullptr;
        c->h_info_cap = 0;
        FROI_CUDA(cudaMallocHost((void**)&c->h_info, sizeof(PairInfo) * jobs.size()));
        c->h_info_cap = jobs.size();
    }
    while (c->bev.size() < nb) {
        std::array<cudaEvent_t, 8> a;
        for (auto& e : a) FROI_CUDA(cudaEventCreate(&e));
        c->bev.push_back(a);
    }
    for (size_t b = 0; b < nb; ++b) event_at(c->delivered, b), event_at(c->d2h_ev, b);
    uint8_t* d_full = nullptr;  // egress without the ring (ensemble / device destinations)
    if (!ring_out) {
        if (io.dev_masks) d_full = io.dev_masks;
        else {
            ensure_seq_out(c, mb * nk);
            d_full = c->d_seq_out;
        }
    }
    if (any_staged) ensure_staging(c);
    const bool general_out = ring_out && (io.sink || io.put || io.layout != FROI_MASK_PBM || [&] {
        const std::vector<char> f = pinned_flags(std::vector<const uint8_t*>(io.mask.begin(), io.mask.end()), mb);
        for (char x : f)
            if (!x) return true;
        return false;
    }());
    if (general_out) ensure_host_outring(c);
    auto dest = [&](int w, int t) -> uint8_t* {
        if (!io.sink) return io.mask[(size_t)w * n + t];
        uint8_t* d = io.sink(io.sink_user, w, t);
        if (!d) throw Error(1, "mask sink returned a null destination");
        return d;
    };
    // one finished mask into the caller's hands: written to its destination, or -- for a put
    // callback -- unpacked into this thread's scratch and handed over
    auto deliver = [&](const uint8_t* pbm, int w, int t) {
        if (io.put) {
            thread_local std::vector<uint8_t> scratch;
            scratch.resize(io.layout == FROI_MASK_PBM ? mb : (size_t)g.W * g.H);
            put_mask(g, pbm, io.layout, scratch.data());
            if (io.put(io.sink_user, w, t, scratch.data()) != 0) throw Error(1, "mask put callback failed");
            return;
        }
        put_mask(g, pbm, io.layout, dest(w, t));
    };

    c->times = froi_stage_times{};
    c->ktimes = froi_kernel_times{};
    c->launches = 0;
    const int CH = c->ring_chunk, RF = c->ring_frames;
    std::vector<int> last_reader(RF, -1);     // batch that last reads each ring slot
    std::vector<cudaEvent_t> ready(nk, nullptr);
    size_t next_k = 0, n_chunks = 0, n_staged = 0;
    std::vector<HostPool::TaskPtr> tasks(nb);
    // the previous call's kernels may still read the rings: order this call's copies after them
    FROI_CUDA(cudaEventRecord(c->ev[7], c->stream));
    FROI_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev[7], 0));

    // upload every host frame with index <= kmax that is not resident yet
    auto upload_to = [&](size_t kmax) {
        while (next_k <= kmax && next_k < nk) {
            // first chunk in 8-frame sub-chunks: the first batch's denoise follows the copy
            // exactly the frames this batch still needs, at most one staging chunk, never across
            // the ring's wrap
            const size_t k0 = next_k, cap = k0 < (size_t)CH ? 8 : (size_t)CH;
            const size_t k1 = std::min({nk, kmax + 1, k0 + cap, (k0 / RF + 1) * (size_t)RF});
            next_k = k1;
            bool any = false, direct = true;
            int wait_b = -1;
            for (size_t k = k0; k < k1; ++k) {
                if (!io.host[k]) continue;
                any = true;
                direct &= io.src_bytes == g.sample_bytes && src_pinned[k];
                wait_b = std::max(wait_b, last_reader[k % RF]);
            }
            if (!any) continue;
            if (wait_b >= 0) FROI_CUDA(cudaStreamWaitEvent(c->copy_stream, c->bev[wait_b][7], 0));
            uint8_t* dst = c->d_ring + fb * (k0 % RF);
            if (direct) {
                for (size_t k = k0; k < k1;) {  // contiguous runs of pinned frames: one copy each
                    if (!io.host[k]) {
                        ++k;
                        continue;
                    }
                    size_t e = k + 1;
                    while (e < k1 && io.host[e] && io.host[e] == io.host[e - 1] + fb) ++e;
                    FROI_CUDA(cudaMemcpyAsync(dst + fb * (k - k0), io.host[k], fb * (e - k), cudaMemcpyHostToDevice,
                                              c->copy_stream));
                    k = e;
                }
            } else {
                const size_t slot = n_staged++ % kStageChunks;
                const double tw0 = trace_on() ? now_ms() : 0.0;
                FROI_CUDA(cudaEventSynchronize(c->stage_free[slot]));  // its previous copy is done
                if (trace_on()) t_stage_wait += now_ms() - tw0;
                uint8_t* st = c->h_stage + fb * CH * slot;
                const size_t px = (size_t)g.W * g.H;
                const double tc0 = trace_on() ? now_ms() : 0.0;
                c->pool->parallel_for(k1 - k0, [&](size_t i) {
                    if (io.host[k0 + i]) convert_frame(io.host[k0 + i], io.src_bytes, st + fb * i, g.sample_bytes, px);
                });
                if (trace_on()) t_convert += now_ms() - tc0;
                FROI_CUDA(cudaMemcpyAsync(dst, st, fb * (k1 - k0), cudaMemcpyHostToDevice, c->copy_stream));
                FROI_CUDA(cudaEventRecord(c->stage_free[slot], c->copy_stream));
            }
            if (io.new_carry)  // a well's last frame becomes the next push's carry
                for (size_t k = k0; k < k1; ++k)
                    if ((int)(k % n) == n - 1 && io.host[k])
                        FROI_CUDA(cudaMemcpyAsync(io.new_carry + fb * (k / n), dst + fb * (k - k0), fb,
                                                  cudaMemcpyDeviceToDevice, c->copy_stream));
            cudaEvent_t e = event_at(c->chunk_ready, n_chunks++);
            FROI_CUDA(cudaEventRecord(e, c->copy_stream));
            for (size_t k = k0; k < k1; ++k) ready[k] = e;
        }
    };
    auto frame_ptr = [&](int w, int t) -> const uint8_t* {
        if (t < 0) return io.carry[w];
        const size_t k = (size_t)w * n + t;
        return io.host[k] ? c->d_ring + fb * (k % RF) : io.dev[k];
    };
    froi_ctx* lane = nb >= 2 ? lane_of(c) : nullptr;
    if (lane) {
        FROI_CUDA(cudaEventRecord(c->ev_fork, c->stream));
        FROI_CUDA(cudaStreamWaitEvent(lane->stream, c->ev_fork, 0));
    }
    auto settle = [&] {  // on error: let everything queued finish before buffers are reused
        for (auto& t : tasks)
            if (t) try {
                    t->wait();
                } catch (...) {
                }
        cudaStreamSynchronize(c->copy_stream);
        if (lane) cudaStreamSynchronize(lane->stream);
        cudaStreamSynchronize(c->d2h_stream);
        cudaStreamSynchronize(c->stream);
    };
    try {
        for (size_t b = 0; b < nb; ++b) {
            const size_t j0 = bstart(b), j1 = bstart(b + 1);
            // frames of this batch: uploaded (in order) just before it is enqueued
            size_t kmax = 0;
            for (size_t j = j0; j < j1; ++j) kmax = std::max(kmax, (size_t)wt[j].first * n + wt[j].second);
            upload_to(kmax);
            for (size_t j = j0; j < j1; ++j) {
                const int w = wt[j].first, t = wt[j].second;
                PairJob& J = jobs[j];
                J.raw_prev = frame_ptr(w, t - 1);
                J.raw_next = frame_ptr(w, t);
                const size_t kn = (size_t)w * n + t;
                J.ready = io.host[kn] ? ready[kn] : nullptr;
                if (t > 0 && io.host[kn - 1]) {
                    // prev frame's chunk: the first batch waits on both (frame runs share events)
                    if (!J.ready) J.ready = ready[kn - 1];
                    last_reader[(kn - 1) % RF] = (int)b;
                }
                if (io.host[kn]) last_reader[kn % RF] = (int)b;
                J.out_index = ring_out ? (long long)((b % kOutBatches) * P + (j - j0)) : (long long)kn;
                J.stats_index = (long long)kn;
            }
            froi_ctx* x = (lane && (b & 1)) ? lane : c;
            if (ring_out && b >= (size_t)kOutBatches)  // its egress slot has reached the host
                FROI_CUDA(cudaStreamWaitEvent(x->stream, c->delivered[b - kOutBatches], 0));
            // jobs whose two frames come from different chunks: make the prev chunk's event the
            // one on the frame-slot run (run_batch dedups consecutive frames by pointer)
            run_batch(x, c, jobs, j0, j1, ring_out ? c->d_outring : d_full, b, j0);
            if (!ring_out) continue;
            // ---- egress of batch b
            FROI_CUDA(cudaEventRecord(c->d2h_ev[b], x->stream));
            FROI_CUDA(cudaStreamWaitEvent(c->d2h_stream, c->d2h_ev[b], 0));
            const uint8_t* dsrc = c->d_outring + mb * P * (b % kOutBatches);
            if (!general_out) {
                for (size_t j = j0; j < j1;) {  // runs of contiguous pinned destinations
                    size_t e = j + 1;
                    while (e < j1 && io.mask[(size_t)wt[e].first * n + wt[e].second] ==
                                         io.mask[(size_t)wt[e - 1].first * n + wt[e - 1].second] + mb)
                        ++e;
                    FROI_CUDA(cudaMemcpyAsync(io.mask[(size_t)wt[j].first * n + wt[j].second], dsrc + mb * (j - j0),
                                              mb * (e - j), cudaMemcpyDeviceToHost, c->d2h_stream));
                    j = e;
                }
                if (io.frame0_rule)
                    for (size_t j = j0; j < j1; ++j)
                        if (wt[j].second == 1)
                            FROI_CUDA(cudaMemcpyAsync(io.mask[(size_t)wt[j].first * n], dsrc + mb * (j - j0), mb,
                                                      cudaMemcpyDeviceToHost, c->d2h_stream));
                FROI_CUDA(cudaEventRecord(c->delivered[b], c->d2h_stream));
            } else {
                if (b >= (size_t)kOutBatches) tasks[b - kOutBatches]->wait();  // pinned slot is free
                uint8_t* hslot = c->h_outring + mb * P * (b % kOutBatches);
                FROI_CUDA(cudaMemcpyAsync(hslot, dsrc, mb * (j1 - j0), cudaMemcpyDeviceToHost, c->d2h_stream));
                cudaEvent_t done = c->delivered[b];
                FROI_CUDA(cudaEventRecord(done, c->d2h_stream));
                HostPool* pool = c->dpool.get();
                tasks[b] = c->courier->submit([&, done, hslot, j0, j1, pool] {
                    FROI_CUDA(cudaEventSynchronize(done));
                    pool->parallel_for(j1 - j0, [&](size_t i) {
                        const int w = wt[j0 + i].first, t = wt[j0 + i].second;
                        deliver(hslot + mb * i, w, t);
                        if (io.frame0_rule && t == 1) deliver(hslot + mb * i, w, 0);
                    });
                });
            }
        }
        upload_to(nk ? nk - 1 : 0);  // frames no pair reads (e.g. a push's carry-only tail)
        const double te0 = trace_on() ? now_ms() : 0.0;
        for (auto& t : tasks)
            if (t) t->wait();
        if (trace_on()) t_tail_tasks = now_ms() - te0;
        FROI_CUDA(cudaEventRecord(c->d2h_done, c->d2h_stream));
        FROI_CUDA(cudaStreamWaitEvent(c->stream, c->d2h_done, 0));
        FROI_CUDA(cudaEventRecord(c->ev[6], c->copy_stream));  // carry copies
        FROI_CUDA(cudaStreamWaitEvent(c->stream, c->ev[6], 0));
        if (lane) {
            FROI_CUDA(cudaEventRecord(c->ev_join, lane->stream));
            FROI_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        }
        if (!ring_out) {
            if (io.frame0_rule)
                for (int w = 0; w < nw; ++w)
                    FROI_CUDA(cudaMemcpyAsync(d_full + mb * ((size_t)w * n), d_full + mb * ((size_t)w * n + 1), mb,
                                              cudaMemcpyDeviceToDevice, c->stream));
            if (c->params.adjacent_factor > 0) {  // temporal ensemble (roi.hpp:356-362)
                ensure_seq_tmp(c, mb * n);
                for (int w = 0; w < nw; ++w) {
                    uint8_t* base = d_full + mb * ((size_t)w * n);
                    launch_ensemble(g, base, c->d_seq_tmp, n, c->params.adjacent_factor, c->stream);
                    FROI_CUDA(cudaMemcpyAsync(base, c->d_seq_tmp, mb * n, cudaMemcpyDeviceToDevice, c->stream));
                    ++c->launches;
                }
            }
            if (!io.dev_masks) {  // deliver through the pinned egress twin, kOutBatches*Pcap at a time
                ensure_host_outring(c);
                const size_t step = P * kOutBatches;
                for (size_t m0 = 0; m0 < nk; m0 += step) {
                    const size_t m1 = std::min(nk, m0 + step);
                    FROI_CUDA(cudaMemcpyAsync(c->h_outring, d_full + mb * m0, mb * (m1 - m0), cudaMemcpyDeviceToHost,
                                              c->stream));
                    FROI_CUDA(cudaStreamSynchronize(c->stream));
                    c->pool->parallel_for(m1 - m0, [&](size_t i) {
                        deliver(c->h_outring + mb * i, (int)((m0 + i) / n), (int)((m0 + i) % n));
                    });
                }
            }
        }
        FROI_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
        settle();
        throw;
    }
    accumulate_batch_times(c, nb);
    infos.assign(c->h_info, c->h_info + jobs.size());
    if (trace_on())
        fprintf(stderr, "froi trace: host call %.2f ms: conversion %.2f, staging waits %.2f, delivery tail %.2f (%zu batches)\n",
                now_ms() - t_call0, t_convert, t_stage_wait, t_tail_tasks, nb);
}

// Per-frame stats of a host call: pair rows in (well, frame) order, frame 0 of a well borrows
// frame 1's row with the identity shift (roi.hpp:348-349).
void stats_for_call(froi_ctx* c, const HostCall& io, const std::vector<PairInfo>& infos,
                    froi_frame_stats* stats) {
    if (!stats) return;
    size_t k = 0;
    for (int w = 0; w < io.n_wells; ++w) {
        froi_frame_stats* s = stats + (size_t)w * io.n_frames;
        for (int t = io.t_begin; t < io.n_frames; ++t) fill_stats(c->g, infos[k++], &s[t]);
        if (io.t_begin == 1) {
            s[0] = s[1];
            s[0].dx = 0;
            s[0].dy = 0;
            s[0].confidence = 1.0;
        }
    }
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char* froi_version(void) { return "froi-b200 0.1 (sm_100a)"; }

const char* froi_last_error(void) { return g_last_error.c_str(); }

void froi_params_default(froi_params* p) {
    if (!p) return;
    p->denoise_enabled = 1;
    p->median_radius = 1;
    p->bilateral_sigma_spatial = 2.0;
    p->bilateral_sigma_range = 0.04;
    p->bilateral_radius = 2;
    p->pyramid_levels = 3;
    p->pyramid_scale = 0.5;
    p->window_size = 15;
    p->iterations = 3;
    p->poly_n = 5;
    p->poly_sigma = 1.1;
    p->roi_threshold = 0.2;
    p->flow_weight = 0.7;
    p->adjacent_factor = 0;
    p->min_area = 20;
    p->open_radius = 1;
    p->close_radius = 1;
    p->gradient_source = FROI_GRADIENT_IMAGE;
    p->max_shift = 16;
}

int froi_params_validate(const froi_params* p) {
    const std::string m = validate(p);
    if (!m.empty()) return fail(1, m);
    return 0;
}

int froi_pyramid_levels(const froi_params* p, int width, int height, int* levels_out, int* widths,
                        int* heights) {
    const std::string m = validate(p);
    if (!m.empty()) return fail(1, m);
    if (width <= 0 || height <= 0) return fail(2, "frame dimensions must be positive");
    const std::string gm = check_geometry(*p, width, height);
    if (!gm.empty()) return fail(1, gm);
    const Geom g = make_geom(*p, width, height, 8);
    if (levels_out) *levels_out = g.L;
    for (int l = 0; l < g.L; ++l) {
        if (widths) widths[l] = g.lw[l];
        if (heights) heights[l] = g.lh[l];
    }
    return 0;
}

int froi_device_count(int* count) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = e == cudaSuccess ? n : 0;
    if (e != cudaSuccess) return fail(3, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    return 0;
}

int froi_ctx_create(int device, const froi_params* p, int width, int height, int depth, int max_pairs,
                    froi_ctx** out) {
    if (!out) return fail(1, "out must not be null");
    *out = nullptr;
    const std::string m = validate(p);
    if (!m.empty()) return fail(1, m);
    if (width <= 0 || height <= 0) return fail(2, "frame dimensions must be positive");
    if (depth != 8 && depth != 16) return fail(2, "unsupported bit depth " + std::to_string(depth));
    if (p->max_shift < 1 || p->max_shift >= std::min(width, height) / 4)
        return fail(1, "estimate_shift: max_shift must be in [1, min(w,h)/4)");
    if (next_pow2(width) > 8192 || next_pow2(height) > 8192)
        return fail(1, "frames wider or taller than 8192 px are not supported by the GPU FFT");
    {
        const std::string gm = check_geometry(*p, width, height);
        if (!gm.empty()) return fail(1, gm);
    }
    froi_ctx* c = new froi_ctx();
    ABI_TRY
    c->device = device;
    c->params = *p;
    c->g = make_geom(*p, width, height, depth);
    c->dp = make_dev_params(*p);
    c->f64c = make_flow64_const(*p);
    FROI_CUDA(cudaSetDevice(device));
    FROI_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    if (max_pairs <= 0) {
        const double mpx = double(width) * height / (1024.0 * 1024.0);
        // 64 pairs per batch at 1024^2 (~10.6 GB per execution lane): the level-0 flow grid then
        // fills 13.8 waves instead of 6.9 (one-lane stage time -3.7 %, two-lane frames/s +1.1 %
        // over 32, profiles/tools/pcap_ab.sh); proportionally fewer for larger frames
        max_pairs = std::max(2, std::min(FROI_PCAP_MAX, int(64.0 / std::max(mpx, 0.25))));
    }
    c->Pcap = max_pairs;
    c->Fcap = 2 * max_pairs;
    ctx_alloc(c);
    *out = c;
    return 0;
    }
    catch (const froi::Error& e) {
        ctx_free(c);
        delete c;
        return fail(e.status, e.what());
    }
    catch (const std::exception& e) {
        ctx_free(c);
        delete c;
        return fail(3, e.what());
    }
}

void froi_ctx_destroy(froi_ctx* ctx) {
    if (!ctx) return;
    ctx_free(ctx);
    delete ctx;
}

int froi_ctx_get_params(const froi_ctx* ctx, froi_params* out) {
    if (!ctx || !out) return fail(1, "null argument");
    *out = ctx->params;
    return 0;
}

int froi_ctx_set_params(froi_ctx* ctx, const froi_params* p) {
    if (!ctx) return fail(1, "null context");
    const std::string m = validate(p);
    if (!m.empty()) return fail(1, m);
    const froi_params& o = ctx->params;
    if (p->pyramid_levels != o.pyramid_levels || p->pyramid_scale != o.pyramid_scale ||
        p->max_shift != o.max_shift || p->bilateral_radius != o.bilateral_radius ||
        p->bilateral_sigma_spatial != o.bilateral_sigma_spatial ||
        p->bilateral_sigma_range != o.bilateral_sigma_range)
        return fail(1, "set_params cannot change pyramid geometry, max_shift or bilateral tables; "
                       "create a new context");
    ctx->params = *p;
    ctx->dp = make_dev_params(*p);
    ctx->dp.norm_lut = ctx->d_norm_lut;
    set_grad_params(ctx);
    ctx->f64c = make_flow64_const(*p);
    // captured batch graphs hold the old parameters as kernel arguments
    ABI_TRY
    FROI_CUDA(cudaSetDevice(ctx->device));
    FROI_CUDA(cudaStreamSynchronize(ctx->stream));
    drop_graphs(ctx);
    if (ctx->lane) {
        FROI_CUDA(cudaStreamSynchronize(ctx->lane->stream));
        drop_graphs(ctx->lane);
    }
    ABI_CATCH
}

int froi_ctx_stage_times(const froi_ctx* ctx, froi_stage_times* out) {
    if (!ctx || !out) return fail(1, "null argument");
    *out = ctx->times;
    return 0;
}

int froi_ctx_kernel_times(const froi_ctx* ctx, froi_kernel_times* out) {
    if (!ctx || !out) return fail(1, "null argument");
    *out = ctx->ktimes;
    return 0;
}

int froi_ctx_stream(const froi_ctx* ctx, void** stream_out) {
    if (!ctx || !stream_out) return fail(1, "null argument");
    *stream_out = (void*)ctx->stream;
    return 0;
}

int froi_ctx_set_lanes(froi_ctx* ctx, int lanes) {
    if (!ctx) return fail(1, "null context");
    if (lanes != 1 && lanes != 2) return fail(1, "lanes must be 1 or 2");
    ctx->lanes = lanes;
    return 0;
}

int froi_ctx_set_fork(froi_ctx* ctx, int fork) {
    if (!ctx) return fail(1, "null context");
    if (fork != 0 && fork != 1) return fail(1, "fork must be 0 or 1");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(ctx->device));
    FROI_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->fork = fork != 0;
    drop_graphs(ctx);  // the captured graphs hold the old branch structure
    if (ctx->lane) {
        FROI_CUDA(cudaStreamSynchronize(ctx->lane->stream));
        ctx->lane->fork = ctx->fork;
        drop_graphs(ctx->lane);
    }
    ABI_CATCH
}

int froi_ctx_set_flow_exact(froi_ctx* ctx, int exact) {
    if (!ctx) return fail(1, "null context");
    if (exact != 0 && exact != 1) return fail(1, "exact must be 0 or 1");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(ctx->device));
    FROI_CUDA(cudaStreamSynchronize(ctx->stream));
    if (exact) ensure_flow64(ctx);  // the lane's on its next use (lane_of)
    if (ctx->flow_exact != (exact != 0)) drop_graphs(ctx);  // captured graphs hold the other flow
    ctx->flow_exact = exact != 0;
    ABI_CATCH
}

int froi_ctx_get_flow_exact(const froi_ctx* ctx, int* out) {
    if (!ctx || !out) return fail(1, "null argument");
    *out = ctx->flow_exact ? 1 : 0;
    return 0;
}

int froi_ctx_launch_count(const froi_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return fail(1, "null argument");
    *out = ctx->launches;
    return 0;
}

int froi_extract_wells(froi_ctx* c, const void* frames, int sample_bytes, size_t stride, int n_wells,
                       int n_frames, int layout, uint8_t* masks_out, froi_frame_stats* stats_out) {
    if (!c || !frames || !masks_out) return fail(1, "null argument");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(1, "sample_bytes must be 1 or 2");
    if (!check_layout(layout)) return fail(1, "unknown mask layout");
    if (n_wells < 1) return fail(2, "need at least one well");
    if (n_frames < 2) return fail(2, "extract_roi: sequence needs at least 2 frames");
    if (stride < (size_t)c->g.W * c->g.H * sample_bytes) return fail(1, "frame stride too small");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t nk = (size_t)n_wells * n_frames;
    const size_t ms = layout == FROI_MASK_PBM ? (size_t)c->g.H * c->g.SB : (size_t)c->g.W * c->g.H;
    HostCall io;
    io.n_wells = n_wells;
    io.n_frames = n_frames;
    io.src_bytes = sample_bytes;
    io.layout = layout;
    io.host.resize(nk);
    io.dev.assign(nk, nullptr);
    io.mask.resize(nk);
    for (size_t k = 0; k < nk; ++k) {
        io.host[k] = (const uint8_t*)frames + stride * k;
        io.mask[k] = masks_out + ms * k;
    }
    std::vector<PairInfo> infos;
    run_host_call(c, io, infos);
    stats_for_call(c, io, infos, stats_out);
    ABI_CATCH
}

int froi_extract_roi(froi_ctx* c, const void* frames, int sample_bytes, size_t stride, int n_frames,
                     int layout, uint8_t* masks_out, froi_frame_stats* stats_out) {
    return froi_extract_wells(c, frames, sample_bytes, stride, 1, n_frames, layout, masks_out, stats_out);
}

int froi_extract_frames_put(froi_ctx* c, const void* const* frames, int sample_bytes, int n_frames,
                            int layout, froi_mask_put put, void* user, froi_frame_stats* stats_out) {
    if (!c || !frames || !put) return fail(1, "null argument");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(1, "sample_bytes must be 1 or 2");
    if (!check_layout(layout)) return fail(1, "unknown mask layout");
    if (n_frames < 2) return fail(2, "extract_roi: sequence needs at least 2 frames");
    for (int t = 0; t < n_frames; ++t)
        if (!frames[t]) return fail(1, "null frame pointer");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    HostCall io;
    io.n_wells = 1;
    io.n_frames = n_frames;
    io.src_bytes = sample_bytes;
    io.layout = layout;
    io.host.assign((const uint8_t* const*)frames, (const uint8_t* const*)frames + n_frames);
    io.dev.assign(n_frames, nullptr);
    io.put = put;
    io.sink_user = user;
    std::vector<PairInfo> infos;
    run_host_call(c, io, infos);
    stats_for_call(c, io, infos, stats_out);
    ABI_CATCH
}

int froi_extract_frames_sink(froi_ctx* c, const void* const* frames, int sample_bytes, int n_frames,
                             int layout, froi_mask_sink sink, void* user, froi_frame_stats* stats_out) {
    if (!c || !frames || !sink) return fail(1, "null argument");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(1, "sample_bytes must be 1 or 2");
    if (!check_layout(layout)) return fail(1, "unknown mask layout");
    if (n_frames < 2) return fail(2, "extract_roi: sequence needs at least 2 frames");
    for (int t = 0; t < n_frames; ++t)
        if (!frames[t]) return fail(1, "null frame pointer");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    HostCall io;
    io.n_wells = 1;
    io.n_frames = n_frames;
    io.src_bytes = sample_bytes;
    io.layout = layout;
    io.host.assign((const uint8_t* const*)frames, (const uint8_t* const*)frames + n_frames);
    io.dev.assign(n_frames, nullptr);
    io.sink = sink;
    io.sink_user = user;
    std::vector<PairInfo> infos;
    run_host_call(c, io, infos);
    stats_for_call(c, io, infos, stats_out);
    ABI_CATCH
}

int froi_extract_frames(froi_ctx* c, const void* const* frames, int sample_bytes, int n_frames, int layout,
                        uint8_t* const* masks, froi_frame_stats* stats_out) {
    if (!c || !frames || !masks) return fail(1, "null argument");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(1, "sample_bytes must be 1 or 2");
    if (!check_layout(layout)) return fail(1, "unknown mask layout");
    if (n_frames < 2) return fail(2, "extract_roi: sequence needs at least 2 frames");
    for (int t = 0; t < n_frames; ++t)
        if (!frames[t] || !masks[t]) return fail(1, "null frame or mask pointer");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    HostCall io;
    io.n_wells = 1;
    io.n_frames = n_frames;
    io.src_bytes = sample_bytes;
    io.layout = layout;
    io.host.assign((const uint8_t* const*)frames, (const uint8_t* const*)frames + n_frames);
    io.dev.assign(n_frames, nullptr);
    io.mask.assign(masks, masks + n_frames);
    std::vector<PairInfo> infos;
    run_host_call(c, io, infos);
    stats_for_call(c, io, infos, stats_out);
    ABI_CATCH
}

int froi_extract_wells_device(froi_ctx* c, const void* d_frames, int sample_bytes, size_t stride,
                              int n_wells, int n_frames, uint8_t* d_masks_pbm,
                              froi_frame_stats* stats_out) {
    if (!c || !d_frames || !d_masks_pbm) return fail(1, "null argument");
    if (sample_bytes != c->g.sample_bytes) return fail(1, "device frames must use the context sample width");
    if (n_wells < 1) return fail(2, "need at least one well");
    if (n_frames < 2) return fail(2, "extract_roi: sequence needs at least 2 frames");
    if (stride < c->frame_bytes) return fail(1, "frame stride too small");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    std::vector<PairInfo> infos;
    extract_wells_dev(c, (const uint8_t*)d_frames, stride, n_wells, n_frames, d_masks_pbm, infos);
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    stats_for_wells(c, infos, n_wells, n_frames, stats_out);
    ABI_CATCH
}

int froi_stream_reset(froi_ctx* c, int n_wells) {
    if (!c) return fail(1, "null context");
    if (n_wells < 1) return fail(2, "need at least one well");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    c->stream_wells = n_wells;
    c->stream_next_t.assign(n_wells, 0);
    const size_t need = c->frame_bytes * n_wells;
    if (c->carry_cap < need) {
        for (auto& d : c->d_carry) {
            if (d) FROI_CUDA(cudaFree(d));
            d = nullptr;
        }
        c->carry_cap = 0;
        for (auto& d : c->d_carry) FROI_CUDA(cudaMalloc(&d, need));
        c->carry_cap = need;
    }
    ABI_CATCH
}

}  // extern "C"

namespace {
// Shared body of froi_stream_push / froi_stream_push_frames: frame k = w*chunk + t at
// frame_at(k), mask k at mask_at(k) (host) or masks_out + k*mb (device PBM).
template <typename FrameAt, typename MaskAt>
int stream_push_impl(froi_ctx* c, FrameAt frame_at, int frames_on_device, int sample_bytes, int chunk,
                     int layout, MaskAt mask_at, uint8_t* dev_masks, froi_frame_stats* stats_out) {
    const bool first = c->stream_next_t[0] == 0;
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const int nw = c->stream_wells;
    const size_t nk = (size_t)nw * chunk, fb = c->frame_bytes;
    // the pushed frames stream through the same rings as froi_extract_wells; the previous push's
    // last frame of each well (the carry) is the first pair's prev, and this push's last frames
    // become the next carry (double-buffered, so reading one never races writing the other)
    HostCall io;
    io.n_wells = nw;
    io.n_frames = chunk;
    io.t_begin = first ? 1 : 0;
    io.frame0_rule = first;
    io.src_bytes = sample_bytes;
    io.layout = layout;
    io.host.assign(nk, nullptr);
    io.dev.assign(nk, nullptr);
    for (size_t k = 0; k < nk; ++k) (frames_on_device ? io.dev[k] : io.host[k]) = frame_at(k);
    for (int w = 0; w < nw; ++w) io.carry.push_back(c->d_carry[c->carry_cur] + fb * w);
    uint8_t* next_carry = c->d_carry[1 - c->carry_cur];
    if (!frames_on_device) io.new_carry = next_carry;
    if (dev_masks) io.dev_masks = dev_masks;
    else {
        io.mask.resize(nk);
        for (size_t k = 0; k < nk; ++k) io.mask[k] = mask_at(k);
    }
    std::vector<PairInfo> infos;
    run_host_call(c, io, infos);
    if (frames_on_device) {
        for (int w = 0; w < nw; ++w)
            FROI_CUDA(cudaMemcpyAsync(next_carry + fb * w, io.dev[(size_t)w * chunk + chunk - 1], fb,
                                      cudaMemcpyDeviceToDevice, c->stream));
        FROI_CUDA(cudaStreamSynchronize(c->stream));
    }
    c->carry_cur = 1 - c->carry_cur;
    stats_for_call(c, io, infos, stats_out);
    for (int w = 0; w < nw; ++w) c->stream_next_t[w] += chunk;
    ABI_CATCH
}

int stream_push_checks(froi_ctx* c, int frames_on_device, int sample_bytes, int chunk, int layout,
                       int masks_on_device) {
    if (c->stream_wells < 1) return fail(1, "froi_stream_reset first");
    if (c->params.adjacent_factor != 0) return fail(1, "streaming requires adjacent_factor == 0");
    if (!check_layout(layout)) return fail(1, "unknown mask layout");
    if (masks_on_device && layout != FROI_MASK_PBM) return fail(1, "device masks are PBM only");
    if (chunk < 1) return fail(2, "chunk must be >= 1");
    if (sample_bytes != 1 && sample_bytes != 2) return fail(1, "sample_bytes must be 1 or 2");
    if (c->stream_next_t[0] == 0 && chunk < 2) return fail(2, "the first push of a sequence needs at least 2 frames");
    if (frames_on_device && sample_bytes != c->g.sample_bytes)
        return fail(1, "device frames must use the context sample width");
    return 0;
}
}  // namespace

extern "C" {

int froi_stream_push_frames(froi_ctx* c, const void* const* frames, int sample_bytes, int chunk, int layout,
                            uint8_t* const* masks, froi_frame_stats* stats_out) {
    if (!c || !frames || !masks) return fail(1, "null argument");
    if (int rc = stream_push_checks(c, 0, sample_bytes, chunk, layout, 0)) return rc;
    const size_t nk = (size_t)c->stream_wells * chunk;
    for (size_t k = 0; k < nk; ++k)
        if (!frames[k] || !masks[k]) return fail(1, "null frame or mask pointer");
    return stream_push_impl(
        c, [&](size_t k) { return (const uint8_t*)frames[k]; }, 0, sample_bytes, chunk, layout,
        [&](size_t k) { return masks[k]; }, nullptr, stats_out);
}

int froi_stream_push(froi_ctx* c, const void* frames, int frames_on_device, int sample_bytes,
                     size_t stride, int chunk, int layout, uint8_t* masks_out, int masks_on_device,
                     froi_frame_stats* stats_out) {
    if (!c || !frames || !masks_out) return fail(1, "null argument");
    if (int rc = stream_push_checks(c, frames_on_device, sample_bytes, chunk, layout, masks_on_device)) return rc;
    if (stride < (size_t)c->g.W * c->g.H * sample_bytes) return fail(1, "frame stride too small");
    const size_t ms = layout == FROI_MASK_PBM ? (size_t)c->g.H * c->g.SB : (size_t)c->g.W * c->g.H;
    return stream_push_impl(
        c, [&](size_t k) { return (const uint8_t*)frames + stride * k; }, frames_on_device, sample_bytes, chunk,
        layout, [&](size_t k) { return masks_out + ms * k; }, masks_on_device ? masks_out : nullptr, stats_out);
}

// ------------------------------------------------------------------ sub-operator taps
namespace {

// Puts 1..2 host uint16 frames into raw slots 0..n-1 (converted to the context sample type).
void taps_upload(froi_ctx* c, const uint16_t* const* frames, int n) {
    for (int i = 0; i < n; ++i) upload_frames(c, frames[i], 2, (size_t)c->g.W * c->g.H * 2, 1, c->d_raw + c->frame_bytes * i);
    const void* ptrs[2] = {c->d_raw, c->d_raw + c->frame_bytes};
    FROI_CUDA(cudaMemcpyAsync(c->d_frame_raw[0], ptrs, sizeof(void*) * 2, cudaMemcpyHostToDevice, c->stream));
    const int prev = 0, next = 1;
    FROI_CUDA(cudaMemcpyAsync(c->d_prev[0], &prev, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    FROI_CUDA(cudaMemcpyAsync(c->d_next[0], &next, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    const long long zero = 0;
    FROI_CUDA(cudaMemcpyAsync(c->d_out_index[0], &zero, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
}

void taps_copy_den(froi_ctx* c, int n) {  // den := raw, sums (denoise disabled)
    DevParams d = c->dp;
    d.denoise_enabled = 0;
    FROI_CUDA(cudaMemsetAsync(c->d_sums, 0, sizeof(unsigned long long) * n, c->stream));
    launch_denoise(c->g, d, c->d_frame_raw[0], c->d_den, c->d_sums, c->h_spatial.data(), c->d_lut, n, c->stream);
}

void taps_set_info(froi_ctx* c, int dx, int dy) {
    PairInfo I{};
    I.dx = dx;
    I.dy = dy;
    I.shifted = 0;  // taps never use the shifted-expansion buffers
    I.confidence = 1.0;
    FROI_CUDA(cudaMemcpyAsync(c->d_info, &I, sizeof(I), cudaMemcpyHostToDevice, c->stream));
}

void words_to_bytes(const Geom& g, const std::vector<uint32_t>& words, uint8_t* out) {
    for (int y = 0; y < g.H; ++y)
        for (int x = 0; x < g.W; ++x) out[(size_t)y * g.W + x] = (words[(size_t)y * g.WW + (x >> 5)] >> (x & 31)) & 1u;
}

void pbm_to_bytes(const Geom& g, const std::vector<uint8_t>& pbm, uint8_t* out) {
    for (int y = 0; y < g.H; ++y)
        for (int x = 0; x < g.W; ++x) out[(size_t)y * g.W + x] = (pbm[(size_t)y * g.SB + (x >> 3)] >> (7 - (x & 7))) & 1u;
}

void upload_mask_words(froi_ctx* c, const uint8_t* mask) {
    const size_t px = (size_t)c->g.W * c->g.H;
    ensure_seq_tmp(c, px);
    FROI_CUDA(cudaMemcpyAsync(c->d_seq_tmp, mask, px, cudaMemcpyHostToDevice, c->stream));
    launch_pack_bytes_to_words(c->g, c->d_seq_tmp, c->d_bits_thr, c->stream);
}

void upload_flow(froi_ctx* c, const float* u, const float* v) {
    const size_t px = (size_t)c->g.W * c->g.H;
    std::vector<float2> f(px);
    for (size_t i = 0; i < px; ++i) f[i] = make_float2(u[i], v[i]);
    // on the context stream (non-blocking: the legacy stream would not order it), and complete
    // before the staging vector goes away
    FROI_CUDA(cudaMemcpyAsync(c->d_flow0, f.data(), sizeof(float2) * px, cudaMemcpyHostToDevice, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace

int froi_denoise(froi_ctx* c, const uint16_t* in, uint16_t* out) {
    if (!c || !in || !out) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const uint16_t* fr[1] = {in};
    taps_upload(c, fr, 1);
    FROI_CUDA(cudaMemsetAsync(c->d_sums, 0, sizeof(unsigned long long), c->stream));
    launch_denoise(c->g, c->dp, c->d_frame_raw[0], c->d_den, c->d_sums, c->h_spatial.data(), c->d_lut, 1, c->stream);
    const size_t px = (size_t)c->g.W * c->g.H;
    std::vector<uint8_t> h(c->frame_bytes);
    FROI_CUDA(cudaMemcpyAsync(h.data(), c->d_den, c->frame_bytes, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < px; ++i) out[i] = c->g.sample_bytes == 1 ? h[i] : ((const uint16_t*)h.data())[i];
    ABI_CATCH
}

int froi_estimate_shift(froi_ctx* c, const uint16_t* reference, const uint16_t* moving, int max_shift,
                        froi_shift* out) {
    if (!c || !reference || !moving || !out) return fail(1, "null argument");
    if (max_shift < 1 || max_shift >= std::min(c->g.W, c->g.H) / 4)
        return fail(1, "estimate_shift: max_shift must be in [1, min(w,h)/4)");
    if (max_shift > c->params.max_shift) return fail(1, "max_shift exceeds the context's max_shift");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const uint16_t* fr[2] = {reference, moving};
    taps_upload(c, fr, 2);
    taps_copy_den(c, 2);
    launch_fft_forward(c->g, c->d_den, c->d_sums, c->d_wx, c->d_wy, c->d_tw_row, c->d_tw_col, c->d_spec, 2, c->stream);
    DevParams d = c->dp;
    d.max_shift = max_shift;
    launch_register_pairs(c->g, d, c->d_spec, c->d_prev[0], c->d_next[0], c->d_itw_row, c->d_itw_col, c->d_cols,
                          c->d_surf, c->d_info, 1, c->stream);
    PairInfo I;
    FROI_CUDA(cudaMemcpyAsync(&I, c->d_info, sizeof(I), cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    out->dx = I.est_dx;
    out->dy = I.est_dy;
    out->confidence = I.confidence;
    ABI_CATCH
}

int froi_compute_flow(froi_ctx* c, const uint16_t* prev, const uint16_t* next, float* u, float* v) {
    if (!c || !prev || !next || !u || !v) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const uint16_t* fr[2] = {prev, next};
    taps_upload(c, fr, 2);
    taps_copy_den(c, 2);
    FlowBuffers fb = c->flow_buffers();
    taps_set_info(c, 0, 0);
    int cur = 0;
    if (c->flow_exact) {
        const Flow64Buffers fb64 = c->flow64_buffers();
        launch_expand_frames64(c->g, c->f64c, fb64, c->d_den, 2, c->stream);
        launch_flow64(c->g, c->dp, fb64, c->d_prev[0], c->d_next[0], c->d_info, 1, c->stream, &cur);
    } else {
        launch_expand_frames(c->g, c->dp, fb, 2, c->stream);
        cur = launch_flow(c->g, c->dp, fb, c->d_prev[0], c->d_next[0], c->d_info, 1, c->stream);
    }
    const size_t px = (size_t)c->g.W * c->g.H;
    std::vector<float2> f(px);
    FROI_CUDA(cudaMemcpyAsync(f.data(), cur ? c->d_flow1 : c->d_flow0, sizeof(float2) * px, cudaMemcpyDeviceToHost,
                              c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < px; ++i) {
        u[i] = f[i].x;
        v[i] = f[i].y;
    }
    ABI_CATCH
}

int froi_polynomial_expansion(froi_ctx* c, const float* image, float* planes) {
    if (!c || !image || !planes) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)c->g.W * c->g.H;
    float* d_img = nullptr;
    FROI_CUDA(cudaMalloc(&d_img, sizeof(float) * 7 * px));
    struct Guard {
        float* p;
        ~Guard() { cudaFree(p); }
    } guard{d_img};
    float* d_planes = d_img + px;
    FROI_CUDA(cudaMemcpyAsync(d_img, image, sizeof(float) * px, cudaMemcpyHostToDevice, c->stream));
    launch_expand_image(c->g, c->dp, d_img, d_planes, c->stream);
    FROI_CUDA(cudaMemcpyAsync(planes, d_planes, sizeof(float) * 6 * px, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    ABI_CATCH
}

int froi_saliency(froi_ctx* c, const float* u, const float* v, const uint16_t* frame, double* out) {
    if (!c || !u || !v || !frame || !out) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const uint16_t* fr[1] = {frame};
    taps_upload(c, fr, 1);
    const void* rp = c->d_raw;
    FROI_CUDA(cudaMemcpyAsync(c->d_pair_raw[0], &rp, sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    upload_flow(c, u, v);
    taps_set_info(c, 0, 0);
    const size_t px = (size_t)c->g.W * c->g.H;
    double* d_out = (double*)c->d_flow1;
    MaskBuffers mb = c->mask_buffers(0);
    mb.flow = c->d_flow0;
    launch_saliency_map(c->g, c->dp, mb, d_out, c->stream);
    FROI_CUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * px, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    ABI_CATCH
}

int froi_threshold_mask(froi_ctx* c, const double* map, double roi_threshold, uint8_t* mask) {
    if (!c || !map || !mask) return fail(1, "null argument");
    if (!(roi_threshold > 0.0 && roi_threshold < 1.0))
        return fail(1, "threshold_mask: roi_threshold must be in (0,1)");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)c->g.W * c->g.H;
    double* d_map = (double*)c->d_flow1;
    FROI_CUDA(cudaMemcpyAsync(d_map, map, sizeof(double) * px, cudaMemcpyHostToDevice, c->stream));
    taps_set_info(c, 0, 0);
    MaskBuffers mb = c->mask_buffers(0);
    mb.flow = c->d_flow0;
    launch_threshold_from_map(c->g, c->dp, mb, d_map, roi_threshold, c->stream);
    std::vector<uint32_t> words((size_t)c->g.H * c->g.WW);
    FROI_CUDA(cudaMemcpyAsync(words.data(), c->d_bits_thr, words.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    words_to_bytes(c->g, words, mask);
    ABI_CATCH
}

int froi_morph_cleanup(froi_ctx* c, uint8_t* mask, int open_radius, int close_radius, int min_area) {
    if (!c || !mask) return fail(1, "null argument");
    if (open_radius < 0 || close_radius < 0 || open_radius > 31 || close_radius > 31)
        return fail(1, "roi: radii must be in [0, 31]");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    upload_mask_words(c, mask);
    taps_set_info(c, 0, 0);
    const long long zero = 0;
    FROI_CUDA(cudaMemcpyAsync(c->d_out_index[0], &zero, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    MaskBuffers mb = c->mask_buffers(0);
    mb.flow = c->d_flow0;
    launch_cleanup_only(c->g, c->dp, mb, open_radius, close_radius, min_area, c->stream);
    std::vector<uint8_t> pbm((size_t)c->g.H * c->g.SB);
    FROI_CUDA(cudaMemcpyAsync(pbm.data(), c->d_out_batch, pbm.size(), cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    pbm_to_bytes(c->g, pbm, mask);
    ABI_CATCH
}

static int dwt_check(froi_ctx* c, int levels) {
    if (levels < 1) return fail(1, "dwt: levels must be >= 1");
    if (c->g.W < (1 << levels) || c->g.H < (1 << levels))
        return fail(2, "dwt: frame too small for " + std::to_string(levels) + " levels");
    return 0;
}

int froi_dwt_forward(froi_ctx* c, const uint16_t* frame, int levels, int32_t* coeffs) {
    if (!c || !frame || !coeffs) return fail(1, "null argument");
    if (int rc = dwt_check(c, levels)) return rc;
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)c->g.W * c->g.H;
    uint16_t* d_in = nullptr;
    int32_t* d_c = nullptr;
    FROI_CUDA(cudaMalloc(&d_in, px * sizeof(uint16_t)));
    FROI_CUDA(cudaMalloc(&d_c, px * sizeof(int32_t)));
    try {
        FROI_CUDA(cudaMemcpyAsync(d_in, frame, px * sizeof(uint16_t), cudaMemcpyHostToDevice, c->stream));
        launch_dwt_forward(d_in, 2, c->g.W, c->g.H, c->g.depth, 1, levels, d_c, c->stream);
        FROI_CUDA(cudaMemcpyAsync(coeffs, d_c, px * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        FROI_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
        cudaFree(d_in);
        cudaFree(d_c);
        throw;
    }
    cudaFree(d_in);
    cudaFree(d_c);
    ABI_CATCH
}

int froi_dwt_inverse(froi_ctx* c, const int32_t* coeffs, int levels, uint16_t* frame) {
    if (!c || !frame || !coeffs) return fail(1, "null argument");
    if (int rc = dwt_check(c, levels)) return rc;
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)c->g.W * c->g.H;
    uint16_t* d_out = nullptr;
    int32_t* d_c = nullptr;
    FROI_CUDA(cudaMalloc(&d_out, px * sizeof(uint16_t)));
    FROI_CUDA(cudaMalloc(&d_c, px * sizeof(int32_t)));
    try {
        FROI_CUDA(cudaMemcpyAsync(d_c, coeffs, px * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
        launch_dwt_inverse(d_c, c->g.W, c->g.H, c->g.depth, 1, levels, d_out, c->stream);
        FROI_CUDA(cudaMemcpyAsync(frame, d_out, px * sizeof(uint16_t), cudaMemcpyDeviceToHost, c->stream));
        FROI_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
        cudaFree(d_out);
        cudaFree(d_c);
        throw;
    }
    cudaFree(d_out);
    cudaFree(d_c);
    ABI_CATCH
}

int froi_dwt_forward_device(froi_ctx* c, const void* d_frames, int n, int levels, int32_t* d_coeffs) {
    if (!c || !d_frames || !d_coeffs) return fail(1, "null argument");
    if (n < 1) return fail(2, "need at least one frame");
    if (int rc = dwt_check(c, levels)) return rc;
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    launch_dwt_forward(d_frames, c->g.sample_bytes, c->g.W, c->g.H, c->g.depth, n, levels, d_coeffs, c->stream);
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    ABI_CATCH
}

int froi_map_mask_to_subbands(froi_ctx* c, const uint8_t* mask, int levels, uint8_t* out, size_t cap,
                              size_t* out_len) {
    if (!c || !mask || !out || !out_len) return fail(1, "null argument");
    if (levels < 1) return fail(1, "map_mask_to_subbands: levels must be >= 1");
    const int W = c->g.W, H = c->g.H;
    size_t total = 0;
    for (int l = 1, w = W, h = H; l <= levels; ++l) {
        w = (w + 1) / 2;
        h = (h + 1) / 2;
        total += (size_t)w * h;
    }
    *out_len = total;
    if (cap < total) return fail(1, "map_mask_to_subbands: output buffer too small");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)W * H;
    bool any = false;
    for (size_t i = 0; i < px && !any; ++i) any = mask[i] != 0;
    uint8_t *d_m = nullptr, *d_o = nullptr;
    FROI_CUDA(cudaMalloc(&d_m, px));
    FROI_CUDA(cudaMalloc(&d_o, total));
    try {
        FROI_CUDA(cudaMemcpyAsync(d_m, mask, px, cudaMemcpyHostToDevice, c->stream));
        launch_map_mask_to_subbands(d_m, W, H, levels, any, d_o, c->stream);
        FROI_CUDA(cudaMemcpyAsync(out, d_o, total, cudaMemcpyDeviceToHost, c->stream));
        FROI_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
        cudaFree(d_m);
        cudaFree(d_o);
        throw;
    }
    cudaFree(d_m);
    cudaFree(d_o);
    ABI_CATCH
}

int froi_component_areas(froi_ctx* c, const uint8_t* mask, uint32_t* areas_out, size_t cap,
                         size_t* n_components) {
    if (!c || !mask || !n_components) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    upload_mask_words(c, mask);
    taps_set_info(c, 0, 0);
    const long long zero = 0;
    FROI_CUDA(cudaMemcpyAsync(c->d_out_index[0], &zero, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    MaskBuffers mb = c->mask_buffers(0);
    mb.flow = c->d_flow0;
    launch_cleanup_only(c->g, c->dp, mb, 0, 0, 2, c->stream);  // no morphology, CCL forced
    const Geom& g = c->g;
    const size_t runs = (size_t)g.H * g.RMAX;
    std::vector<int> rn(g.H), par(runs);
    std::vector<unsigned int> area(runs);
    FROI_CUDA(cudaMemcpyAsync(rn.data(), c->d_run_n, sizeof(int) * g.H, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaMemcpyAsync(par.data(), c->d_run_par, sizeof(int) * runs, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaMemcpyAsync(area.data(), c->d_run_area, sizeof(unsigned int) * runs, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    size_t n = 0;
    for (int y = 0; y < g.H; ++y)
        for (int k = 0; k < rn[y]; ++k) {
            const int id = y * g.RMAX + k;
            if (par[id] != id) continue;  // not a component root
            if (areas_out && n < cap) areas_out[n] = area[id];
            ++n;
        }
    *n_components = n;
    ABI_CATCH
}

int froi_mask_from_flow(froi_ctx* c, const float* u, const float* v, const uint16_t* raw_frame, int dx,
                        int dy, uint8_t* mask, froi_frame_stats* stats) {
    if (!c || !u || !v || !raw_frame || !mask) return fail(1, "null argument");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const uint16_t* fr[1] = {raw_frame};
    taps_upload(c, fr, 1);
    const void* rp = c->d_raw;
    FROI_CUDA(cudaMemcpyAsync(c->d_pair_raw[0], &rp, sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    upload_flow(c, u, v);
    taps_set_info(c, dx, dy);
    MaskBuffers mb = c->mask_buffers(0);
    mb.flow = c->d_flow0;
    uint64_t l = 0;
    launch_mask_stage(c->g, c->dp, mb, 1, c->stream, &l);
    std::vector<uint8_t> pbm((size_t)c->g.H * c->g.SB);
    PairInfo I;
    FROI_CUDA(cudaMemcpyAsync(pbm.data(), c->d_out_batch, pbm.size(), cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaMemcpyAsync(&I, c->d_info, sizeof(I), cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    pbm_to_bytes(c->g, pbm, mask);
    if (stats) fill_stats(c->g, I, stats);
    ABI_CATCH
}

int froi_debug_pair_stats(froi_ctx* c, int pair, double* out, int n) {
    if (!c || !out) return fail(1, "null argument");
    if (pair < 0 || pair >= c->Pcap) return fail(1, "pair slot out of range");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    PairInfo I;
    FROI_CUDA(cudaMemcpy(&I, c->d_info + pair, sizeof(I), cudaMemcpyDeviceToHost));
    const double v[9] = {I.fmag_lo, I.fmag_hi, I.grad_lo, I.grad_hi, I.boundary, (double)I.count_gt,
                         (double)I.need, (double)I.target, (double)I.thr_mode};
    for (int i = 0; i < n && i < 9; ++i) out[i] = v[i];
    ABI_CATCH
}

int froi_temporal_ensemble(froi_ctx* c, const uint8_t* masks, int n, int k, uint8_t* out) {
    if (!c || !masks || !out) return fail(1, "null argument");
    if (n < 1) return fail(2, "temporal_ensemble: need at least one mask");
    if (k < 0) return fail(1, "roi: adjacent_factor must be >= 0");
    ABI_TRY
    FROI_CUDA(cudaSetDevice(c->device));
    const size_t px = (size_t)c->g.W * c->g.H;
    ensure_seq_tmp(c, 2 * px * n);
    FROI_CUDA(cudaMemcpyAsync(c->d_seq_tmp, masks, px * n, cudaMemcpyHostToDevice, c->stream));
    Geom g1 = c->g;  // byte-per-pixel layout: treat each row as W "bytes"
    g1.SB = g1.W;
    launch_ensemble(g1, c->d_seq_tmp, c->d_seq_tmp + px * n, n, k, c->stream);
    FROI_CUDA(cudaMemcpyAsync(out, c->d_seq_tmp + px * n, px * n, cudaMemcpyDeviceToHost, c->stream));
    FROI_CUDA(cudaStreamSynchronize(c->stream));
    ABI_CATCH
}

}  // extern "C"
