// k_mask.cu — mask stage (roi.hpp:47-246, registration.hpp:111-121), bit-exact given the flow.
//
// Per pair, on the level-0 flow (registered coordinates) and the raw frame t:
//   saliency   S = w*N(|flow|) + (1.0-w)*N(|grad I|) recomputed on the fly wherever needed:
//              |flow| is glibc hypotf (float), |grad I| the restated glibc hypot of central
//              differences of apply_shift(raw, s)/maxval, N the 1st/99th-percentile clamp.
//   selection  exact order statistics on the IEEE bit patterns (integer histograms, no float
//              atomics): the first pass bins keys by an exponent window (sign | exponent | 7
//              mantissa bits over 31 octaves), which normally isolates few enough keys (<= 16384)
//              to collect and finish by an 8-bit-digit radix select in shared memory; 11-bit
//              radix digits remain the fallback.  The four percentiles run as one set of passes,
//              then the round(t*n)-th largest saliency; a pass also records min/max of the
//              still-matching keys so tied groups finish early.
//   threshold  S > boundary plus ties admitted in row-major order (per-chunk tie counts, an
//              exclusive scan, then warp-ballot ranks), written as 32-bit packed words.
//   cleanup    open(r_o) then close(r_c) on packed words in shared memory (square windows,
//              shrinking at the borders), then 8-connected CCL: tile-local union-find in shared
//              memory, boundary merge with atomicMin union-find in global memory, area sums at
//              the roots, area filter (min_area).
//   output     unshift (zero fill) fused with the area filter into PBM-layout bytes
//              (MSB first, row stride ceil(W/8)), plus the pixel count and component count.
#include "kernels.cuh"

namespace froi {
namespace {

// ------------------------------------------------------------------ per-pixel sources
template <typename T>
struct PairPix {
    const float2* flow;
    const T* raw;
    int W, H, dx, dy;
    double inv_maxval;
    int grad_src;
    const double* lut;  // shared-memory v/maxval table for 8-bit frames (nullptr: convert)

    __device__ __forceinline__ float fmag(int x, int y) const {
        const float2 f = flow[y * W + x];
        return hypotf_glibc(f.x, f.y);
    }
    // normalize_frame(apply_shift(raw, s)) at clamped coordinates
    __device__ __forceinline__ double img(int x, int y) const {
        const int sx = clampi(clampi(x, 0, W - 1) + dx, 0, W - 1);
        const int sy = clampi(clampi(y, 0, H - 1) + dy, 0, H - 1);
        const int v = raw[sy * W + sx];
        return sizeof(T) == 1 ? lut[v] : dmul((double)v, inv_maxval);  // 8-bit: shared table (k_mag_grad)
    }
    // gradient_magnitude (roi.hpp:65-74)
    __device__ __forceinline__ double grad(int x, int y) const {
        double gx, gy;
        if (grad_src == 0) {
            gx = dmul(0.5, dsub(img(x + 1, y), img(x - 1, y)));
            gy = dmul(0.5, dsub(img(x, y + 1), img(x, y - 1)));
        } else {
            gx = dmul(0.5, dsub((double)fmag(min(x + 1, W - 1), y), (double)fmag(max(x - 1, 0), y)));
            gy = dmul(0.5, dsub((double)fmag(x, min(y + 1, H - 1)), (double)fmag(x, max(y - 1, 0))));
        }
        return hypot_glibc(gx, gy);
    }
};

// Branch-free: a degenerate range has inv = 0, so t is +-0 -- the same key and the same order as
// the reference's 0 (keys map -0 to +0; -0 + x == x for x != 0).  `zero` is kept for callers.
__device__ __forceinline__ double normalize(double v, double lo, double inv, int zero) {
    (void)zero;
    const double t = dmul(dsub(v, lo), inv);
    return t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
}

template <typename T>
__device__ __forceinline__ PairPix<T> make_pix(const Geom& g, const DevParams& P,
                                               const MaskBuffers& b, const PairInfo& I, int p) {
    PairPix<T> px;
    px.flow = opaque(b.flow + (size_t)p * b.flow_stride);
    px.raw = (const T*)b.raw[p];
    px.W = g.W;
    px.H = g.H;
    px.dx = I.dx;
    px.dy = I.dy;
    px.inv_maxval = 1.0 / (double)g.maxval;
    px.grad_src = P.gradient_source;
    px.lut = nullptr;
    return px;
}

// ------------------------------------------------------------------ radix select
// Exact k-th order statistics over 64-bit keys (IEEE bit patterns of non-negative doubles).
// Each query walks MSD digits of 11 bits with integer histograms; a pass also records min/max of
// the keys still matching the prefix (all equal -> done), and once the selected bin holds at most
// kSelCap keys the next pass collects them and k_sel_scan finishes them in shared memory.  The
// first pass uses an exponent-window digit; for phase A it is fused into the producer that
// materialises |flow| and |grad I|.
constexpr int SNT = 512;

// |flow| keys: the float's own bit pattern in the high word (monotone for non-negative floats,
// no float->double conversion per element); |grad I| and S keys: the double's bit pattern.
__device__ __forceinline__ unsigned long long fkey(float f) {
    return f == 0.f ? 0ull : ((unsigned long long)__float_as_uint(f) << 32);
}
__device__ __forceinline__ double ffromkey(unsigned long long k) {
    return (double)__uint_as_float((unsigned int)(k >> 32));
}

__device__ __forceinline__ void sel_digit(int bits_done, int& shift, int& width) {
    width = min(kSelBits, 64 - bits_done);
    shift = 64 - bits_done - width;
}


// Exponent-window first digit: for a non-negative key, bin 1 + 128*(e - e0) + (top 7 mantissa
// bits) over the 31 octaves [2^-26, 2^5), bin 0 below (zero included), bin kFpwBins-1 above.  A
// regular bin is exactly the key prefix sign|exponent|7 mantissa bits (19 bits for a double, 16
// for an fkey), so one pass resolves the 1/128 of an octave holding the rank -- typically few
// enough keys to collect directly.  Ranks in the two open bins fall back to radix digits.
constexpr int kFpwOct = 31, kFpwSub = 7, kFpwBins = 2 + (kFpwOct << kFpwSub);
static_assert(kFpwBins <= kHistBins, "exponent window must fit the histogram");

__device__ __forceinline__ int fpw_bin(unsigned long long k, int kind) {
    int e, m;
    if (kind == 1) {
        e = (int)((k >> 52) & 0x7ff) - (1023 - 26);
        m = (int)((k >> (52 - kFpwSub)) & ((1 << kFpwSub) - 1));
    } else {
        e = (int)((k >> 55) & 0xff) - (127 - 26);
        m = (int)((k >> (55 - kFpwSub)) & ((1 << kFpwSub) - 1));
    }
    if (e < 0) return 0;
    if (e >= kFpwOct) return kFpwBins - 1;
    return 1 + (e << kFpwSub) + m;
}

// prefix and its length for a regular bin
__device__ __forceinline__ unsigned long long fpw_prefix(int bin, int kind, int& bits) {
    const unsigned long long e = (unsigned long long)((bin - 1) >> kFpwSub);
    const unsigned long long m = (unsigned long long)((bin - 1) & ((1 << kFpwSub) - 1));
    if (kind == 1) {
        bits = 12 + kFpwSub;
        return ((e + 1023 - 26) << 52) | (m << (52 - kFpwSub));
    }
    bits = 9 + kFpwSub;
    return ((e + 127 - 26) << 55) | (m << (55 - kFpwSub));
}

// Key sources.  Phase A: |flow| for queries 0,1 and |grad I| for 2,3 (materialised buffers).
// Phase B: saliency for query 0, computed from the buffers, or read from a given map (tap).
// keys4 reads elements i..i+3 (i % 4 == 0, plane size % 4 == 0) with vector loads.
struct SrcBufA {
    const float* fm;
    const double* gr;
    static constexpr int NQ = 4;
    __device__ __forceinline__ void keys(long long i, unsigned long long* k) const {
        k[0] = k[1] = fkey(fm[i]);
        k[2] = k[3] = dkey(gr[i]);
    }
    // raw loads of four pixels, issued one step ahead of their use (sel_pass_body)
    struct Raw {
        float4 f;
        double2 g0, g1;
    };
    __device__ __forceinline__ Raw load4(long long i) const {
        return Raw{__ldg((const float4*)(fm + i)), __ldg((const double2*)(gr + i)), __ldg((const double2*)(gr + i + 2))};
    }
    __device__ __forceinline__ void keys4(long long i, unsigned long long (*k)[4]) const { keys_of(load4(i), k); }
    __device__ __forceinline__ void keys_of(const Raw& r, unsigned long long (*k)[4]) const {
        const float4 f = r.f;
        const double2 g0 = r.g0, g1 = r.g1;
        k[0][0] = k[1][0] = fkey(f.x);
        k[0][1] = k[1][1] = fkey(f.y);
        k[0][2] = k[1][2] = fkey(f.z);
        k[0][3] = k[1][3] = fkey(f.w);
        k[2][0] = k[3][0] = dkey(g0.x);
        k[2][1] = k[3][1] = dkey(g0.y);
        k[2][2] = k[3][2] = dkey(g1.x);
        k[2][3] = k[3][3] = dkey(g1.y);
    }
};

__device__ __forceinline__ double sal_from(const PairInfo& I, double w, double w1, float f, double gg) {
    const double nf = normalize((double)f, I.fmag_lo, I.fmag_inv, I.fmag_zero);
    const double ng = normalize(gg, I.grad_lo, I.grad_inv, I.grad_zero);
    return dadd(dmul(w, nf), dmul(w1, ng));
}

struct SrcSal {
    const float* fm;
    const double* gr;
    PairInfo I;
    double w, w1;
    static constexpr int NQ = 1;
    __device__ __forceinline__ double value(long long i) const { return sal_from(I, w, w1, fm[i], gr[i]); }
    __device__ __forceinline__ void keys(long long i, unsigned long long* k) const { k[0] = dkey(value(i)); }
    struct Raw {
        float4 f;
        double2 g0, g1;
    };
    __device__ __forceinline__ Raw load4(long long i) const {
        return Raw{__ldg((const float4*)(fm + i)), __ldg((const double2*)(gr + i)), __ldg((const double2*)(gr + i + 2))};
    }
    __device__ __forceinline__ void keys4(long long i, unsigned long long (*k)[4]) const { keys_of(load4(i), k); }
    __device__ __forceinline__ void keys_of(const Raw& r, unsigned long long (*k)[4]) const {
        const float4 f = r.f;
        const double2 g0 = r.g0, g1 = r.g1;
        k[0][0] = dkey(sal_from(I, w, w1, f.x, g0.x));
        k[0][1] = dkey(sal_from(I, w, w1, f.y, g0.y));
        k[0][2] = dkey(sal_from(I, w, w1, f.z, g1.x));
        k[0][3] = dkey(sal_from(I, w, w1, f.w, g1.y));
    }
};

struct SrcMap {
    const double* map;
    static constexpr int NQ = 1;
    __device__ __forceinline__ double value(long long i) const { return map[i]; }
    __device__ __forceinline__ void keys(long long i, unsigned long long* k) const { k[0] = dkey(map[i]); }
    struct Raw {
        double2 g0, g1;
    };
    __device__ __forceinline__ Raw load4(long long i) const {
        return Raw{__ldg((const double2*)(map + i)), __ldg((const double2*)(map + i + 2))};
    }
    __device__ __forceinline__ void keys4(long long i, unsigned long long (*k)[4]) const { keys_of(load4(i), k); }
    __device__ __forceinline__ void keys_of(const Raw& r, unsigned long long (*k)[4]) const {
        const double2 g0 = r.g0, g1 = r.g1;
        k[0][0] = dkey(g0.x);
        k[0][1] = dkey(g0.y);
        k[0][2] = dkey(g1.x);
        k[0][3] = dkey(g1.y);
    }
};

// warp-aggregated shared histogram increment (one atomic when the warp's keys share a bin);
// every lane of the warp must call it
__device__ __forceinline__ void hist_add(unsigned int* h, bool m, unsigned int bin, int lane) {
    const unsigned int bal = __ballot_sync(0xffffffffu, m);
    if (!bal) return;
    const int leader = __ffs(bal) - 1;
    const unsigned int b0 = __shfl_sync(0xffffffffu, bin, leader);
    if (__all_sync(0xffffffffu, !m || bin == b0)) {
        if (lane == leader) atomicAdd(&h[b0], (unsigned int)__popc(bal));
    } else if (m) {
        atomicAdd(&h[bin], 1u);
    }
}

// One pass of every active query of one pair over a contiguous range of the pair's pixels, four
// consecutive pixels per thread: histogram of the next digit (exponent window first for
// single-query sources) for queries in HIST mode, warp-aggregated candidate append for queries in
// COLLECT mode.  All threads of the CTA run the same number of iterations (warp votes inside).
// write_bits (single-query sources, W % 32 == 0): a COLLECT pass also writes the threshold words
// of every pixel outside the boundary bin (above -> 1, below -> 0; the bin's candidates are 0
// until k_thr_fixup) and records each candidate's pixel index.
template <class Src>
__device__ void sel_pass_body(const Geom& g, const MaskBuffers& b, int p, const Src& src,
                              bool write_bits = false, int bi = -1, int nb = 0) {
    // this CTA's share of the pair's pixels: block bi of nb (default: blockIdx.x of gridDim.x)
    if (bi < 0) {
        bi = blockIdx.x;
        nb = gridDim.x;
    }
    constexpr int NQ = Src::NQ;
    constexpr int NB = NQ == 1 ? kHistBins : kSelBins;
    constexpr int CB = NQ == 1 ? 2048 : 1024;
    // dynamic shared memory (pass_smem): COLLECT staging [NQ][CB] keys, then HIST [NQ][NB] bins
    extern __shared__ __align__(16) unsigned char dsm[];
    unsigned long long (*cbuf)[CB] = reinterpret_cast<unsigned long long (*)[CB]>(dsm);
    unsigned int (*hist)[NB] = reinterpret_cast<unsigned int (*)[NB]>(dsm + sizeof(unsigned long long) * NQ * CB);
    unsigned int* cidx = reinterpret_cast<unsigned int*>(dsm + (sizeof(unsigned long long) * CB + sizeof(unsigned int) * NB) * NQ);
    __shared__ SelState st[NQ];
    __shared__ unsigned long long smn[NQ], smx[NQ];
    // COLLECT: candidates staged per block in shared memory (one global reservation per query)
    __shared__ unsigned int ccnt[NQ], cbase[NQ];
    __syncthreads();  // a previous pass / scan of this CTA (k_sel_rest_*) is done with shared memory
    if (threadIdx.x < NQ) {
        st[threadIdx.x] = b.sel[p * kMaxQueries + threadIdx.x];
        smn[threadIdx.x] = ~0ull;
        smx[threadIdx.x] = 0ull;
        ccnt[threadIdx.x] = 0u;
    }
    __syncthreads();
    bool anyh = false, anyc = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        anyh |= st[q].mode == SEL_HIST;
        anyc |= st[q].mode == SEL_COLLECT;
    }
    if (!anyh && !anyc) return;
    if (anyh) {
        for (int i = threadIdx.x; i < NQ * NB; i += blockDim.x) (&hist[0][0])[i] = 0;
        __syncthreads();
    }
    unsigned hqm = 0u, cqm = 0u;  // queries in HIST / COLLECT mode (bit q)
    int sh[NQ], wd[NQ], fp[NQ], ms[NQ];
    unsigned long long mp[NQ], lmn[NQ], lmx[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        hqm |= (st[q].mode == SEL_HIST ? 1u : 0u) << q;
        cqm |= (st[q].mode == SEL_COLLECT ? 1u : 0u) << q;
        sel_digit(st[q].bits_done, sh[q], wd[q]);
        fp[q] = (NQ == 1 && st[q].bits_done == 0) ? st[q].fpw : 0;
        ms[q] = 64 - st[q].bits_done;  // keys match when key >> ms == prefix >> ms (ms < 64)
        mp[q] = ms[q] < 64 ? st[q].prefix >> ms[q] : 0ull;
        lmn[q] = ~0ull;
        lmx[q] = 0ull;
    }
    // high-word prefix test (HI passes): (hi >> s32) & m32 == p32, with m32 = 0 matching every key
    // while no digit is fixed yet
    unsigned s32[NQ], m32[NQ], p32[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const bool all = ms[q] >= 64;
        s32[q] = all ? 0u : (unsigned)max(0, ms[q] - 32);
        m32[q] = all ? 0u : ~0u;
        p32[q] = all ? 0u : (unsigned)mp[q];
    }
    const long long n = (long long)g.W * g.H;
    const bool vec = (n & 3) == 0;
    const bool bits = NQ == 1 && write_bits && (cqm & 1u);
    // word-aligned block ranges when writing bits (every warp step covers 4 whole words)
    const long long gran = bits ? 4ll * blockDim.x : 4ll;
    const long long per = cdiv<long long>(cdiv<long long>(n, nb), gran) * gran;
    const long long i0 = bi * per, i1 = min(n, i0 + per);
    const int lane = threadIdx.x & 31;
    // HI: every active query's prefix lies in the keys' high 32 bits (ms >= 32, e.g. right after
    // the exponent-window digit): prefix tests on the high word alone
    bool hi = true;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
        if ((((hqm >> q) & 1u) || ((cqm >> q) & 1u)) && ms[q] < 32) hi = false;
    auto main_loop = [&](auto hi_tag) {
    constexpr bool HI = decltype(hi_tag)::value;
    // the next step's raw loads are issued before this step's keys are processed (two steps of
    // loads in flight per thread)
    typename Src::Raw nxt{};
    if (vec && i0 + 4ll * threadIdx.x + 3 < i1) nxt = src.load4(i0 + 4ll * threadIdx.x);
    for (long long base0 = i0; base0 < i1; base0 += 4ll * blockDim.x) {
        const long long base = base0 + 4ll * threadIdx.x;
        unsigned long long k[NQ][4];
        bool v[4];
        const typename Src::Raw cur = nxt;
        const long long nb = base + 4ll * blockDim.x;
        if (vec && nb + 3 < i1) nxt = src.load4(nb);
        if (vec && base + 3 < i1) {
            src.keys_of(cur, k);
            v[0] = v[1] = v[2] = v[3] = true;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[e] = base + e < i1;
                unsigned long long t[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) t[q] = 0;
                if (v[e]) src.keys(base + e, t);
#pragma unroll
                for (int q = 0; q < NQ; ++q) k[q][e] = t[q];
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (((hqm >> q) & 1u)) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool m = v[e] && (HI ? (((unsigned)(k[q][e] >> 32) >> s32[q]) & m32[q]) == p32[q]
                                               : (ms[q] >= 64 || (k[q][e] >> ms[q]) == mp[q]));
                    const unsigned int bin = fp[q] ? (unsigned int)fpw_bin(k[q][e], fp[q])
                                                   : (unsigned int)((k[q][e] >> sh[q]) & ((1u << wd[q]) - 1u));
                    if (fp[q]) {  // exponent-window bins are spread out: plain shared atomics
                        if (m) atomicAdd(&hist[q][bin], 1u);
                    } else {
                        hist_add(hist[q], m, bin, lane);
                    }
                    if (m) {
                        lmn[q] = min(lmn[q], k[q][e]);
                        lmx[q] = max(lmx[q], k[q][e]);
                    }
                }
            } else if (((cqm >> q) & 1u)) {
                bool m[4], any = false;
                unsigned int nib = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const unsigned long long kp = HI ? (unsigned long long)(((unsigned)(k[q][e] >> 32) >> s32[q]) & m32[q])
                                                     : (ms[q] < 64 ? k[q][e] >> ms[q] : 0ull);
                    m[e] = v[e] && (HI ? (unsigned)kp == p32[q] : (ms[q] >= 64 || kp == mp[q]));
                    any |= m[e];
                    if (v[e] && ms[q] < 64 && (HI ? (unsigned)kp > p32[q] : kp > mp[q])) nib |= 1u << e;
                }
                if (bits) {
                    // lane l holds bits 4(l%8)..+3 of word (base0 + 128 w_l)/32 + l/8
                    unsigned int word = nib << (4 * (lane & 7));
                    word |= __shfl_xor_sync(0xffffffffu, word, 1);
                    word |= __shfl_xor_sync(0xffffffffu, word, 2);
                    word |= __shfl_xor_sync(0xffffffffu, word, 4);
                    if ((lane & 7) == 0 && base < i1)
                        b.bits_thr[(size_t)p * g.H * g.WW + (size_t)(base >> 5)] = word;
                }
                if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const unsigned int bal = __ballot_sync(0xffffffffu, m[e]);
                        if (!bal) continue;
                        unsigned int basei = 0;
                        const int leader = __ffs(bal) - 1;
                        if (lane == leader) basei = atomicAdd(&ccnt[q], __popc(bal));
                        basei = __shfl_sync(0xffffffffu, basei, leader);
                        if (m[e]) {
                            const unsigned int idx = basei + __popc(bal & ((1u << lane) - 1u));
                            if (idx < (unsigned)CB) {
                                cbuf[q][idx] = k[q][e];
                                if (bits) cidx[idx] = (unsigned int)(base + e);
                            } else {  // staging full: straight to the global list
                                const unsigned int gi = atomicAdd(b.cand_count + p * kMaxQueries + q, 1u);
                                if (gi < (unsigned)kSelCap) {
                                    b.cand[((size_t)p * kMaxQueries + q) * kSelCap + gi] = k[q][e];
                                    if (bits) b.cand_idx[(size_t)p * kSelCap + gi] = (unsigned int)(base + e);
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    };
    if (hi) main_loop(std::true_type{});
    else main_loop(std::false_type{});
    if (anyc) {
        __syncthreads();
        if (threadIdx.x < NQ && ((cqm >> threadIdx.x) & 1u)) {
            const unsigned int c = min(ccnt[threadIdx.x], (unsigned int)CB);
            cbase[threadIdx.x] = c ? atomicAdd(b.cand_count + p * kMaxQueries + threadIdx.x, c) : 0u;
        }
        __syncthreads();
        for (int q = 0; q < NQ; ++q) {
            if (!((cqm >> q) & 1u)) continue;
            const unsigned int c = min(ccnt[q], (unsigned int)CB);
            unsigned long long* dst = b.cand + ((size_t)p * kMaxQueries + q) * kSelCap;
            for (unsigned int i = threadIdx.x; i < c; i += blockDim.x)
                if (cbase[q] + i < (unsigned)kSelCap) {
                    dst[cbase[q] + i] = cbuf[q][i];
                    if (bits) b.cand_idx[(size_t)p * kSelCap + cbase[q] + i] = cidx[i];
                }
        }
    }
    if (!anyh) return;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        if (!((hqm >> q) & 1u)) continue;
        unsigned long long a = lmn[q], c = lmx[q];
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
        }
        if (lane == 0) {
            atomicMin(&smn[q], a);
            atomicMax(&smx[q], c);
        }
    }
    __syncthreads();
    for (int q = 0; q < NQ; ++q) {
        if (!((hqm >> q) & 1u)) continue;
        unsigned int* gh = b.hist + ((size_t)p * kMaxQueries + q) * kHistBins;
        for (int i = threadIdx.x; i < NB; i += blockDim.x)
            if (hist[q][i]) atomicAdd(gh + i, hist[q][i]);
        if (threadIdx.x == 0) {
            atomicMin(&b.sel[p * kMaxQueries + q].mn, smn[q]);
            atomicMax(&b.sel[p * kMaxQueries + q].mx, smx[q]);
        }
    }
}

// Phase-A producer: |flow| (glibc hypotf) and |grad I| materialised + the first pass.
constexpr int PNT_MG = 256;

// Row-blocked: each CTA owns whole rows of one pair (32-bit indexing).  Queries 0/1 (|flow|
// percentiles) and 2/3 (|grad I|) share their first-pass histograms, so two are built (the
// exponent-window digit) and added to both queries of each pair.
#ifndef FROI_MG_FAST
#define FROI_MG_FAST 0
#endif
#ifndef FROI_MG_NPX
#define FROI_MG_NPX 4
#endif
#ifndef FROI_MG_MINB
#define FROI_MG_MINB 4
#endif
// TAB: 8-bit frames with the context's |grad I| table (DevParams::grad_tab)
template <typename T, bool TAB>
__global__ void __launch_bounds__(PNT_MG, FROI_MG_MINB) k_mag_grad(Geom g, DevParams P, MaskBuffers b) {
    __shared__ double lut[256];
    __shared__ unsigned int hist[2][kFpwBins];
    __shared__ unsigned long long smn[2], smx[2];
    const int p = blockIdx.y;
    const PairInfo I = b.info[p];
    PairPix<T> px = make_pix<T>(g, P, b, I, p);
    if (sizeof(T) == 1) {
        for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = dmul((double)v, px.inv_maxval);
        px.lut = lut;
    }
    for (int i = threadIdx.x; i < 2 * kFpwBins; i += blockDim.x) (&hist[0][0])[i] = 0u;
    if (threadIdx.x < 2) {
        smn[threadIdx.x] = ~0ull;
        smx[threadIdx.x] = 0ull;
    }
    __syncthreads();
    const int W = g.W, H = g.H;
    float* fm = opaque(b.fm + (size_t)p * W * H);
    double* gr = opaque(b.gr + (size_t)p * W * H);
    const int rows = (H + gridDim.x - 1) / gridDim.x;
    const int y0 = blockIdx.x * rows, y1 = min(H, y0 + rows);
    const int lane = threadIdx.x & 31;
    // extremes tracked on the values (the keys are monotone in them), keyed after the loop
    float mnf = __int_as_float(0x7f800000), mxf = 0.f;
    double mng = __longlong_as_double(0x7ff0000000000000ll), mxg = 0.0;
    // NPX pixels per thread per step: all their loads (flow, the four gradient neighbours) are
    // issued before any of their arithmetic, so each thread keeps ~NPX*5 loads in flight
    constexpr int NPX = FROI_MG_NPX;
    const float2* __restrict__ flw = px.flow;
    const T* __restrict__ raw = px.raw;
    for (int y = y0; y < y1; ++y) {
        const int row = y * W;
        const int sy = clampi(y + px.dy, 0, H - 1);
        const int sym = clampi(clampi(y - 1, 0, H - 1) + px.dy, 0, H - 1);
        const int syp = clampi(clampi(y + 1, 0, H - 1) + px.dy, 0, H - 1);
        // row bases once per row (opaque: each gather is then one 32-bit-offset add)
        const float2* flr = opaque(flw + (unsigned)row);
        const T* rs = opaque(raw + (unsigned)(sy * W));
        const T* rm = opaque(raw + (unsigned)(sym * W));
        const T* rp = opaque(raw + (unsigned)(syp * W));
        for (int xb = 0; xb < W; xb += NPX * PNT_MG) {
            float2 fl[NPX];
            int vl[NPX], vr[NPX], vu[NPX], vd[NPX];
            constexpr bool tab = TAB && sizeof(T) == 1;  // launched only with gradient_source 0
#pragma unroll
            for (int k = 0; k < NPX; ++k) {
                const int x = min(xb + (int)threadIdx.x + k * PNT_MG, W - 1);
                fl[k] = __ldg(flr + (unsigned)x);
                if (sizeof(T) == 1 && P.gradient_source == 0) {
                    const unsigned sx = clampi(x + px.dx, 0, W - 1);
                    const unsigned sxm = clampi(clampi(x - 1, 0, W - 1) + px.dx, 0, W - 1);
                    const unsigned sxp = clampi(clampi(x + 1, 0, W - 1) + px.dx, 0, W - 1);
                    vl[k] = __ldg(rs + sxm);
                    vr[k] = __ldg(rs + sxp);
                    vu[k] = __ldg(rm + sx);
                    vd[k] = __ldg(rp + sx);
                }
            }
            // 8-bit frames: |grad I| = grad_tab[index(|gx|)][index(|gy|)], the exact value
            // hypot_glibc(gx, gy) gives (hypot only sees |gx|, |gy|); all table reads in flight
            double gt[NPX];
            if constexpr (tab) {
                unsigned ix[NPX], iy[NPX];
#pragma unroll
                for (int k = 0; k < NPX; ++k) {
                    ix[k] = __ldg(P.grad_map + ((unsigned)vr[k] << 8) + (unsigned)vl[k]);
                    iy[k] = __ldg(P.grad_map + ((unsigned)vd[k] << 8) + (unsigned)vu[k]);
                }
#pragma unroll
                for (int k = 0; k < NPX; ++k) gt[k] = __ldg(P.grad_tab + ix[k] * (unsigned)P.grad_nv + iy[k]);
            }
            // a whole chunk inside the row (every chunk when W is a multiple of NPX*PNT_MG) runs
            // without per-pixel validity branches
            auto consume = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int k = 0; k < NPX; ++k) {
                const int x = xb + threadIdx.x + k * PNT_MG;
                const bool v = FULL || x < W;
                unsigned long long kf = 0, kg = 0;
                if (v) {
#if FROI_MG_FAST
                    // branch-free fast paths of the sqrt / division sequences (common.cuh): the
                    // same bits whenever their range test passes, the rare rest redone exactly
                    const double fx = fl[k].x, fy = fl[k].y;
                    const double f2 = dadd(dmul(fx, fx), dmul(fy, fy));
                    bool okf;
                    const double fs = dsqrt_fast(f2, okf);
                    const float f = (float)(okf ? fs : dsqrt(f2));
#else
                    const float f = hypotf_glibc(fl[k].x, fl[k].y);
#endif
                    double gg;
                    if constexpr (tab) {
                        gg = gt[k];
                    } else if (sizeof(T) == 1 && P.gradient_source == 0) {
                        const double gx = dmul(0.5, dsub(lut[vr[k]], lut[vl[k]]));
                        const double gy = dmul(0.5, dsub(lut[vd[k]], lut[vu[k]]));
#if FROI_MG_FAST
                        bool okg;
                        gg = hypot_glibc_fast(gx, gy, okg);
                        if (!okg) gg = hypot_glibc(gx, gy);
#elif defined(FROI_DIAG_MG_NOHYPOT)
                        gg = dadd(fabs(gx), fabs(gy));
#else
                        gg = hypot_glibc(gx, gy);
#endif
                    } else {
                        gg = px.grad(x, y);
                    }
                    fm[(unsigned)(row + x)] = f;
                    gr[(unsigned)(row + x)] = gg;
                    kf = fkey(f);
                    kg = dkey(gg);
                    mnf = fminf(mnf, f);
                    mxf = fmaxf(mxf, f);
                    mng = gg < mng ? gg : mng;
                    mxg = gg > mxg ? gg : mxg;
                }
#ifndef FROI_DIAG_MG_NOHIST
                if (v) {  // exponent-window bins are spread out: plain shared atomics
                    atomicAdd(&hist[0][fpw_bin(kf, 2)], 1u);
                    atomicAdd(&hist[1][fpw_bin(kg, 1)], 1u);
                }
#endif
            }
            };
            if (xb + NPX * PNT_MG <= W) consume(std::true_type{});
            else consume(std::false_type{});
        }
    }
    unsigned long long kmnf = mnf == __int_as_float(0x7f800000) ? ~0ull : fkey(mnf), kmxf = fkey(mxf);
    unsigned long long kmng = mng == __longlong_as_double(0x7ff0000000000000ll) ? ~0ull : dkey(mng);
    unsigned long long kmxg = dkey(mxg);
    for (int o = 16; o > 0; o >>= 1) {
        kmnf = min(kmnf, __shfl_xor_sync(0xffffffffu, kmnf, o));
        kmxf = max(kmxf, __shfl_xor_sync(0xffffffffu, kmxf, o));
        kmng = min(kmng, __shfl_xor_sync(0xffffffffu, kmng, o));
        kmxg = max(kmxg, __shfl_xor_sync(0xffffffffu, kmxg, o));
    }
    if (lane == 0) {
        atomicMin(&smn[0], kmnf);
        atomicMax(&smx[0], kmxf);
        atomicMin(&smn[1], kmng);
        atomicMax(&smx[1], kmxg);
    }
    __syncthreads();
    unsigned int* gh = b.hist + (size_t)p * kMaxQueries * kHistBins;
    for (int i = threadIdx.x; i < kFpwBins; i += blockDim.x) {
        const unsigned int hf = hist[0][i], hg = hist[1][i];
        if (hf) {
            atomicAdd(gh + i, hf);
            atomicAdd(gh + kHistBins + i, hf);
        }
        if (hg) {
            atomicAdd(gh + 2 * kHistBins + i, hg);
            atomicAdd(gh + 3 * kHistBins + i, hg);
        }
    }
    if (threadIdx.x < 4) {
        const int k = threadIdx.x >> 1;
        atomicMin(&b.sel[p * kMaxQueries + threadIdx.x].mn, smn[k]);
        atomicMax(&b.sel[p * kMaxQueries + threadIdx.x].mx, smx[k]);
    }
}

__global__ void __launch_bounds__(SNT, 2) k_sel_pass_a(Geom g, MaskBuffers b) {
    const int p = blockIdx.y;
    SrcBufA src{opaque(b.fm + (size_t)p * g.W * g.H), opaque(b.gr + (size_t)p * g.W * g.H)};
    sel_pass_body(g, b, p, src);
}

__global__ void __launch_bounds__(SNT, 2) k_sel_pass_b(Geom g, DevParams P, MaskBuffers b, const double* map,
                                                   int write_bits) {
    const int p = blockIdx.y;
    if (map) {
        SrcMap src{map};
        sel_pass_body(g, b, p, src, write_bits != 0);
    } else {
        SrcSal src{opaque(b.fm + (size_t)p * g.W * g.H), opaque(b.gr + (size_t)p * g.W * g.H), b.info[p],
                   P.flow_weight, 1.0 - P.flow_weight};
        sel_pass_body(g, b, p, src, write_bits != 0);
    }
}

constexpr size_t pass_smem(int nq) {
    return (sizeof(unsigned long long) * (nq == 1 ? 2048 : 1024) + sizeof(unsigned int) * (nq == 1 ? kHistBins : kSelBins)) * nq +
           (nq == 1 ? sizeof(unsigned int) * 2048 : 0);
}

// One CTA per (pair, query): narrow the prefix after a histogram pass, or finish a collected
// group (<= kSelCap keys, all sharing the prefix) by an 8-bit-digit radix select in shared memory.
constexpr int SCT = 1024;

// One (pair, query) step of the selection by a CTA of SCT threads; cs: kSelCap keys of shared
// memory.  Shared by k_sel_scan (one CTA per query) and k_sel_rest_* (one CTA per pair).
__device__ void sel_scan_body(const MaskBuffers& b, int p, int q, int bits, unsigned long long* cs) {
    SelState* sp = b.sel + p * kMaxQueries + q;
    __shared__ SelState s;
    __shared__ unsigned int part[SCT];
    __syncthreads();  // a previous step of this CTA is done with shared memory
    if (threadIdx.x == 0) s = *sp;
    __syncthreads();
    if (s.mode == SEL_DONE) return;
    if (s.mode == SEL_COLLECT) {
        __shared__ unsigned int h8[256];
        __shared__ unsigned long long s_pfx, s_r;
        __shared__ unsigned int s_cnt;
        unsigned int* cc = b.cand_count + p * kMaxQueries + q;
        const int n = (int)min((unsigned int)kSelCap, *cc);
        const unsigned long long* src = b.cand + ((size_t)p * kMaxQueries + q) * kSelCap;
        for (int i = threadIdx.x; i < n; i += SCT) cs[i] = src[i];
        if (threadIdx.x == 0) {
            s_pfx = s.prefix;
            s_r = s.rank;
            s_cnt = (unsigned int)n;
        }
        __syncthreads();
        for (int bd = s.bits_done; bd < 64;) {
            const int w = min(8, 64 - bd), sh = 64 - bd - w;
            if (threadIdx.x < 256) h8[threadIdx.x] = 0u;
            __syncthreads();
            const unsigned long long pf = s_pfx;
            for (int i = threadIdx.x; i < n; i += SCT) {
                const unsigned long long k = cs[i];
                if (bd == 0 || (k >> (64 - bd)) == (pf >> (64 - bd)))
                    atomicAdd(&h8[(unsigned int)(k >> sh) & ((1u << w) - 1u)], 1u);
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                unsigned int c8[8], sum = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    c8[j] = h8[lane * 8 + j];
                    sum += c8[j];
                }
                unsigned int incl = sum;
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const unsigned long long r = s_r;
                unsigned long long c = incl - sum;
                if (r >= c && r < (unsigned long long)incl) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (r >= c && r < c + c8[j]) {
                            s_pfx = pf | ((unsigned long long)(lane * 8 + j) << sh);
                            s_r = r - c;
                            s_cnt = c8[j];
                        }
                        c += c8[j];
                    }
                }
            }
            __syncthreads();
            bd += w;
        }
        if (threadIdx.x == 0) {
            SelState ns = s;
            ns.result = s_pfx;
            ns.count_lt = s.k0 - s_r;
            ns.count_eq = s_cnt;
            ns.mode = SEL_DONE;
            *sp = ns;
            *cc = 0;
            if (bits) {  // the collect pass that fed this select wrote the threshold words
                b.info[p].bits_ready = 1;
                b.info[p].n_cand = (unsigned int)n;
            }
        }
        return;
    }
    unsigned int* gh = b.hist + ((size_t)p * kMaxQueries + q) * kHistBins;
    constexpr int PER = kHistBins / SCT;
    unsigned int loc[PER];
    unsigned int tot = 0;
    for (int j = 0; j < PER; ++j) {
        loc[j] = gh[threadIdx.x * PER + j];
        tot += loc[j];
    }
    part[threadIdx.x] = tot;
    __syncthreads();
    for (int o = 1; o < SCT; o <<= 1) {
        const unsigned int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    const unsigned long long before = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
    const unsigned long long r = s.rank;
    if (r >= before && r < (unsigned long long)part[threadIdx.x]) {
        unsigned long long c = before;
        for (int j = 0; j < PER; ++j) {
            if (r < c + loc[j]) {
                const int bin = threadIdx.x * PER + j;
                int shift, width;
                sel_digit(s.bits_done, shift, width);
                SelState n = s;
                const bool fp = s.bits_done == 0 && s.fpw;
                n.fpw = 0;
                if (s.mn == s.mx) {  // every key of the prefix group equals the answer
                    n.mode = SEL_DONE;
                    n.result = s.mn;
                    n.count_lt = s.k0 - s.rank;
                    n.count_eq = s.count;
                } else if (fp && (bin == 0 || bin == kFpwBins - 1)) {
                    // outside the exponent window: radix digits from the top
                } else if (fp) {
                    int bits;
                    n.prefix = fpw_prefix(bin, s.fpw, bits);
                    n.rank = r - c;
                    n.count = loc[j];
                    n.bits_done = bits;
                    if (n.count <= (unsigned long long)kSelCap) n.mode = SEL_COLLECT;
                } else {
                    n.prefix = s.prefix | ((unsigned long long)bin << shift);
                    n.rank = r - c;
                    n.count = loc[j];
                    n.bits_done = s.bits_done + width;
                    if (n.bits_done >= 64) {
                        n.mode = SEL_DONE;
                        n.result = n.prefix;
                        n.count_lt = s.k0 - n.rank;
                        n.count_eq = n.count;
                    } else if (n.count <= (unsigned long long)kSelCap) {
                        n.mode = SEL_COLLECT;
                    }
                }
                n.mn = ~0ull;
                n.mx = 0ull;
                *sp = n;
                break;
            }
            c += loc[j];
        }
    }
    for (int j = 0; j < PER; ++j) gh[threadIdx.x * PER + j] = 0u;
}

__global__ void __launch_bounds__(SCT) k_sel_scan(MaskBuffers b, int nq, int bits = 0) {
    extern __shared__ unsigned long long cs[];  // kSelCap candidates
    sel_scan_body(b, blockIdx.x / nq, blockIdx.x % nq, bits, cs);
}

// The selection's remaining steps, one CTA per pair, looping pass + scans in the CTA until every
// query is done.  Launched once after the passes that normally finish the selection, so the
// worst case (long runs of equal keys) needs no extra launches and the common case costs one
// launch that exits at once.
template <class Src, int NQ>
__device__ void sel_rest(const Geom& g, const MaskBuffers& b, int p, const Src& src, bool write_bits) {
    extern __shared__ unsigned long long cs[];
    __shared__ int open;
    for (int it = 0; it < 64; ++it) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int o = 0;
            for (int q = 0; q < NQ; ++q) o |= b.sel[p * kMaxQueries + q].mode != SEL_DONE;
            open = o;
        }
        __syncthreads();
        if (!open) return;
        sel_pass_body(g, b, p, src, write_bits, 0, 1);
        __syncthreads();
        for (int q = 0; q < NQ; ++q) sel_scan_body(b, p, q, write_bits ? 1 : 0, cs);
    }
}

__global__ void __launch_bounds__(SCT) k_sel_rest_a(Geom g, MaskBuffers b) {
    const int p = blockIdx.x;
    SrcBufA src{opaque(b.fm + (size_t)p * g.W * g.H), opaque(b.gr + (size_t)p * g.W * g.H)};
    sel_rest<SrcBufA, 4>(g, b, p, src, false);
}

__global__ void __launch_bounds__(SCT) k_sel_rest_b(Geom g, DevParams P, MaskBuffers b, const double* map,
                                                    int write_bits) {
    const int p = blockIdx.x;
    if (map) {
        SrcMap src{map};
        sel_rest<SrcMap, 1>(g, b, p, src, write_bits != 0);
    } else {
        SrcSal src{opaque(b.fm + (size_t)p * g.W * g.H), opaque(b.gr + (size_t)p * g.W * g.H), b.info[p],
                   P.flow_weight, 1.0 - P.flow_weight};
        sel_rest<SrcSal, 1>(g, b, p, src, write_bits != 0);
    }
}

__device__ __forceinline__ SelState sel_init(unsigned long long k0, unsigned long long n, bool done,
                                             int fpw) {
    SelState s;
    s.prefix = 0;
    s.rank = k0;
    s.k0 = k0;
    s.result = 0;
    s.mn = ~0ull;
    s.mx = 0;
    s.count = n;
    s.count_lt = 0;
    s.count_eq = 0;
    s.bits_done = 0;
    s.mode = done ? SEL_DONE : SEL_HIST;
    s.fpw = fpw;
    return s;
}

__global__ void k_sel_init_a(MaskBuffers b, unsigned long long n, unsigned long long ilo,
                             unsigned long long ihi) {
    const int p = blockIdx.x;
    if (threadIdx.x < kMaxQueries)
        b.sel[p * kMaxQueries + threadIdx.x] = sel_init((threadIdx.x & 1) ? ihi : ilo, n, false,
                                                        threadIdx.x < 2 ? 2 : 1);
}

// robust_normalize parameters (roi.hpp:47-63), then the threshold query (roi.hpp:114-120).
__global__ void k_sel_init_b(MaskBuffers b, unsigned long long n, unsigned long long target,
                             int from_stats) {
    const int p = blockIdx.x;
    if (threadIdx.x != 0) return;
    PairInfo& I = b.info[p];
    if (from_stats) {
        const SelState* s = b.sel + p * kMaxQueries;
        I.fmag_lo = ffromkey(s[0].result);
        I.fmag_hi = ffromkey(s[1].result);
        I.grad_lo = dfromkey(s[2].result);
        I.grad_hi = dfromkey(s[3].result);
        const double df = dsub(I.fmag_hi, I.fmag_lo), dg = dsub(I.grad_hi, I.grad_lo);
        I.fmag_zero = !(df > 1e-12);
        I.grad_zero = !(dg > 1e-12);
        I.fmag_inv = I.fmag_zero ? 0.0 : ddiv(1.0, df);
        I.grad_inv = I.grad_zero ? 0.0 : ddiv(1.0, dg);
    }
    I.target = target;
    I.bits_ready = 0;
    I.n_cand = 0;
    // (target-1)-th largest == (n-target)-th smallest
    b.sel[p * kMaxQueries] = sel_init(target ? n - target : 0, n, target == 0, from_stats ? 1 : 0);
    for (int q = 1; q < kMaxQueries; ++q) b.sel[p * kMaxQueries + q].mode = SEL_DONE;
}

// ------------------------------------------------------------------ threshold
constexpr int TNT = 256;
constexpr int TROWS = 4;  // rows per tie chunk

// threshold_mask decision (roi.hpp:114-137) from the exact counts of the selection.
__global__ void k_sel_finish_b(MaskBuffers b, unsigned long long n) {
    const int p = blockIdx.x;
    if (threadIdx.x != 0) return;
    PairInfo& I = b.info[p];
    const SelState s = b.sel[p * kMaxQueries];
    if (I.target == 0) {
        I.thr_mode = 1;
        I.boundary = 0.0;
        return;
    }
    I.boundary = dfromkey(s.result);
    if (!(I.boundary > 0.0)) {
        I.thr_mode = 2;
        return;
    }
    I.count_eq = s.count_eq;
    I.count_gt = n - s.count_lt - s.count_eq;
    I.need = I.target - I.count_gt;
    I.thr_mode = I.need >= I.count_eq ? 0 : 3;
}

template <class Src>
__device__ __forceinline__ Src make_thr_src(const Geom& g, const DevParams& P, const MaskBuffers& b,
                                            int p, const double* map);
template <>
__device__ __forceinline__ SrcSal make_thr_src<SrcSal>(const Geom& g, const DevParams& P,
                                                       const MaskBuffers& b, int p, const double*) {
    return SrcSal{opaque(b.fm + (size_t)p * g.W * g.H), opaque(b.gr + (size_t)p * g.W * g.H), b.info[p],
                  P.flow_weight, 1.0 - P.flow_weight};
}
template <>
__device__ __forceinline__ SrcMap make_thr_src<SrcMap>(const Geom&, const DevParams&,
                                                       const MaskBuffers&, int, const double* map) {
    return SrcMap{map};
}

// Per-chunk tie counts, only for pairs that admit part of a tie group (thr_mode 3).
// (grid-stride over the nch row chunks: a few CTAs per pair, so the common case -- no partial tie
// group -- costs a handful of early exits instead of one per chunk)
template <class Src>
__global__ void __launch_bounds__(TNT) k_thr_count(Geom g, DevParams P, MaskBuffers b,
                                                   const double* map, int nch) {
    const int p = blockIdx.y;
    const PairInfo& I = b.info[p];
    if (I.thr_mode != 3 || I.bits_ready) return;
    __shared__ unsigned long long se;
    const Src src = make_thr_src<Src>(g, P, b, p, map);
    const double bd = I.boundary;
    for (int chunk = blockIdx.x; chunk < nch; chunk += gridDim.x) {
        if (threadIdx.x == 0) se = 0;
        __syncthreads();
        const int y0 = chunk * TROWS, y1 = min(g.H, y0 + TROWS);
        unsigned int ce = 0;
        for (long long i = (long long)y0 * g.W + threadIdx.x; i < (long long)y1 * g.W; i += TNT)
            ce += src.value(i) == bd;
        for (int o = 16; o > 0; o >>= 1) ce += __shfl_xor_sync(0xffffffffu, ce, o);
        if ((threadIdx.x & 31) == 0 && ce) atomicAdd(&se, (unsigned long long)ce);
        __syncthreads();
        if (threadIdx.x == 0) b.tie_cnt[(size_t)p * nch + chunk] = se;
        __syncthreads();
    }
}

// Exclusive scan of the per-chunk tie counts (thr_mode 3 only).
__global__ void __launch_bounds__(1024) k_thr_scan(MaskBuffers b, int nch) {
    const int p = blockIdx.x;
    if (b.info[p].thr_mode != 3 || b.info[p].bits_ready) return;
    __shared__ unsigned long long seq[1024];
    unsigned long long* tc = b.tie_cnt + (size_t)p * nch;
    const int per = cdiv(nch, 1024);
    unsigned long long e = 0;
    for (int j = 0; j < per; ++j) {
        const int c = threadIdx.x * per + j;
        if (c < nch) e += tc[c];
    }
    seq[threadIdx.x] = e;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned long long ve = threadIdx.x >= o ? seq[threadIdx.x - o] : 0;
        __syncthreads();
        seq[threadIdx.x] += ve;
        __syncthreads();
    }
    unsigned long long run = threadIdx.x ? seq[threadIdx.x - 1] : 0;
    for (int j = 0; j < per; ++j) {
        const int c = threadIdx.x * per + j;
        if (c < nch) {
            const unsigned long long ce = tc[c];
            tc[c] = run;
            run += ce;
        }
    }
}

// Packed thresholded mask, bit x%32 of word (y, x/32); ties admitted in row-major order.
template <class Src>
__device__ __forceinline__ void thr_write_chunk(const Geom& g, const DevParams& P, const MaskBuffers& b,
                                                const double* map, const PairInfo& I, int p, int chunk,
                                                int nch, unsigned int* wcnt, unsigned long long& base) {
    const int y0 = chunk * TROWS, y1 = min(g.H, y0 + TROWS);
    uint32_t* out = b.bits_thr + (size_t)p * g.H * g.WW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = TNT / 32;
    const int nwords = (y1 - y0) * g.WW;
    if (I.thr_mode == 1) {
        for (int i = threadIdx.x; i < nwords; i += TNT) out[(size_t)y0 * g.WW + i] = 0u;
        return;
    }
    const Src src = make_thr_src<Src>(g, P, b, p, map);
    if (I.thr_mode != 3) {
        // no partial tie group: S >= b (mode 0) or S > 0 (mode 2), one word per warp
        for (int wi = warp; wi < nwords; wi += NW) {
            const int y = y0 + wi / g.WW, x = (wi % g.WW) * 32 + lane;
            bool on = false;
            if (x < g.W) {
                const double s = src.value((long long)y * g.W + x);
                on = I.thr_mode == 0 ? (s >= I.boundary) : (s > 0.0);
            }
            const unsigned int word = __ballot_sync(0xffffffffu, on);
            if (lane == 0) out[(size_t)y0 * g.WW + wi] = word;
        }
        return;
    }
    __syncthreads();  // the previous chunk is done with base / wcnt
    if (threadIdx.x == 0) base = b.tie_cnt[(size_t)p * nch + chunk];
    __syncthreads();
    for (int r0 = 0; r0 < nwords; r0 += NW) {
        const int wi = r0 + warp;
        bool gt = false, eq = false;
        if (wi < nwords) {
            const int y = y0 + wi / g.WW, x = (wi % g.WW) * 32 + lane;
            if (x < g.W) {
                const double s = src.value((long long)y * g.W + x);
                gt = s > I.boundary;
                eq = s == I.boundary;
            }
        }
        const unsigned int eqm = __ballot_sync(0xffffffffu, eq);
        const unsigned int gtm = __ballot_sync(0xffffffffu, gt);
        if (lane == 0) wcnt[warp] = __popc(eqm);
        __syncthreads();
        unsigned long long before = base;
        for (int k = 0; k < warp; ++k) before += wcnt[k];
        const unsigned long long rank = before + __popc(eqm & ((1u << lane) - 1u));
        const bool admit = eq && rank < I.need;
        const unsigned int word = gtm | __ballot_sync(0xffffffffu, admit);
        if (lane == 0 && wi < nwords) out[(size_t)y0 * g.WW + wi] = word;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int k = 0; k < NW; ++k) t += wcnt[k];
            base += t;
        }
        __syncthreads();
    }
}

// Packed thresholded mask, bit x%32 of word (y, x/32); ties admitted in row-major order.
// Grid-stride over the row chunks (see k_thr_count).
template <class Src>
__global__ void __launch_bounds__(TNT) k_thr_write(Geom g, DevParams P, MaskBuffers b,
                                                   const double* map, int nch) {
    const int p = blockIdx.y;
    const PairInfo I = b.info[p];
    if (I.bits_ready) return;  // written by the collect pass, settled by k_thr_fixup
    __shared__ unsigned int wcnt[TNT / 32];
    __shared__ unsigned long long base;
    for (int chunk = blockIdx.x; chunk < nch; chunk += gridDim.x)
        thr_write_chunk<Src>(g, P, b, map, I, p, chunk, nch, wcnt, base);
}

// Settles the boundary bin's candidates after phase B's collect pass wrote every other pixel's
// threshold bit (one CTA per pair): mode 0 admits S >= boundary, mode 2 S > 0, mode 3 S >
// boundary plus the first `need` tied pixels in row-major order (their indices sorted here).
constexpr int FXT = 1024;

__global__ void __launch_bounds__(FXT) k_thr_fixup(const Geom g, MaskBuffers b) {
    extern __shared__ unsigned int tie_idx[];  // kSelCap
    __shared__ unsigned int n_tie;
    const int p = blockIdx.x;
    const PairInfo I = b.info[p];
    if (!I.bits_ready) return;
    if (threadIdx.x == 0) n_tie = 0;
    __syncthreads();
    const unsigned int n = I.n_cand;
    const unsigned long long* keys = b.cand + (size_t)p * kMaxQueries * kSelCap;
    const unsigned int* idx = b.cand_idx + (size_t)p * kSelCap;
    uint32_t* bits = b.bits_thr + (size_t)p * g.H * g.WW;
    const unsigned long long kb = dkey(I.boundary);
    for (unsigned int i = threadIdx.x; i < n; i += FXT) {
        const unsigned long long k = keys[i];
        bool on;
        if (I.thr_mode == 0) on = k >= kb;
        else if (I.thr_mode == 2) on = k > 0ull;
        else {
            on = k > kb;
            if (k == kb) tie_idx[atomicAdd(&n_tie, 1u)] = idx[i];
        }
        if (on) atomicOr(bits + (idx[i] >> 5), 1u << (idx[i] & 31));
    }
    if (I.thr_mode != 3) return;
    __syncthreads();
    const unsigned int nt = n_tie;
    int np2 = 1;
    while (np2 < (int)nt) np2 <<= 1;
    for (int i = nt + threadIdx.x; i < np2; i += FXT) tie_idx[i] = 0xffffffffu;
    __syncthreads();
    for (int k2 = 2; k2 <= np2; k2 <<= 1)
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np2; i += FXT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k2) == 0;
                    const unsigned int a = tie_idx[i], c = tie_idx[ixj];
                    if ((a > c) == up) {
                        tie_idx[i] = c;
                        tie_idx[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (unsigned int i = threadIdx.x; i < nt && i < I.need; i += FXT)
        atomicOr(bits + (tie_idx[i] >> 5), 1u << (tie_idx[i] & 31));
}

// ------------------------------------------------------------------ morphology
constexpr int MROWS = 32, MNT = 256;

// One separable square op on rows [va, vb) of buffer `in` (rows ya.. in smem), result in `out`.
__device__ void morph_op(const uint32_t* in, uint32_t* out, uint32_t* tmp, int nrows, int WW,
                         int W, int H, int ya, int& va, int& vb, int r, bool erode) {
    if (r <= 0) {
        for (int i = threadIdx.x; i < nrows * WW; i += MNT) out[i] = in[i];
        __syncthreads();
        return;
    }
    const uint32_t fill = erode ? 0xffffffffu : 0u;
    const int tail = W & 31;
    const uint32_t tail_mask = tail ? ((1u << tail) - 1u) : 0xffffffffu;
    // horizontal pass: outside-the-row pixels act as `fill` (shrinking windows)
    for (int i = threadIdx.x; i < nrows * WW; i += MNT) {
        const int row = i / WW, j = i - row * WW;
        auto word = [&](int jj) -> uint32_t {
            if (jj < 0 || jj >= WW) return fill;
            uint32_t v = in[row * WW + jj];
            if (jj == WW - 1) v = (v & tail_mask) | (fill & ~tail_mask);
            return v;
        };
        const uint32_t c = word(j), lft = word(j - 1), rgt = word(j + 1);
        uint32_t acc = c;
        for (int k = 1; k <= r; ++k) {
            // pixel x-k: shift left by k bringing bits from the left word; x+k likewise
            const uint32_t sl = k < 32 ? ((c << k) | (lft >> (32 - k))) : lft;
            const uint32_t sr = k < 32 ? ((c >> k) | (rgt << (32 - k))) : rgt;
            acc = erode ? (acc & sl & sr) : (acc | sl | sr);
        }
        if (j == WW - 1) acc &= tail_mask;
        tmp[i] = acc;
    }
    __syncthreads();
    // vertical pass: rows outside the image are skipped (not filled)
    const int nva = (va == 0) ? 0 : va + r, nvb = (vb == H) ? H : vb - r;
    for (int i = threadIdx.x; i < nrows * WW; i += MNT) {
        const int row = i / WW, j = i - row * WW;
        const int y = ya + row;
        if (y < nva || y >= nvb) continue;
        uint32_t acc = erode ? 0xffffffffu : 0u;
        const int lo = max(0, y - r), hi = min(H - 1, y + r);
        for (int t = lo; t <= hi; ++t) {
            const uint32_t v = tmp[(t - ya) * WW + j];
            acc = erode ? (acc & v) : (acc | v);
        }
        out[i] = acc;
    }
    va = nva;
    vb = nvb;
    __syncthreads();
}

// morph_close(morph_open(m, ro), rc) (roi.hpp:179-180, 239) on a band of MROWS rows.
__global__ void __launch_bounds__(MNT) k_morph(Geom g, MaskBuffers b, int ro, int rc) {
    extern __shared__ uint32_t msm[];
    const int p = blockIdx.y;
    const int y0 = blockIdx.x * MROWS;
    const int halo = 2 * ro + 2 * rc;
    const int ya = max(0, y0 - halo), yb = min(g.H, y0 + MROWS + halo);
    const int nrows = yb - ya;
    uint32_t* A = msm;
    uint32_t* B = A + nrows * g.WW;
    uint32_t* Tm = B + nrows * g.WW;
    const uint32_t* src = b.bits_thr + (size_t)p * g.H * g.WW;
    for (int i = threadIdx.x; i < nrows * g.WW; i += MNT) A[i] = src[(size_t)ya * g.WW + i];
    __syncthreads();
    int va = ya, vb = yb;
    morph_op(A, B, Tm, nrows, g.WW, g.W, g.H, ya, va, vb, ro, true);   // erode
    morph_op(B, A, Tm, nrows, g.WW, g.W, g.H, ya, va, vb, ro, false);  // dilate
    morph_op(A, B, Tm, nrows, g.WW, g.W, g.H, ya, va, vb, rc, false);  // dilate
    morph_op(B, A, Tm, nrows, g.WW, g.W, g.H, ya, va, vb, rc, true);   // erode
    uint32_t* dst = b.bits_clean + (size_t)p * g.H * g.WW;
    const int ye = min(g.H, y0 + MROWS);
    for (int i = threadIdx.x; i < (ye - y0) * g.WW; i += MNT)
        dst[(size_t)y0 * g.WW + i] = A[(y0 - ya) * g.WW + i];
}

// ------------------------------------------------------------------ connected components
// 8-connected labelling on runs of set pixels (label_components roi.hpp:184-234 defines only
// the partition and the areas, which is all the area filter uses).  A run [x0, x1] of row y
// touches a run [c, d] of row y-1 iff c <= x1+1 and d >= x0-1.  Runs are extracted from the
// packed words with bit tricks (one warp per row), unions are lock-free atomicMin union-find on
// run ids, areas are summed at the roots, and surviving runs are painted into a keep mask.
constexpr int RNT = 256;  // 8 warps = 8 rows per CTA

__device__ __forceinline__ int rfind(int* P, int x) {
    while (true) {
        const int p = __ldcg(P + x);
        if (p == x) return x;
        x = p;
    }
}
__device__ __forceinline__ void runite(int* P, int a, int b) {
    bool done = false;
    while (!done) {
        a = rfind(P, a);
        b = rfind(P, b);
        if (a < b) {
            const int old = atomicMin(&P[b], a);
            done = old == b;
            b = old;
        } else if (b < a) {
            const int old = atomicMin(&P[a], b);
            done = old == a;
            a = old;
        } else {
            done = true;
        }
    }
}

__device__ __forceinline__ unsigned int warp_excl_scan(unsigned int v, unsigned int& total) {
    const int lane = threadIdx.x & 31;
    unsigned int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__global__ void __launch_bounds__(RNT) k_ccl_runs(Geom g, MaskBuffers b) {
    const int p = blockIdx.y, lane = threadIdx.x & 31;
    const int y = blockIdx.x * (RNT / 32) + (threadIdx.x >> 5);
    if (y >= g.H) return;
    const uint32_t* m = b.bits_clean + ((size_t)p * g.H + y) * g.WW;
    uint32_t* keep = b.bits_keep + ((size_t)p * g.H + y) * g.WW;
    const size_t rbase = ((size_t)p * g.H + y) * g.RMAX;
    uint16_t* x0 = b.run_x0 + rbase;
    uint16_t* x1 = b.run_x1 + rbase;
    int* par = b.run_par + (size_t)p * g.H * g.RMAX;
    unsigned int* area = b.run_area + (size_t)p * g.H * g.RMAX;
    unsigned int off_s = 0, off_e = 0;
    uint32_t carry = 0;  // last word of the previous 32-word chunk
    for (int w0 = 0; w0 < g.WW; w0 += 32) {
        const int j = w0 + lane;
        const uint32_t cur = j < g.WW ? m[j] : 0u;
        if (j < g.WW) keep[j] = 0u;
        uint32_t prv = __shfl_up_sync(0xffffffffu, cur, 1);
        if (lane == 0) prv = carry;
        uint32_t nxt = __shfl_down_sync(0xffffffffu, cur, 1);
        if (lane == 31) nxt = (j + 1 < g.WW) ? m[j + 1] : 0u;
        const uint32_t starts = cur & ~((cur << 1) | (prv >> 31));
        const uint32_t ends = cur & ~((cur >> 1) | (nxt << 31));
        unsigned int ts, te;
        unsigned int ks = off_s + warp_excl_scan(__popc(starts), ts);
        unsigned int ke = off_e + warp_excl_scan(__popc(ends), te);
        FROI_DCHECK(ks + __popc(starts) <= (unsigned)g.RMAX && ke + __popc(ends) <= (unsigned)g.RMAX);
        for (uint32_t bits = starts; bits; bits &= bits - 1) x0[ks++] = (uint16_t)(j * 32 + __ffs(bits) - 1);
        for (uint32_t bits = ends; bits; bits &= bits - 1) x1[ke++] = (uint16_t)(j * 32 + __ffs(bits) - 1);
        off_s += ts;
        off_e += te;
        carry = __shfl_sync(0xffffffffu, cur, 31);
    }
    if (lane == 0) b.run_n[(size_t)p * g.H + y] = (int)off_s;
    for (unsigned int k = lane; k < off_s; k += 32) {
        const int id = y * g.RMAX + (int)k;
        par[id] = id;
        area[id] = 0u;
    }
}

__global__ void __launch_bounds__(RNT) k_ccl_union(Geom g, MaskBuffers b) {
    const int p = blockIdx.y, lane = threadIdx.x & 31;
    const int y = blockIdx.x * (RNT / 32) + (threadIdx.x >> 5);
    if (y < 1 || y >= g.H) return;
    const int* rn = b.run_n + (size_t)p * g.H;
    const int n = rn[y], np = rn[y - 1];
    if (n == 0 || np == 0) return;
    const size_t base = (size_t)p * g.H * g.RMAX;
    const uint16_t* x0 = b.run_x0 + base + (size_t)y * g.RMAX;
    const uint16_t* x1 = b.run_x1 + base + (size_t)y * g.RMAX;
    const uint16_t* px0 = b.run_x0 + base + (size_t)(y - 1) * g.RMAX;
    const uint16_t* px1 = b.run_x1 + base + (size_t)(y - 1) * g.RMAX;
    int* par = b.run_par + base;
    for (int k = lane; k < n; k += 32) {
        const int a = x0[k], e = x1[k];
        int lo = 0, hi = np;  // first run of row y-1 with x1 >= a-1
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)px1[mid] < a - 1) lo = mid + 1; else hi = mid;
        }
        FROI_DCHECK(n <= g.RMAX && np <= g.RMAX && a <= e && e < g.W);
        for (int j = lo; j < np && (int)px0[j] <= e + 1; ++j)
            runite(par, y * g.RMAX + k, (y - 1) * g.RMAX + j);
    }
}

__global__ void __launch_bounds__(RNT) k_ccl_area(Geom g, MaskBuffers b) {
    const int p = blockIdx.y, lane = threadIdx.x & 31;
    const int y = blockIdx.x * (RNT / 32) + (threadIdx.x >> 5);
    if (y >= g.H) return;
    const int n = b.run_n[(size_t)p * g.H + y];
    const size_t base = (size_t)p * g.H * g.RMAX;
    int* par = b.run_par + base;
    for (int k = lane; k < n; k += 32) {
        const int id = y * g.RMAX + k;
        const int len = (int)b.run_x1[base + id] - (int)b.run_x0[base + id] + 1;
        atomicAdd(&b.run_area[base + rfind(par, id)], (unsigned int)len);
    }
}

// Paints the runs of components with area >= min_area into the keep mask; counts components.
__global__ void __launch_bounds__(RNT) k_ccl_keep(Geom g, DevParams P, MaskBuffers b) {
    const int p = blockIdx.y, lane = threadIdx.x & 31;
    const int y = blockIdx.x * (RNT / 32) + (threadIdx.x >> 5);
    unsigned int comps = 0;
    if (y < g.H) {
        const int n = b.run_n[(size_t)p * g.H + y];
        const size_t base = (size_t)p * g.H * g.RMAX;
        int* par = b.run_par + base;
        uint32_t* keep = b.bits_keep + ((size_t)p * g.H + y) * g.WW;
        for (int k = lane; k < n; k += 32) {
            const int id = y * g.RMAX + k;
            const int r = rfind(par, id);
            const bool ok = b.run_area[base + r] >= (unsigned int)P.min_area;
            comps += (ok && r == id);
            if (!ok) continue;
            const int a = b.run_x0[base + id], e = b.run_x1[base + id];
            for (int wd = a >> 5; wd <= (e >> 5); ++wd) {
                const int lo = max(a, wd * 32) - wd * 32, hi = min(e, wd * 32 + 31) - wd * 32;
                const uint32_t msk = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
                atomicOr(keep + wd, msk);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) comps += __shfl_xor_sync(0xffffffffu, comps, o);
    if (lane == 0 && comps) atomicAdd(&b.info[p].components, comps);
}

__device__ __forceinline__ bool bit_at(const uint32_t* m, int WW, int x, int y) {
    return (m[(size_t)y * WW + (x >> 5)] >> (x & 31)) & 1u;
}

// Area filter result (keep mask or the cleaned mask) + unshift_mask + PBM packing + pixel count.
// One thread per PBM byte.
// 8 source bits at columns sx0 .. sx0+7 of one packed row (0 outside [0, W)), bit k = column sx0+k
__device__ __forceinline__ unsigned int src_bits8(const uint32_t* row, int WW, int W, int sx0) {
    const int wi = sx0 >> 5, sh = sx0 & 31;  // floor division also for negative sx0
    const uint32_t lo = (wi >= 0 && wi < WW) ? row[wi] : 0u;
    const uint32_t hi = (wi + 1 >= 0 && wi + 1 < WW) ? row[wi + 1] : 0u;
    unsigned int v = (unsigned int)(((((unsigned long long)hi) << 32) | lo) >> sh) & 0xffu;
    const int valid = W - sx0;  // columns >= W are outside
    if (valid < 8) v &= valid <= 0 ? 0u : ((1u << valid) - 1u);
    return v;
}

// unshift_mask (registration.hpp:111-121) fused with the PBM packing: output byte (y, x0..x0+7)
// takes source columns x0-dx .. x0-dx+7 of source row y-dy (zero outside), MSB first.
__global__ void __launch_bounds__(256) k_output(Geom g, DevParams P, MaskBuffers b, int use_ccl) {
    const int p = blockIdx.y;
    const PairInfo I = b.info[p];
    const int nbytes = g.H * g.SB;
    const uint32_t* m = (use_ccl ? b.bits_keep : b.bits_clean) + (size_t)p * g.H * g.WW;
    uint8_t* out = b.out_pbm + (size_t)b.out_index[p] * nbytes;
    unsigned int cnt = 0;
    for (int bi = blockIdx.x * 256 + threadIdx.x; bi < nbytes; bi += gridDim.x * 256) {
        const int y = bi / g.SB, x0 = (bi - y * g.SB) * 8;
        const int sy = y - I.dy;
        unsigned int byte = 0;
        if (sy >= 0 && sy < g.H) {
            unsigned int v = src_bits8(m + (size_t)sy * g.WW, g.WW, g.W, x0 - I.dx);
            const int outw = g.W - x0;  // output columns beyond W stay 0
            if (outw < 8) v &= outw <= 0 ? 0u : ((1u << outw) - 1u);
            byte = __brev(v) >> 24;  // column x0 -> bit 7
        }
        out[bi] = (uint8_t)byte;
        cnt += __popc(byte);
    }
    // one atomic per CTA (per-warp atomics on one counter per pair serialise)
    __shared__ unsigned int wsum[8];
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int t = 0;
        for (int k = 0; k < 8; ++k) t += wsum[k];
        if (t) atomicAdd(&b.info[p].mask_count, t);
    }
}

__global__ void k_reset_counts(MaskBuffers b) {
    b.info[blockIdx.x].mask_count = 0;
    b.info[blockIdx.x].components = 0;
}

__global__ void k_unpack_masks(const uint8_t* pbm, uint8_t* bytes, int W, int H, int SB, int n) {
    const long long per = (long long)W * H;
    const long long total = per * n;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
        const long long k = i / per, r = i - k * per;
        const int y = (int)(r / W), x = (int)(r - (long long)y * W);
        bytes[i] = (pbm[k * H * SB + (long long)y * SB + (x >> 3)] >> (7 - (x & 7))) & 1u;
    }
}

__global__ void k_pack_words(const uint8_t* bytes, uint32_t* words, int W, int H, int WW) {
    const long long n = (long long)H * WW;
    for (long long wi = blockIdx.x * 256LL + threadIdx.x; wi < n; wi += (long long)gridDim.x * 256) {
        const int y = (int)(wi / WW), xb = (int)(wi % WW) * 32;
        uint32_t v = 0;
        for (int k = 0; k < 32; ++k) {
            const int x = xb + k;
            if (x < W && bytes[(size_t)y * W + x]) v |= 1u << k;
        }
        words[wi] = v;
    }
}

__global__ void k_ensemble(const uint8_t* in, uint8_t* out, long long per, int n, int k) {
    const long long total = per * n;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
        const int t = (int)(i / per);
        const long long o = i - (long long)t * per;
        uint8_t v = 0;
        const int lo = max(0, t - k), hi = min(n - 1, t + k);
        for (int j = lo; j <= hi; ++j) v |= in[(long long)j * per + o];
        out[i] = v;
    }
}

__global__ void __launch_bounds__(256) k_saliency_map(Geom g, DevParams P, MaskBuffers b,
                                                      double* out) {
    const SrcSal src = make_thr_src<SrcSal>(g, P, b, 0, nullptr);
    const long long n = (long long)g.W * g.H;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
        out[i] = dadd(src.value(i), 0.0);  // -0 (degenerate range, see normalize) reads as +0
}

int grid_for(long long work, int per_block) {
    long long b = cdiv<long long>(work, per_block);
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

// grid-wide pass + scan launches per phase that normally finish the selection (after the first
// pass fused into k_mag_grad for phase A); whatever is left is finished by k_sel_rest_*
constexpr int kSelPassesA = 1, kSelPassesB = 2;
// FROI_SEL_GRID_PASSES=n overrides both counts (0: every step through k_sel_rest_*; a test knob)
int sel_passes(int dflt) {
    static const int v = [] {
        const char* e = getenv("FROI_SEL_GRID_PASSES");
        return e ? atoi(e) : -1;
    }();
    return v >= 0 ? v : dflt;
}

size_t scan_smem() { return sizeof(unsigned long long) * kSelCap; }
size_t rest_smem() { return std::max(scan_smem(), std::max(pass_smem(4), pass_smem(1))); }

// kernel attributes are per device: set on every call (one host thread may drive several devices)
void set_scan_smem() {
    FROI_CUDA(cudaFuncSetAttribute(k_sel_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem(4)));
    FROI_CUDA(cudaFuncSetAttribute(k_sel_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem(1)));
    FROI_CUDA(cudaFuncSetAttribute(k_sel_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem()));
    FROI_CUDA(cudaFuncSetAttribute(k_thr_fixup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(unsigned int) * kSelCap)));
    FROI_CUDA(cudaFuncSetAttribute(k_sel_rest_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rest_smem()));
    FROI_CUDA(cudaFuncSetAttribute(k_sel_rest_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rest_smem()));
}

// CTAs per pair for the row-/range-blocked mask kernels: a whole number of waves over the SMs
// (ctas_per_sm resident CTAs each), so no wave runs a few stragglers alone -- e.g. 32 pairs x 19
// blocks on 2 x 148 slots was 2.05 waves, i.e. three rounds.
int sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}
int blocks_per_pair(const Geom& g, int n_pairs, int ctas_per_sm, int waves = 2) {
    const long long n = (long long)g.W * g.H;
    const int bpp = (int)std::max<long long>(1, (long long)waves * sm_count() * ctas_per_sm / n_pairs);
    return (int)std::max<long long>(1, std::min<long long>(bpp, cdiv<long long>(n, 8192)));
}

// Phase A: the four robust_normalize percentiles.
template <typename T>
void run_stats(const Geom& g, const DevParams& P, const MaskBuffers& b, int n_pairs, cudaStream_t s,
               uint64_t* launches) {
    const long long n = (long long)g.W * g.H;
    const int bpp = blocks_per_pair(g, n_pairs, 2);  // k_sel_pass_a: 2 CTAs per SM
    const int mgb = blocks_per_pair(g, n_pairs, 4);  // k_mag_grad: 4 CTAs per SM
    set_scan_smem();
    k_sel_init_a<<<n_pairs, 32, 0, s>>>(b, (unsigned long long)n, (unsigned long long)(0.01 * (double)(n - 1)),
                                       (unsigned long long)(0.99 * (double)(n - 1)));
    if (sizeof(T) == 1 && P.gradient_source == 0 && P.grad_tab)
        k_mag_grad<T, true><<<dim3(mgb, n_pairs), PNT_MG, 0, s>>>(g, P, b);
    else
        k_mag_grad<T, false><<<dim3(mgb, n_pairs), PNT_MG, 0, s>>>(g, P, b);
    k_sel_scan<<<n_pairs * 4, SCT, scan_smem(), s>>>(b, 4);
    FROI_LAUNCH_CHECK();
    *launches += 3;
    for (int it = 0; it < sel_passes(kSelPassesA); ++it) {
        k_sel_pass_a<<<dim3(bpp, n_pairs), SNT, pass_smem(4), s>>>(g, b);
        k_sel_scan<<<n_pairs * 4, SCT, scan_smem(), s>>>(b, 4);
        FROI_LAUNCH_CHECK();
        *launches += 2;
    }
    k_sel_rest_a<<<n_pairs, SCT, rest_smem(), s>>>(g, b);
    FROI_LAUNCH_CHECK();
    ++*launches;
}

// Phase B: the round(t*n)-th largest saliency (or map value) and the tie decision.
void run_boundary(const Geom& g, const DevParams& P, const MaskBuffers& b, int n_pairs,
                  const double* map, bool from_stats, cudaStream_t s, uint64_t* launches) {
    const long long n = (long long)g.W * g.H;
    const int bpp = blocks_per_pair(g, n_pairs, 2);  // k_sel_pass_b: 2 CTAs per SM
    set_scan_smem();
    const unsigned long long target = (unsigned long long)llround(P.roi_threshold * (double)n);
    k_sel_init_b<<<n_pairs, 32, 0, s>>>(b, (unsigned long long)n, target, from_stats ? 1 : 0);
    FROI_LAUNCH_CHECK();
    ++*launches;
    // threshold words fused into the collect pass when rows are whole 32-bit words
    const int bits = g.W % 32 == 0 ? 1 : 0;
    // frames above 2 Mpx (C4's 2048^2): the boundary's exponent-window bin usually exceeds the
    // kSelCap keys a collect can take, so an 11-bit radix pass comes before the collect -- run that
    // third pass on the whole grid too instead of in k_sel_rest_b's one CTA per pair
    const int passes_b = sel_passes(n > (1ll << 21) ? kSelPassesB + 1 : kSelPassesB);
    for (int it = 0; it < passes_b; ++it) {
        k_sel_pass_b<<<dim3(bpp, n_pairs), SNT, pass_smem(1), s>>>(g, P, b, map, bits);
        k_sel_scan<<<n_pairs, SCT, scan_smem(), s>>>(b, 1, bits);
        FROI_LAUNCH_CHECK();
        *launches += 2;
    }
    k_sel_rest_b<<<n_pairs, SCT, rest_smem(), s>>>(g, P, b, map, bits);
    FROI_LAUNCH_CHECK();
    ++*launches;
    k_sel_finish_b<<<n_pairs, 32, 0, s>>>(b, (unsigned long long)n);
    FROI_LAUNCH_CHECK();
    ++*launches;
    if (bits) {
        k_thr_fixup<<<n_pairs, FXT, sizeof(unsigned int) * kSelCap, s>>>(g, b);
        FROI_LAUNCH_CHECK();
        ++*launches;
    }
}

template <class Src>
void run_threshold(const Geom& g, const DevParams& P, const MaskBuffers& b, int n_pairs,
                   const double* map, cudaStream_t s, uint64_t* launches) {
    const int nch = cdiv(g.H, TROWS);
    const int gx = std::min(nch, 16);
    k_thr_count<Src><<<dim3(gx, n_pairs), TNT, 0, s>>>(g, P, b, map, nch);
    k_thr_scan<<<n_pairs, 1024, 0, s>>>(b, nch);
    k_thr_write<Src><<<dim3(gx, n_pairs), TNT, 0, s>>>(g, P, b, map, nch);
    FROI_LAUNCH_CHECK();
    *launches += 3;
}

void run_cleanup_output(const Geom& g, const DevParams& P, const MaskBuffers& b, int n_pairs,
                        int ro, int rc, int min_area, cudaStream_t s, uint64_t* launches) {
    DevParams Q = P;
    Q.min_area = min_area;
    k_reset_counts<<<n_pairs, 1, 0, s>>>(b);
    const int halo = 2 * ro + 2 * rc;
    const size_t smem = sizeof(uint32_t) * 3 * (size_t)(MROWS + 2 * halo) * g.WW;
    if (smem > 48 * 1024)
        FROI_CUDA(cudaFuncSetAttribute(k_morph, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_morph<<<dim3(cdiv(g.H, MROWS), n_pairs), MNT, smem, s>>>(g, b, ro, rc);
    FROI_LAUNCH_CHECK();
    *launches += 2;
    const bool use_ccl = min_area > 1;
    if (use_ccl) {
        dim3 rows(cdiv(g.H, RNT / 32), n_pairs);
        k_ccl_runs<<<rows, RNT, 0, s>>>(g, b);
        k_ccl_union<<<rows, RNT, 0, s>>>(g, b);
        k_ccl_area<<<rows, RNT, 0, s>>>(g, b);
        k_ccl_keep<<<rows, RNT, 0, s>>>(g, Q, b);
        FROI_LAUNCH_CHECK();
        *launches += 4;
    }
    k_output<<<dim3(grid_for((long long)g.H * g.SB, 4096), n_pairs), 256, 0, s>>>(g, Q, b, use_ccl ? 1 : 0);
    FROI_LAUNCH_CHECK();
    ++*launches;
}

}  // namespace

__global__ void k_grad_table(const double* __restrict__ mag, int nv, double* __restrict__ tab) {
    const int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nv) tab[(size_t)i * nv + j] = hypot_glibc(mag[i], mag[j]);
}

void launch_grad_table(const double* d_mag, int nv, double* d_tab, cudaStream_t s) {
    k_grad_table<<<dim3(cdiv(nv, 256), nv), 256, 0, s>>>(d_mag, nv, d_tab);
    FROI_LAUNCH_CHECK();
}

void launch_mask_stage(const Geom& g, const DevParams& P, const MaskBuffers& b, int n_pairs,
                       cudaStream_t s, uint64_t* launches) {
    if (n_pairs <= 0) return;
    if (g.sample_bytes == 1) run_stats<uint8_t>(g, P, b, n_pairs, s, launches);
    else run_stats<uint16_t>(g, P, b, n_pairs, s, launches);
    run_boundary(g, P, b, n_pairs, nullptr, true, s, launches);
    run_threshold<SrcSal>(g, P, b, n_pairs, nullptr, s, launches);
    run_cleanup_output(g, P, b, n_pairs, P.open_radius, P.close_radius, P.min_area, s, launches);
}

void launch_saliency_map(const Geom& g, const DevParams& P, const MaskBuffers& b, double* d_out,
                         cudaStream_t s) {
    uint64_t l = 0;
    if (g.sample_bytes == 1) run_stats<uint8_t>(g, P, b, 1, s, &l);
    else run_stats<uint16_t>(g, P, b, 1, s, &l);
    run_boundary(g, P, b, 1, nullptr, true, s, &l);
    k_saliency_map<<<grid_for((long long)g.W * g.H, 256), 256, 0, s>>>(g, P, b, d_out);
    FROI_LAUNCH_CHECK();
}

void launch_threshold_from_map(const Geom& g, const DevParams& P, const MaskBuffers& b,
                               const double* d_map, double threshold, cudaStream_t s) {
    uint64_t l = 0;
    DevParams Q = P;
    Q.roi_threshold = threshold;
    run_boundary(g, Q, b, 1, d_map, false, s, &l);
    run_threshold<SrcMap>(g, Q, b, 1, d_map, s, &l);
}

void launch_cleanup_only(const Geom& g, const DevParams& P, const MaskBuffers& b,
                         int open_radius, int close_radius, int min_area, cudaStream_t s) {
    uint64_t l = 0;
    run_cleanup_output(g, P, b, 1, open_radius, close_radius, min_area, s, &l);
}

void launch_unpack_pbm(const Geom& g, const uint8_t* d_pbm, uint8_t* d_bytes, int n_masks,
                       cudaStream_t s) {
    if (n_masks <= 0) return;
    k_unpack_masks<<<grid_for((long long)g.W * g.H * n_masks, 256), 256, 0, s>>>(d_pbm, d_bytes, g.W,
                                                                               g.H, g.SB, n_masks);
    FROI_LAUNCH_CHECK();
}

void launch_pack_bytes_to_words(const Geom& g, const uint8_t* d_bytes, uint32_t* d_words,
                                cudaStream_t s) {
    k_pack_words<<<grid_for((long long)g.H * g.WW, 256), 256, 0, s>>>(d_bytes, d_words, g.W, g.H, g.WW);
    FROI_LAUNCH_CHECK();
}

void launch_ensemble(const Geom& g, const uint8_t* d_in, uint8_t* d_out, int n, int k,
                     cudaStream_t s) {
    const long long per = (long long)g.H * g.SB;
    k_ensemble<<<grid_for(per * n, 256), 256, 0, s>>>(d_in, d_out, per, n, k);
    FROI_LAUNCH_CHECK();
}

}  // namespace froi
