// Input side of the decoder (harness, not the hot path): frozen-set
// construction and the BPSK/AWGN channel (include/polar_b200_sim.h).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <curand_kernel.h>

#include "../../include/polar_b200_sim.h"
#include "channel.h"

namespace plb {

// ---- frozen sets ---------------------------------------------------------

// Bhattacharyya profile in natural order: the left (check-node) child of a
// node with parameter v gets 2v - v^2, the right child v^2 (code.cpp:35-43).
static void bhat_fill(std::vector<double>& z, size_t lo, size_t sz, double v) {
    if (sz == 1) {
        z[lo] = v;
        return;
    }
    bhat_fill(z, lo, sz / 2, 2.0 * v - v * v);
    bhat_fill(z, lo + sz / 2, sz / 2, v * v);
}

// Gaussian approximation (Trifonov 2012, Chung's phi): mean LLR of each bit
// channel.  Left child: phi^-1(1 - (1 - phi(m))^2); right child: 2m.
// Evaluated in the log domain so large means do not underflow.
static double ln_phi(double x) {
    if (x <= 0) return 0.0;
    if (x <= 10.0) return -0.4527 * std::pow(x, 0.86) + 0.0218;
    return 0.5 * std::log(M_PI / x) - x / 4.0 + std::log1p(-10.0 / (7.0 * x));
}

static double inv_ln_phi(double target) {
    // ln_phi is decreasing on (0, inf)
    double lo = 0.0, hi = 1.0;
    while (ln_phi(hi) > target) hi *= 2.0;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (ln_phi(mid) > target) lo = mid;
        else hi = mid;
        if (hi - lo <= 1e-12 * hi) break;
    }
    return 0.5 * (lo + hi);
}

static double ga_check(double m) {
    // phi_out = 1 - (1 - phi)^2 = phi (2 - phi)
    const double lp = ln_phi(m);
    const double p = std::exp(lp);
    const double lout = lp + std::log(2.0 - p);
    return inv_ln_phi(lout);
}

static void ga_fill(std::vector<double>& mu, size_t lo, size_t sz, double m) {
    if (sz == 1) {
        mu[lo] = m;
        return;
    }
    ga_fill(mu, lo, sz / 2, ga_check(m));
    ga_fill(mu, lo + sz / 2, sz / 2, 2.0 * m);
}

static bool pow2(int n) { return n >= 2 && (n & (n - 1)) == 0; }

} // namespace plb

extern "C" int pl_construct_frozen_bhat(int32_t n, int32_t reliable, double design,
                                        uint8_t* out) {
    if (!out || !plb::pow2(n) || reliable < 1 || reliable > n || !(design > 0.0) || !(design < 1.0))
        return PL_ERR_CONFIG;
    std::vector<double> z(static_cast<size_t>(n));
    plb::bhat_fill(z, 0, size_t(n), design);
    std::vector<int> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    // frozen first: largest erasure figure, ties toward the lower index
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return z[size_t(a)] > z[size_t(b)]; });
    std::memset(out, 0, size_t(n));
    for (int j = 0; j < n - reliable; ++j) out[idx[size_t(j)]] = 1;
    return PL_OK;
}

extern "C" int pl_construct_frozen_ga(int32_t n, int32_t reliable, double design_ebn0_db,
                                      double rate, uint8_t* out) {
    if (!out || !plb::pow2(n) || reliable < 1 || reliable > n || !(rate > 0.0)) return PL_ERR_CONFIG;
    const double sigma2 = 1.0 / (2.0 * rate * std::pow(10.0, design_ebn0_db / 10.0));
    std::vector<double> mu(static_cast<size_t>(n));
    plb::ga_fill(mu, 0, size_t(n), 2.0 / sigma2);
    std::vector<int> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return mu[size_t(a)] < mu[size_t(b)]; });
    std::memset(out, 0, size_t(n));
    for (int j = 0; j < n - reliable; ++j) out[idx[size_t(j)]] = 1;
    return PL_OK;
}

namespace plb {

// ---- host channel (FrameRng semantics, channel.hpp:17-89) ----------------

struct HostChannelCode {
    int n, k, width;
    std::vector<int> info_pos;
    std::vector<uint64_t> amask; // open positions, MSB-first words
    pl_crc crc;
    // crc over k message bits as an affine map (c0, columns), MSB-first value
    uint64_t c0 = 0;
    std::vector<uint64_t> col;
};

// in-place n-fold butterfly on an MSB-first packed word (code.cpp:12-31)
void polar_transform_words(uint64_t* w, int n) {
    static const uint64_t stride_mask[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull,
                                            0xF0F0F0F0F0F0F0F0ull, 0xFF00FF00FF00FF00ull,
                                            0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
    const int nw = (n + 63) / 64;
    for (int inc = 1; inc < n; inc <<= 1) {
        if (inc < 64) {
            int lg = 0;
            while ((1 << lg) < inc) ++lg;
            const uint64_t m = stride_mask[lg];
            for (int j = 0; j < nw; ++j) w[j] ^= (w[j] << inc) & m;
        } else {
            const int ws = inc / 64;
            for (int j = 0; j < nw; ++j)
                if ((j & ws) == 0) w[j] ^= w[j + ws];
        }
    }
}

class FrameRng {
public:
    FrameRng(uint64_t seed, uint64_t frame) {
        const uint64_t s = seed ^ frame;
        gen_.seed(uint32_t(s ^ (s >> 32)));
    }
    bool coin() { return (gen_() & 1u) != 0; }
    double gaussian() {
        if (have_) {
            have_ = false;
            return spare_;
        }
        const double u1 = (double(gen_()) + 1.0) * 0x1p-32;
        const double u2 = (double(gen_()) + 1.0) * 0x1p-32;
        const double mag = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * M_PI * u2;
        spare_ = mag * std::sin(ang);
        have_ = true;
        return mag * std::cos(ang);
    }

private:
    std::mt19937 gen_;
    double spare_ = 0;
    bool have_ = false;
};

} // namespace plb

namespace plb {
// frame i of the output is keyed by ids ? ids[i] : frame0 + i
static int channel_core(const pl_code* code, double ebn0_db, uint64_t seed, uint64_t frame0,
                        const uint64_t* ids, int64_t nframes, int32_t precision, float scale,
                        uint8_t* info_out, int64_t info_stride, void* llr_out,
                        int64_t llr_stride, int32_t nthreads);
} // namespace plb

extern "C" int pl_channel_generate(const pl_code* code, double ebn0_db, uint64_t seed,
                                   uint64_t frame0, int64_t nframes, int32_t precision,
                                   float scale, uint8_t* info_out, void* llr_out,
                                   int32_t nthreads) {
    if (!code) return PL_ERR_ARG;
    return plb::channel_core(code, ebn0_db, seed, frame0, nullptr, nframes, precision, scale,
                             info_out, code->k, llr_out, code->n, nthreads);
}

extern "C" int pl_channel_generate_frames(const pl_code* code, double ebn0_db, uint64_t seed,
                                          const uint64_t* frame_ids, int64_t nframes,
                                          int32_t precision, float scale, uint8_t* info_out,
                                          int64_t info_stride, void* llr_out, int64_t llr_stride,
                                          int32_t nthreads) {
    if (!code || (!frame_ids && nframes > 0) || llr_stride < code->n ||
        (info_out && info_stride < code->k))
        return PL_ERR_ARG;
    return plb::channel_core(code, ebn0_db, seed, 0, frame_ids, nframes, precision, scale,
                             info_out, info_stride, llr_out, llr_stride, nthreads);
}

static int plb::channel_core(const pl_code* code, double ebn0_db, uint64_t seed, uint64_t frame0,
                             const uint64_t* ids, int64_t nframes, int32_t precision, float scale,
                             uint8_t* info_out, int64_t info_stride, void* llr_out,
                             int64_t llr_stride, int32_t nthreads) {
    using namespace plb;
    if (!code || !code->frozen || !llr_out || nframes < 0 || !pow2(code->n) || code->k < 1)
        return PL_ERR_ARG;
    if (precision != PL_F32 && precision != PL_I8 && precision != PL_I16) return PL_ERR_CONFIG;
    const int n = code->n, k = code->k, w = code->crc.width;
    std::vector<int> info_pos;
    for (int i = 0; i < n; ++i)
        if (!code->frozen[i]) info_pos.push_back(i);
    if (int(info_pos.size()) != k + w) return PL_ERR_CONFIG;
    const int nw = (n + 63) / 64;
    std::vector<uint64_t> amask(size_t(nw), 0);
    for (int p : info_pos) amask[size_t(p >> 6)] |= 1ull << (63 - (p & 63));
    // CRC of the message via the ABI's engine (crc.cpp semantics)
    uint64_t c0 = 0;
    std::vector<uint64_t> col;
    if (w) {
        std::vector<uint8_t> msg(size_t(k), 0);
        if (pl_crc_compute(&code->crc, msg.data(), k, &c0) != PL_OK) return PL_ERR_CONFIG;
        col.resize(size_t(k));
        for (int j = 0; j < k; ++j) {
            msg[size_t(j)] = 1;
            uint64_t v = 0;
            pl_crc_compute(&code->crc, msg.data(), k, &v);
            col[size_t(j)] = v ^ c0;
            msg[size_t(j)] = 0;
        }
    }
    // puncturing (channel.hpp:62-89): the rate counts transmitted uses only
    const uint8_t* use = code->channel_use;
    int transmitted = n;
    if (use) {
        transmitted = 0;
        for (int i = 0; i < n; ++i) {
            if (use[i] > PL_USE_SHORTENED) return PL_ERR_CONFIG;
            transmitted += use[i] == PL_USE_TRANSMITTED;
        }
        if (transmitted < k + w) return PL_ERR_CONFIG;
    }
    const double rate = double(k) / double(transmitted);
    const double sigma2 = 1.0 / (2.0 * rate * std::pow(10.0, ebn0_db / 10.0));
    const double sigma = std::sqrt(sigma2);
    const double demap = 2.0 / sigma2;
    // default_quant_scale (channel.hpp:94-100)
    const float qs = scale > 0 ? scale : (precision == PL_I8 ? 8.0f : precision == PL_I16 ? 64.0f : 1.0f);
    auto work = [&](int64_t a, int64_t b) {
        std::vector<uint64_t> u(static_cast<size_t>(nw));
        std::vector<uint8_t> info(static_cast<size_t>(k));
        for (int64_t f = a; f < b; ++f) {
            FrameRng rng(seed, ids ? ids[f] : frame0 + uint64_t(f));
            uint64_t crcv = c0;
            for (int i = 0; i < k; ++i) {
                info[size_t(i)] = rng.coin() ? 1 : 0;
                if (w && info[size_t(i)]) crcv ^= col[size_t(i)];
            }
            if (info_out) std::memcpy(info_out + f * info_stride, info.data(), size_t(k));
            std::fill(u.begin(), u.end(), 0);
            auto setbit = [&](int pos) { u[size_t(pos >> 6)] |= 1ull << (63 - (pos & 63)); };
            for (int j = 0; j < k; ++j)
                if (info[size_t(j)]) setbit(info_pos[size_t(j)]);
            for (int j = 0; j < w; ++j)
                if ((crcv >> (w - 1 - j)) & 1) setbit(info_pos[size_t(k + j)]);
            polar_transform_words(u.data(), n);
            for (int j = 0; j < nw; ++j) u[size_t(j)] &= amask[size_t(j)];
            polar_transform_words(u.data(), n);
            for (int i = 0; i < n; ++i) {
                const int ui = use ? use[i] : PL_USE_TRANSMITTED;
                if (ui != PL_USE_TRANSMITTED) { // no noise draw (channel.hpp:70-80)
                    const bool sh = ui == PL_USE_SHORTENED; // known_zero_llr (llr.hpp:105-111)
                    if (precision == PL_F32)
                        static_cast<float*>(llr_out)[f * llr_stride + i] = sh ? 1e9f : 0.0f;
                    else if (precision == PL_I8)
                        static_cast<int8_t*>(llr_out)[f * llr_stride + i] = int8_t(sh ? 127 : 0);
                    else
                        static_cast<int16_t*>(llr_out)[f * llr_stride + i] = int16_t(sh ? 32767 : 0);
                    continue;
                }
                const bool x = (u[size_t(i >> 6)] >> (63 - (i & 63))) & 1;
                const double s = x ? -1.0 : 1.0;
                const double y = s + sigma * rng.gaussian();
                const float v = float(demap * y);
                if (precision == PL_F32) {
                    static_cast<float*>(llr_out)[f * llr_stride + i] = v;
                } else if (precision == PL_I8) {
                    const float q = std::round(v * qs);
                    static_cast<int8_t*>(llr_out)[f * llr_stride + i] =
                        int8_t(std::clamp(q, -127.0f, 127.0f));
                } else {
                    const float q = std::round(v * qs);
                    static_cast<int16_t*>(llr_out)[f * llr_stride + i] =
                        int16_t(std::clamp(q, -32767.0f, 32767.0f));
                }
            }
        }
    };
    int nt = nthreads > 0 ? nthreads : int(std::thread::hardware_concurrency());
    nt = int(std::max<int64_t>(1, std::min<int64_t>(nt, nframes)));
    if (nt == 1) {
        work(0, nframes);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back(work, nframes * t / nt, nframes * (t + 1) / nt);
        for (auto& th : pool) th.join();
    }
    return PL_OK;
}

// ---- device channel (statistically equivalent, Philox keyed by frame) ----
namespace plb {
namespace {

struct ChanParams {
    int n, k, w, rw;
    const int32_t* info_pos; // k + w
    const uint8_t* use;      // n channel uses, nullable
    const uint64_t* col;     // k CRC columns
    uint64_t c0;
    float sigma, demap, qs;
    int precision;
    uint64_t seed, frame0;
    int64_t nframes;
    uint8_t* info_out;
    void* llr_out;
};

// LSB-first words: x[i] ^= x[i + inc] for every i with (i & inc) == 0
__device__ void transform_row(uint32_t* row, int n, int rw, int lane) {
    static constexpr uint32_t mk[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu,
                                       0x0000FFFFu};
    for (int lg = 0; (1 << lg) < n && lg < 5; ++lg) {
        const int inc = 1 << lg;
        for (int j = lane; j < rw; j += 32) row[j] ^= (row[j] >> inc) & mk[lg];
        __syncwarp();
    }
    for (int ws = 1; ws < rw; ws <<= 1) {
        for (int j = lane; j < rw; j += 32)
            if ((j & ws) == 0) row[j] ^= row[j + ws];
        __syncwarp();
    }
}

__global__ void chan_kernel(const ChanParams P) {
    extern __shared__ uint32_t srow[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* row = srow + wib * P.rw;
    const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t f = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib; f < P.nframes; f += nw) {
        curandStatePhilox4_32_10_t st;
        curand_init(P.seed, (P.frame0 + uint64_t(f)) * 32u + uint64_t(lane), 0, &st);
        for (int j = lane; j < P.rw; j += 32) row[j] = 0;
        __syncwarp();
        uint64_t crc = 0;
        for (int j = lane; j < P.k; j += 32) {
            const uint32_t b = curand(&st) & 1u;
            if (P.info_out) P.info_out[f * P.k + j] = uint8_t(b);
            if (b) {
                const int pos = P.info_pos[j];
                atomicOr(row + (pos >> 5), 1u << (pos & 31));
                if (P.w) crc ^= P.col[j];
            }
        }
        if (P.w) {
            for (int off = 16; off >= 1; off >>= 1) {
                const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(crc), off);
                const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(crc >> 32), off);
                crc ^= (uint64_t(hi) << 32) | lo;
            }
            crc ^= P.c0;
            for (int j = lane; j < P.w; j += 32)
                if ((crc >> (P.w - 1 - j)) & 1) {
                    const int pos = P.info_pos[P.k + j];
                    atomicOr(row + (pos >> 5), 1u << (pos & 31));
                }
        }
        __syncwarp();
        // systematic encoding: x = T(mask(T(u))) (code.cpp:128-152)
        transform_row(row, P.n, P.rw, lane);
        // mask to the open positions: rebuild from info_pos bits of T(u)
        // (kept in place: clear frozen positions)
        __syncwarp();
        for (int j = lane; j < P.rw; j += 32) row[j] &= reinterpret_cast<const uint32_t*>(P.col + P.k)[j];
        __syncwarp();
        transform_row(row, P.n, P.rw, lane);
        for (int i = lane; i < P.n; i += 32) {
            const int ui = P.use ? P.use[i] : PL_USE_TRANSMITTED;
            if (ui != PL_USE_TRANSMITTED) {
                const bool sh = ui == PL_USE_SHORTENED;
                if (P.precision == PL_F32) static_cast<float*>(P.llr_out)[f * P.n + i] = sh ? 1e9f : 0.0f;
                else if (P.precision == PL_I8) static_cast<int8_t*>(P.llr_out)[f * P.n + i] = int8_t(sh ? 127 : 0);
                else static_cast<int16_t*>(P.llr_out)[f * P.n + i] = int16_t(sh ? 32767 : 0);
                continue;
            }
            const bool x = (row[i >> 5] >> (i & 31)) & 1u;
            const float y = (x ? -1.0f : 1.0f) + P.sigma * curand_normal(&st);
            const float v = P.demap * y;
            if (P.precision == PL_F32) {
                static_cast<float*>(P.llr_out)[f * P.n + i] = v;
            } else if (P.precision == PL_I8) {
                const float q = fminf(fmaxf(roundf(v * P.qs), -127.0f), 127.0f);
                static_cast<int8_t*>(P.llr_out)[f * P.n + i] = int8_t(q);
            } else {
                const float q = fminf(fmaxf(roundf(v * P.qs), -32767.0f), 32767.0f);
                static_cast<int16_t*>(P.llr_out)[f * P.n + i] = int16_t(q);
            }
        }
        __syncwarp();
    }
}

} // namespace
} // namespace plb

extern "C" int pl_channel_generate_device(const pl_code* code, double ebn0_db, uint64_t seed,
                                          uint64_t frame0, int64_t nframes, int32_t precision,
                                          float scale, uint8_t* info_out, void* llr_out,
                                          void* stream) {
    using namespace plb;
    if (!code || !code->frozen || !llr_out || nframes < 0 || !pow2(code->n) || code->k < 1)
        return PL_ERR_ARG;
    if (precision != PL_F32 && precision != PL_I8 && precision != PL_I16) return PL_ERR_CONFIG;
    if (nframes == 0) return PL_OK;
    const int n = code->n, k = code->k, w = code->crc.width;
    std::vector<int32_t> info_pos;
    for (int i = 0; i < n; ++i)
        if (!code->frozen[i]) info_pos.push_back(i);
    if (int(info_pos.size()) != k + w) return PL_ERR_CONFIG;
    const int rw = n >= 32 ? n / 32 : 1;
    // table: k CRC columns, then the open-position mask as rw u32 words
    std::vector<uint64_t> tab(size_t(k) + size_t(rw + 1) / 2, 0);
    uint64_t c0 = 0;
    if (w) {
        std::vector<uint8_t> msg(static_cast<size_t>(k), 0);
        if (pl_crc_compute(&code->crc, msg.data(), k, &c0) != PL_OK) return PL_ERR_CONFIG;
        for (int j = 0; j < k; ++j) {
            msg[size_t(j)] = 1;
            uint64_t v = 0;
            pl_crc_compute(&code->crc, msg.data(), k, &v);
            tab[size_t(j)] = v ^ c0;
            msg[size_t(j)] = 0;
        }
    }
    uint32_t* amask = reinterpret_cast<uint32_t*>(tab.data() + k);
    for (int p : info_pos) amask[p >> 5] |= 1u << (p & 31);
    const uint8_t* use = code->channel_use;
    int transmitted = n;
    if (use) {
        transmitted = 0;
        for (int i = 0; i < n; ++i) {
            if (use[i] > PL_USE_SHORTENED) return PL_ERR_CONFIG;
            transmitted += use[i] == PL_USE_TRANSMITTED;
        }
        if (transmitted < k + w) return PL_ERR_CONFIG;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t* d_pos = nullptr;
    uint64_t* d_tab = nullptr;
    uint8_t* d_use = nullptr;
    if (use) {
        if (cudaMallocAsync(&d_use, size_t(n), s) != cudaSuccess) return PL_ERR_CUDA;
        cudaMemcpyAsync(d_use, use, size_t(n), cudaMemcpyHostToDevice, s);
    }
    if (cudaMallocAsync(&d_pos, info_pos.size() * 4, s) != cudaSuccess) return PL_ERR_CUDA;
    if (cudaMallocAsync(&d_tab, tab.size() * 8, s) != cudaSuccess) return PL_ERR_CUDA;
    cudaMemcpyAsync(d_pos, info_pos.data(), info_pos.size() * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s);
    ChanParams P{};
    P.n = n;
    P.k = k;
    P.w = w;
    P.rw = rw;
    P.info_pos = d_pos;
    P.use = d_use;
    P.col = d_tab;
    P.c0 = c0;
    const double sigma2 = 1.0 / (2.0 * (double(k) / transmitted) * std::pow(10.0, ebn0_db / 10.0));
    P.sigma = float(std::sqrt(sigma2));
    P.demap = float(2.0 / sigma2);
    P.qs = scale > 0 ? scale : (precision == PL_I8 ? 8.0f : precision == PL_I16 ? 64.0f : 1.0f);
    P.precision = precision;
    P.seed = seed;
    P.frame0 = frame0;
    P.nframes = nframes;
    P.info_out = info_out;
    P.llr_out = llr_out;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int wpb = 8;
    const int64_t blocks = std::min<int64_t>((nframes + wpb - 1) / wpb, int64_t(sms) * 8);
    chan_kernel<<<int(blocks), wpb * 32, size_t(wpb) * rw * 4, s>>>(P);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(d_pos, s);
    cudaFreeAsync(d_tab, s);
    if (d_use) cudaFreeAsync(d_use, s);
    return e == cudaSuccess ? PL_OK : PL_ERR_CUDA;
}
