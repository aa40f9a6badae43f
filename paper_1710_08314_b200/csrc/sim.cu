// Monte-Carlo point driver around the decoder: the
// reference's run_point (sim.cpp:76-135) on the GPU.  Per device batch:
// channel (device Philox or the FrameRng-exact host generator + one H2D
// copy), pl_decode, then an error-count kernel that compares each decoded
// payload with the frame's information bits and accumulates per 1024-frame
// batch (the reference's batch_size, sim.cpp:18): bit errors, frame errors
// and escalation sum.  The host walks those batch records in order and
// applies the stop rule at the same boundaries as the reference, so which
// frames contribute does not depend on the device chunking.
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/polar_b200.h"
#include "../../include/polar_b200_sim.h"

namespace {

constexpr int64_t kBatch = 1024; // sim.cpp:18

// One warp per frame: payload bits [0, k) (MSB-first bytes) against the
// frame's k information bytes (0/1); per-batch sums by atomics.
__global__ void count_errors_kernel(const uint8_t* payload, int64_t pstride, const uint8_t* info,
                                    int k, const uint8_t* esc, int64_t nframes,
                                    unsigned long long* batch_be, unsigned int* batch_fe,
                                    unsigned long long* batch_esc, const uint32_t* lat,
                                    unsigned long long* batch_lsum, unsigned int* batch_lmax) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t f = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); f < nframes;
         f += warps) {
        const uint8_t* pay = payload + f * pstride;
        const uint8_t* inf = info + f * int64_t(k);
        unsigned be = 0;
        for (int q = lane; q < (k + 7) >> 3; q += 32) {
            uint32_t ib = 0, valid = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int i = 8 * q + b;
                if (i < k) {
                    ib |= uint32_t(inf[i] & 1u) << (7 - b);
                    valid |= 1u << (7 - b);
                }
            }
            be += __popc((uint32_t(pay[q]) ^ ib) & valid);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) be += __shfl_xor_sync(0xffffffffu, be, o);
        if (lane == 0) {
            const int64_t b = f / kBatch;
            if (be) {
                atomicAdd(batch_be + b, (unsigned long long)be);
                atomicAdd(batch_fe + b, 1u);
            }
            atomicAdd(batch_esc + b, (unsigned long long)(esc ? esc[f] : 1));
            if (lat) {
                atomicAdd(batch_lsum + b, (unsigned long long)lat[f]);
                atomicMax(batch_lmax + b, lat[f]);
            }
        }
    }
}

// grow-only buffers, kept across points (a sweep reuses them: allocating
// GBs per point cost more than the point's decode)
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* get() const {
        return static_cast<T*>(p);
    }
    cudaError_t alloc(size_t bytes) {
        bytes = std::max<size_t>(bytes, 16);
        if (cap >= bytes) return cudaSuccess;
        release();
        const cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        else p = nullptr;
        return e;
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~HostBuf() { release(); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    cudaError_t alloc(size_t bytes) {
        bytes = std::max<size_t>(bytes, 16);
        if (cap >= bytes) return cudaSuccess;
        release();
        const cudaError_t e = cudaMallocHost(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        else p = nullptr;
        return e;
    }
};

struct SimBuffers {
    int device = -1;
    DevBuf d_llr, d_info, d_pay, d_esc, d_be, d_fe, d_es, d_lat, d_ls, d_lm;
    HostBuf h_llr, h_info;
    void reset() {
        for (DevBuf* b : {&d_llr, &d_info, &d_pay, &d_esc, &d_be, &d_fe, &d_es, &d_lat, &d_ls, &d_lm})
            b->release();
        h_llr.release();
        h_info.release();
    }
};
thread_local SimBuffers g_buf;

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};


} // namespace

extern "C" {

int pl_sim_point(pl_handle* h, const pl_code* code, const pl_sim_config* cfg, pl_point_stats* out) {
    if (!h || !code || !cfg || !out) return PL_ERR_ARG;
    // run_montecarlo's checks (sim.cpp:150-158)
    if (cfg->max_frames == 0 && cfg->max_fe == 0) return PL_ERR_CONFIG;
    const int32_t k = code->k;
    const int64_t n = code->n;
    const int64_t pstride = pl_payload_stride(h);
    if (pl_llr_stride(h) != n) return PL_ERR_ARG; // the handle's own (single) code
    const int32_t prec = pl_precision(h);
    const int64_t esz = prec == PL_I8 ? 1 : prec == PL_I16 ? 2 : 4;
    const uint64_t max_frames = cfg->max_frames ? cfg->max_frames : ~0ull;
    int64_t chunk = cfg->chunk_frames > 0 ? cfg->chunk_frames : (int64_t(1) << 18);
    chunk = (chunk + kBatch - 1) / kBatch * kBatch;
    if (cfg->max_frames) chunk = std::min<int64_t>(chunk, int64_t((cfg->max_frames + kBatch - 1) / kBatch * kBatch));
    const int64_t nb = chunk / kBatch;

    int dev = 0;
    cudaGetDevice(&dev);
    if (g_buf.device != dev) {
        g_buf.reset();
        g_buf.device = dev;
    }
    DevBuf &d_llr = g_buf.d_llr, &d_info = g_buf.d_info, &d_pay = g_buf.d_pay, &d_esc = g_buf.d_esc;
    DevBuf &d_be = g_buf.d_be, &d_fe = g_buf.d_fe, &d_es = g_buf.d_es;
    DevBuf &d_lat = g_buf.d_lat, &d_ls = g_buf.d_ls, &d_lm = g_buf.d_lm;
    HostBuf &h_llr = g_buf.h_llr, &h_info = g_buf.h_info;
    cudaStream_t s = nullptr;
    EventPair ev;
    std::vector<unsigned long long> be(static_cast<size_t>(nb)), es(static_cast<size_t>(nb));
    std::vector<unsigned int> fe(static_cast<size_t>(nb)), lm(static_cast<size_t>(nb));
    std::vector<unsigned long long> ls(static_cast<size_t>(nb));
    auto ck = [](cudaError_t e) { return e == cudaSuccess; };
    if (!ck(d_llr.alloc(size_t(chunk * n * esz))) || !ck(d_info.alloc(size_t(chunk * k))) ||
        !ck(d_pay.alloc(size_t(chunk * pstride))) || !ck(d_esc.alloc(size_t(chunk))) ||
        !ck(d_be.alloc(size_t(nb) * 8)) || !ck(d_fe.alloc(size_t(nb) * 4)) ||
        !ck(d_es.alloc(size_t(nb) * 8)) || !ck(d_lat.alloc(size_t(chunk) * 4)) ||
        !ck(d_ls.alloc(size_t(nb) * 8)) || !ck(d_lm.alloc(size_t(nb) * 4)) ||
        !ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) ||
        !ck(cudaEventCreate(&ev.a)) || !ck(cudaEventCreate(&ev.b))) {
        if (s) cudaStreamDestroy(s);
        return PL_ERR_CUDA;
    }
    if (cfg->channel == PL_CHANNEL_HOST &&
        (!ck(h_llr.alloc(size_t(chunk * n * esz))) || !ck(h_info.alloc(size_t(chunk * k))))) {
        cudaStreamDestroy(s);
        return PL_ERR_CUDA;
    }

    uint64_t done = 0, decoded = 0, tot_be = 0, tot_fe = 0, tot_es = 0, lat_sum = 0;
    uint32_t lat_worst = 0;
    double dec_us = 0;
    // per-frame decode time (pl_frame_latency) over the frames that count
    pl_frame_latency(h, d_lat.get<uint32_t>());
    int rc = PL_OK;
    bool stop = false;
    while (!stop && done < max_frames) {
        const int64_t nf = int64_t(std::min<uint64_t>(uint64_t(chunk), max_frames - done));
        const uint64_t f0 = cfg->frame0 + done;
        if (cfg->channel == PL_CHANNEL_HOST) {
            rc = pl_channel_generate(code, cfg->ebn0_db, cfg->seed, f0, nf, prec, cfg->quant_scale,
                                     static_cast<uint8_t*>(h_info.p), h_llr.p, cfg->host_threads);
            if (rc != PL_OK) break;
            if (!ck(cudaMemcpyAsync(d_llr.p, h_llr.p, size_t(nf * n * esz), cudaMemcpyHostToDevice, s)) ||
                !ck(cudaMemcpyAsync(d_info.p, h_info.p, size_t(nf * k), cudaMemcpyHostToDevice, s))) {
                rc = PL_ERR_CUDA;
                break;
            }
        } else {
            rc = pl_channel_generate_device(code, cfg->ebn0_db, cfg->seed, f0, nf, prec, cfg->quant_scale,
                                            d_info.get<uint8_t>(), d_llr.p, s);
            if (rc != PL_OK) break;
        }
        const int64_t nbc = (nf + kBatch - 1) / kBatch;
        cudaMemsetAsync(d_be.p, 0, size_t(nbc) * 8, s);
        cudaMemsetAsync(d_fe.p, 0, size_t(nbc) * 4, s);
        cudaMemsetAsync(d_es.p, 0, size_t(nbc) * 8, s);
        cudaMemsetAsync(d_ls.p, 0, size_t(nbc) * 8, s);
        cudaMemsetAsync(d_lm.p, 0, size_t(nbc) * 4, s);
        cudaEventRecord(ev.a, s);
        rc = pl_decode(h, d_llr.p, nullptr, nf, d_pay.get<uint8_t>(), nullptr, nullptr,
                       d_esc.get<uint8_t>(), nullptr, s);
        if (rc != PL_OK) break;
        cudaEventRecord(ev.b, s);
        count_errors_kernel<<<1184, 256, 0, s>>>(d_pay.get<uint8_t>(), pstride, d_info.get<uint8_t>(), k,
                                                  d_esc.get<uint8_t>(), nf, d_be.get<unsigned long long>(),
                                                  d_fe.get<unsigned int>(), d_es.get<unsigned long long>(),
                                                  d_lat.get<uint32_t>(), d_ls.get<unsigned long long>(),
                                                  d_lm.get<unsigned int>());
        if (!ck(cudaGetLastError()) ||
            !ck(cudaMemcpyAsync(be.data(), d_be.p, size_t(nbc) * 8, cudaMemcpyDeviceToHost, s)) ||
            !ck(cudaMemcpyAsync(fe.data(), d_fe.p, size_t(nbc) * 4, cudaMemcpyDeviceToHost, s)) ||
            !ck(cudaMemcpyAsync(es.data(), d_es.p, size_t(nbc) * 8, cudaMemcpyDeviceToHost, s)) ||
            !ck(cudaMemcpyAsync(ls.data(), d_ls.p, size_t(nbc) * 8, cudaMemcpyDeviceToHost, s)) ||
            !ck(cudaMemcpyAsync(lm.data(), d_lm.p, size_t(nbc) * 4, cudaMemcpyDeviceToHost, s)) ||
            !ck(cudaStreamSynchronize(s))) {
            rc = PL_ERR_CUDA;
            break;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev.a, ev.b);
        dec_us += 1e3 * double(ms);
        decoded += uint64_t(nf);
        // the reference's batch loop (sim.cpp:91-115), one 1024-frame batch
        // at a time
        for (int64_t b = 0; b < nbc; ++b) {
            const int64_t bf = std::min<int64_t>(kBatch, nf - b * kBatch);
            tot_be += be[size_t(b)];
            tot_fe += fe[size_t(b)];
            tot_es += es[size_t(b)];
            lat_sum += ls[size_t(b)];
            lat_worst = std::max(lat_worst, lm[size_t(b)]);
            done += uint64_t(bf);
            if (cfg->max_fe && tot_fe >= cfg->max_fe) {
                stop = true;
                break;
            }
        }
    }
    pl_frame_latency(h, nullptr);
    cudaStreamDestroy(s);
    if (rc != PL_OK) return rc;

    pl_point_stats p{};
    p.ebn0_db = cfg->ebn0_db;
    p.frames = done;
    p.bit_errors = tot_be;
    p.frame_errors = tot_fe;
    p.esc_sum = tot_es;
    const double kf = double(k) * double(done);
    p.ber = done ? double(tot_be) / kf : 0;
    p.fer = done ? double(tot_fe) / double(done) : 0;
    p.esc_mean = done ? double(tot_es) / double(done) : 0;
    if (dec_us > 0) {
        p.ti_mbps = double(k) * double(decoded) / dec_us; // bits per µs = Mb/s
    }
    if (done) {
        // per frame, as run_frame times each decode() (sim.cpp:54-61, 131-134)
        p.lat_avg_us = double(lat_sum) * 1e-3 / double(done);
        p.lat_worst_us = double(lat_worst) * 1e-3;
    }
    *out = p;
    return PL_OK;
}

int32_t pl_format_csv_row(const pl_point_stats* p, char* buf, int32_t len) {
    if (!p) return -1;
    // report.cpp:19-33 cell formats
    char row[512];
    const int w = std::snprintf(row, sizeof row, "%.6g,%" PRIu64 ",%" PRIu64 ",%" PRIu64
                                ",%.6e,%.6e,%.3f,%.3f,%.3f,%.4f",
                                p->ebn0_db, p->frames, p->bit_errors, p->frame_errors, p->ber, p->fer,
                                p->ti_mbps, p->lat_avg_us, p->lat_worst_us, p->esc_mean);
    if (buf && len > 0) std::snprintf(buf, size_t(len), "%s", row);
    return int32_t(w);
}

} // extern "C"
