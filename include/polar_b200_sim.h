/* polar_b200_sim.h — input-side helpers around the decoder (harness, not
 * the hot path): frozen-set construction and the BPSK/AWGN channel.
 *
 *   reference                                       here
 *   ----------------------------------------------- -------------------------
 *   construct_frozen (Bhattacharyya)  code.cpp:33-77 pl_construct_frozen_bhat
 *   (missing: Gaussian approximation)   pl_construct_frozen_ga
 *   run_frame inputs: FrameRng, random_payload,     pl_channel_generate
 *     encode_systematic, transmit                    (host threads) and
 *     (sim.cpp:45-51, channel.hpp:17-89,             pl_channel_generate_device
 *      code.cpp:12-31, 128-152)                      (sm_100a kernel)
 */
#ifndef POLAR_B200_SIM_H
#define POLAR_B200_SIM_H

#include <stdint.h>

#include "polar_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Bhattacharyya construction, identical ordering to construct_frozen. */
int pl_construct_frozen_bhat(int32_t n, int32_t reliable, double design_erasure,
                             uint8_t* frozen_out);

/* Gaussian-approximation construction (Trifonov) for BPSK/AWGN at a design
 * Eb/N0 and code rate; the n - reliable least reliable positions (ties to
 * the lower index) are frozen. */
int pl_construct_frozen_ga(int32_t n, int32_t reliable, double design_ebn0_db, double rate,
                           uint8_t* frozen_out);

/* Host channel, frame-keyed exactly like FrameRng(seed, frame): MT19937
 * seeded with (s ^ s>>32), s = seed ^ frame; info bits from coin(); systematic
 * encoding with the CRC appended MSB-first; BPSK over AWGN, LLR = 2y/sigma^2,
 * sigma^2 = 1/(2 (k/n) 10^(EbN0/10)); int8 LLRs quantised as
 * round-half-away(x * scale) clamped to +-127.
 *   info_out  k bytes (0/1) per frame, nullable
 *   llr_out   n values per frame (float or int8), host memory */
int pl_channel_generate(const pl_code* code, double ebn0_db, uint64_t seed, uint64_t frame0,
                        int64_t nframes, int32_t precision, float scale, uint8_t* info_out,
                        void* llr_out, int32_t nthreads);

/* Same for an explicit list of global frame indices (mixed-code batches:
 * the frames of one code are scattered through the batch).  Frame i of the
 * output is keyed by frame_ids[i]; llr_stride / info_stride are the output
 * row strides (values / bytes), so rows can land in a wider batch. */
int pl_channel_generate_frames(const pl_code* code, double ebn0_db, uint64_t seed,
                               const uint64_t* frame_ids, int64_t nframes, int32_t precision,
                               float scale, uint8_t* info_out, int64_t info_stride,
                               void* llr_out, int64_t llr_stride, int32_t nthreads);

/* Device channel for large Monte-Carlo runs: statistically equivalent
 * (Philox4x32-10 keyed by (seed, frame), Box-Muller), NOT bit-identical to
 * the host generator.  info_out (k bytes per frame, nullable) and llr_out
 * (n values per frame) are device pointers.  Asynchronous on `stream`. */
int pl_channel_generate_device(const pl_code* code, double ebn0_db, uint64_t seed,
                               uint64_t frame0, int64_t nframes, int32_t precision,
                               float scale, uint8_t* info_out, void* llr_out, void* stream);

/* ---- Monte-Carlo point (run_point, sim.cpp:76-135; SimConfig sim.hpp:14-29,
 * PointStats sim.hpp:31-42).  Frames [frame0, frame0 + max_frames) keyed by
 * (seed, global frame index) are generated, decoded with the handle's
 * decoder and compared with their information bits on the device (an
 * error-count kernel after each decode); the stop rule is evaluated at the
 * reference's 1024-frame batch boundaries, so with the host channel the
 * counts equal run_montecarlo's exactly, for any chunking.  frame0 lets
 * ranks of a multi-GPU run take disjoint frame ranges (sum the counts). */
enum { PL_CHANNEL_HOST = 0, PL_CHANNEL_DEVICE = 1 };

typedef struct pl_sim_config {
    double ebn0_db;
    uint64_t seed;         /* sim.hpp:27 default 42 */
    uint64_t frame0;       /* first global frame index of this run */
    uint64_t max_frames;   /* 0 = unbounded (needs max_fe) */
    uint64_t max_fe;       /* 0 = run to max_frames */
    float quant_scale;     /* 0 = per-precision default (channel.hpp:94-100) */
    int32_t channel;       /* PL_CHANNEL_HOST (FrameRng-exact) or PL_CHANNEL_DEVICE */
    int32_t host_threads;  /* host channel generator threads (0 = all cores) */
    int32_t pad;
    int64_t chunk_frames;  /* frames per device batch, rounded up to 1024 (0 = auto) */
} pl_sim_config;

typedef struct pl_point_stats {
    double ebn0_db;
    uint64_t frames, bit_errors, frame_errors, esc_sum;
    double ber, fer;
    double ti_mbps;      /* info bits over summed decode-kernel time (GPU throughput) */
    double lat_avg_us;   /* mean per-frame decode time on the device (pl_frame_latency:
                            from the start of a frame's decode to its final output,
                            summed over its passes), as run_frame times decode() */
    double lat_worst_us; /* largest per-frame decode time */
    double esc_mean;
} pl_point_stats;

/* One Eb/N0 point.  `code` must be the handle's (single) code. */
int pl_sim_point(pl_handle* h, const pl_code* code, const pl_sim_config* cfg,
                 pl_point_stats* out);
/* The reference's CSV data row (format_csv_row, report.cpp:40-50), no newline;
 * returns the row length (the row is truncated to len - 1 bytes). */
int32_t pl_format_csv_row(const pl_point_stats* p, char* buf, int32_t len);

#ifdef __cplusplus
}
#endif
#endif
