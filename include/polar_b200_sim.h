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

#ifdef __cplusplus
}
#endif
#endif
