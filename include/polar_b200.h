/* polar_b200.h — C ABI of the B200-native batched polar decoder.
 *
 * Drop-in for the reference's decoder API (a header-only C++ template
 * interface, no FFI of its own):
 *
 *   reference                                              here
 *   ------------------------------------------------------ -------------------
 *   make_code(n, k, frozen, crc)  code.hpp:43-45,          pl_code (validated
 *                                 code.cpp:79-126           in pl_create)
 *   CrcSpec / CrcSpec::parse      crc.hpp:16-26,            pl_crc, pl_crc_parse
 *                                 crc.cpp:42-84
 *   PruningConfig                 prune_tree.hpp:25-34      pl_pruning
 *   PruneTree(frozen, cfg)        prune_tree.hpp:49-73,     built inside
 *                                 sim.cpp:161-164            pl_create; exported
 *                                                            for tests: pl_tree_build
 *   DecoderKind                   decoders.hpp:10-18        PL_KIND_*
 *   FrameDecoder<R>(code, tree,   decoders.hpp:37-55        pl_create
 *                   kind, l)
 *   FrameDecoder<R>::decode(R*)   decoders.hpp:60-85        pl_decode (a batch of
 *     -> DecodeResult             decode_result.hpp:7-14     frames per call)
 *   ConfigError / ParseError      errors.hpp:9-21           PL_ERR_CONFIG /
 *                                                            PL_ERR_PARSE +
 *                                                            pl_last_error
 *   CrcEngine::compute            crc.cpp:121-144           pl_crc_compute
 *
 * Plain pointers and sizes only.  Device pointers are CUDA global-memory
 * pointers; `stream` is a cudaStream_t passed as void*.  A handle is not
 * thread-safe (the reference's FrameDecoder is not either);
 * use one handle per host thread.  Calls on one handle may use different
 * streams: each decode waits (cudaStreamWaitEvent) for the previous decode
 * that used the same scratch, so they serialise on the device instead of
 * racing.  Decodes that should overlap need one handle each.  A fully
 * adaptive decode may run the last rungs of its ladder on two internal
 * streams of the handle (forked from and joined back into `stream` with
 * events), so work queued on `stream` after the call still sees complete
 * outputs.  There is no CPU fallback: every decode runs the sm_100a kernels
 * or fails with PL_ERR_CUDA.
 */
#ifndef POLAR_B200_H
#define POLAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the C face of the reference's exceptions) */
#define PL_OK 0
#define PL_ERR_CONFIG 1 /* ConfigError: bad code / decoder / tree parameters */
#define PL_ERR_PARSE 2  /* ParseError: malformed CRC spec text */
#define PL_ERR_CUDA 3   /* device failure (no GPU, launch error, OOM) */
#define PL_ERR_ARG 4    /* null pointer / bad size passed to the ABI */
#define PL_ERR_IO 5     /* IoError: filesystem failure (errors.hpp:19-21) */

/* DecoderKind, decoders.hpp:10-18 — same order */
#define PL_KIND_SC 0
#define PL_KIND_SSC 1
#define PL_KIND_SCL 2
#define PL_KIND_SSCL 3
#define PL_KIND_CA_SSCL 4
#define PL_KIND_PA_SSCL 5
#define PL_KIND_FA_SSCL 6

/* LLR representation (llr.hpp:12-33): float32, int8 saturated to +-127 or
 * int16 saturated to +-32767 */
#define PL_F32 0
#define PL_I8 1
#define PL_I16 2

typedef struct pl_crc {
    int32_t width; /* 0 = code without CRC; else 1..64 */
    int32_t reflect;
    uint64_t poly; /* normal form without the top bit (crc.hpp:16-20) */
    uint64_t init;
    uint64_t xorout;
} pl_crc;

typedef struct pl_code {
    int32_t n;             /* block length, power of two, 2..32768 */
    int32_t k;             /* information bits, CRC excluded (code.hpp:31) */
    const uint8_t* frozen; /* n bytes, nonzero = frozen; host memory */
    pl_crc crc;
    /* PuncturePattern (code.hpp:13-24): n bytes, PL_USE_*; NULL = every
     * position transmitted.  Only the channel side reads it (rate, demap);
     * the decoders take whatever LLRs arrive. */
    const uint8_t* channel_use;
} pl_code;

#define PL_USE_TRANSMITTED 0
#define PL_USE_PUNCTURED 1 /* never sent: LLR 0 */
#define PL_USE_SHORTENED 2 /* known zero: the largest LLR (llr.hpp:105-111) */

typedef struct pl_pruning { /* PruningConfig, prune_tree.hpp:25-34 */
    int32_t rate_zero, rate_one, repetition, single_parity;
    int32_t rep_max; /* 0 = unlimited, else >= 2 */
    int32_t spc_max; /* 0 = unlimited, else >= 4 */
} pl_pruning;

typedef struct pl_decoder {
    int32_t kind;      /* PL_KIND_* */
    int32_t l;         /* list size (Lmax for PA/FA); power of two <= 32 */
    int32_t precision; /* PL_F32 / PL_I8 / PL_I16 */
    pl_pruning pruning;
} pl_decoder;

typedef struct pl_handle pl_handle;

/* Build a decoder for one or more codes (mixed-code batches select a code
 * per frame).  Validates exactly what make_code, PruneTree and FrameDecoder
 * validate and returns PL_ERR_CONFIG where they throw ConfigError.  The
 * handle owns copies of all code data and its device tables. */
int pl_create(const pl_code* codes, int32_t ncodes, const pl_decoder* dec,
              int32_t device, pl_handle** out);

/* Message of the last failure on this handle ("" if none).  With a NULL
 * handle: the last pl_create / pl_crc_parse failure of the calling thread. */
const char* pl_last_error(const pl_handle* h);

void pl_destroy(pl_handle* h);

/* Strides of the batch buffers (elements for LLRs, bytes for the rest). */
int64_t pl_llr_stride(const pl_handle* h);      /* max n over codes */
int64_t pl_payload_stride(const pl_handle* h);  /* max ceil((k+c)/8) */
int64_t pl_codeword_stride(const pl_handle* h); /* max ceil(n/8) */
int32_t pl_precision(const pl_handle* h);       /* PL_F32 / PL_I8 / PL_I16, -1 for NULL */

/* Decode nframes frames resident in device memory.
 *   llr      frame-major, pl_llr_stride elements per frame (float or int8)
 *   code_id  per-frame code index, NULL = code 0 for every frame
 *   payload  pl_payload_stride bytes per frame: the payload (message + CRC)
 *            packed MSB-first, DecodeResult::payload (decode_result.hpp:9)
 *   codeword optional (NULL), pl_codeword_stride bytes per frame, MSB-first
 *   crc_ok   1 byte per frame (optional)
 *   esc      escalation level per frame: the list size that produced the
 *            answer, 1 = SC (optional)
 *   metric   path metric of the returned candidate, float (optional)
 * Asynchronous on `stream`. */
int pl_decode(pl_handle* h, const void* llr, const int32_t* code_id, int64_t nframes,
              uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc,
              float* metric, void* stream);

/* Same with HOST buffers: the call stages through pinned memory, overlaps
 * host<->device copies with decoding in chunks and returns when the outputs
 * are in host memory. */
int pl_decode_host(pl_handle* h, const void* llr, const int32_t* code_id,
                   int64_t nframes, uint8_t* payload, uint8_t* codeword,
                   uint8_t* crc_ok, uint8_t* esc, float* metric);

/* Packed variable-length frames (mixed-code batches without padding every
 * frame to pl_llr_stride): frame i's n LLRs start at element llr_offset[i]
 * of llr.  Offsets ascending, frames not overlapping, every frame 16-byte
 * aligned (offset * sizeof(R) % 16 == 0); PL_ERR_ARG otherwise (host call).
 * The reference decodes each frame from its own buffer of n LLRs
 * (FrameDecoder<R>::decode(const R*), decoders.hpp:60): this is that
 * layout for a batch.
 *   pl_decode_packed       device buffers (llr, llr_offset), async on stream
 *   pl_decode_host_packed  host buffers; only each frame's n LLRs cross the
 *                          host link */
int pl_decode_packed(pl_handle* h, const void* llr, const int64_t* llr_offset,
                     const int32_t* code_id, int64_t nframes, uint8_t* payload,
                     uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc, float* metric,
                     void* stream);
int pl_decode_host_packed(pl_handle* h, const void* llr, const int64_t* llr_offset,
                          const int32_t* code_id, int64_t nframes, uint8_t* payload,
                          uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc, float* metric);

/* Kernel launches issued by the last pl_decode / pl_decode_host call. */
int64_t pl_last_launches(const pl_handle* h);

/* Per-frame decode latency (the reference's run_frame timing, sim.cpp:54-61:
 * lat_sum / lat_worst over decode() calls).  With a device buffer set,
 * every later pl_decode / pl_decode_packed on the handle writes lat_ns[f] =
 * device time (ns, %globaltimer) from the start of frame f's decode to its
 * final output, summed over the passes it runs through (SC, then each rung
 * of an adaptive ladder); NULL switches it off.  The buffer must hold one
 * uint32 per frame of each call. */
int pl_frame_latency(pl_handle* h, uint32_t* lat_ns);

/* The final list of each frame, as ListDecoder<R>::alive_count / is_alive /
 * metric_of expose it (list_decoder.hpp:91-93): with device buffers set, every
 * later pl_decode / pl_decode_packed writes alive[f] = alive-slot mask of
 * frame f's last list pass (bit s = logical slot s, the reference's slot
 * numbering) and metric[f * L + s] = the metric of slot s (L = the handle's
 * list size; dead slots hold stale values, as in the reference).  Passes
 * without a list (SC) leave them untouched; NULL, NULL switches it off. */
int pl_list_paths(pl_handle* h, uint32_t* alive, float* metric);

/* Frames per chunk of pl_decode_host / pl_decode_host_packed (copies of one
 * chunk overlap the decode of others); 0 = automatic (~20 chunks per call,
 * 16 for multi-code handles, 8 for adaptive int8).  Default at pl_create:
 * $PLB_HOST_CHUNK or 0. */
int pl_set_host_chunk(pl_handle* h, int64_t frames);

/* Input layout of pl_decode (device LLRs).  PL_LLR_FRAME_MAJOR (default):
 * frame f at llr + f * pl_llr_stride, the layout of FrameDecoder<R>::decode
 * (const R*) called frame after frame.  PL_LLR_INTERLEAVED32: frames in
 * groups of 32, 16-byte chunks interleaved -- chunk c (16 bytes of values;
 * n values when the frame is shorter) of frame f at chunk index
 * ((f / 32) * chunks_per_frame + c) * 32 + f % 32 -- so that the
 * frame-per-lane SC pass reads the channel with fully coalesced warp loads;
 * the buffer holds a whole number of groups (pad the last one).  Accepted
 * for PL_KIND_SC / PL_KIND_SSC handles with one code, pl_decode only
 * (PL_ERR_CONFIG otherwise): a producer-side option (a demapper that writes
 * LLRs for the GPU can emit this order), measured in DESIGN.md section 4. */
#define PL_LLR_FRAME_MAJOR 0
#define PL_LLR_INTERLEAVED32 1
int pl_set_llr_layout(pl_handle* h, int32_t layout);

/* Live kernel timing: with profiling enabled every launch of pl_decode is
 * bracketed by CUDA events on its stream; pl_last_kernel_ms waits for them
 * and writes the duration (ms) of each launch of the last pl_decode call and
 * its kind (0 = SC pass, 1 = list pass) and list size.  Returns the number
 * of launches written. */
int pl_profile(pl_handle* h, int32_t enable);

/* Device self-test of the packed int8 f/g kernels against their scalar
 * definitions (llr.hpp:55-69), every operand pair: writes the mismatch
 * count (0 expected). */
int pl_kernel_selftest(int32_t device, uint64_t* mismatches);
int32_t pl_last_kernel_ms(pl_handle* h, float* ms, int32_t* kind, int32_t* l, int32_t max);

/* ---- host-side helpers (no GPU needed) ---------------------------------- */

/* CrcSpec::parse (crc.cpp:42-84): "32-GZIP", "16-CCITT", "8" or
 * "width:poly:reflect:init:xorout" (hex fields). */
int pl_crc_parse(const char* text, pl_crc* out);

/* CrcEngine::compute over `len` bits given one per byte (crc.cpp:121-144). */
int pl_crc_compute(const pl_crc* spec, const uint8_t* bits, int64_t len,
                   uint64_t* out);

/* PruneTree node list (prune_tree.cpp:38-71), 6 ints per node:
 * kind, depth, leaf_begin, size, left, right.  Returns the node count, or
 * -1 (bad arguments / buffer too small). */
int32_t pl_tree_build(const uint8_t* frozen, int32_t n, const pl_pruning* cfg,
                      int32_t* out, int32_t max_nodes);

/* Frozen-set files (load_frozen_file / save_frozen_file, code.cpp:164-194):
 * "N K" then one line of N characters, '1' = frozen.  Load with
 * frozen_out = NULL to query n and k; errors are PL_ERR_PARSE / PL_ERR_IO
 * with the reference's messages (pl_last_error(NULL)). */
int pl_frozen_file_load(const char* path, int32_t* n, int32_t* k, uint8_t* frozen_out,
                        int32_t cap);
int pl_frozen_file_save(const char* path, int32_t n, int32_t k, const uint8_t* frozen);
/* Puncture files (load_puncture_file, code.cpp:196-221): "N" then N
 * characters T / P / S -> PL_USE_TRANSMITTED / _PUNCTURED / _SHORTENED. */
int pl_puncture_file_load(const char* path, int32_t* n, uint8_t* use_out, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* POLAR_B200_H */
