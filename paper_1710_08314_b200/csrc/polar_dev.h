// Internal interface between the host orchestration (host.cu) and the
// sm_100a kernels (kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace plb {

// ---- decode schedule --------------------------------------------------
// A decode tree (prune_tree.cpp:38-71) flattened into the order the
// reference's recursive walks visit it (list_decoder.hpp:174-224,
// sc_decoder.hpp:58-94): a branch node emits F, <left ops>, G, <right ops>,
// H; every other node emits one leaf op.  One op is a u32:
//   bits  0..3  op code
//   bits  4..7  depth d of the node (its LLRs live in depth-d segments)
//   bits  8..11 log2(size)
//   bits 12..27 leaf_begin
enum Op : uint32_t {
    OP_F = 0,      // child LLRs  <- f(left half, right half)
    OP_G = 1,      // child LLRs  <- g(left half, right half, left psums)
    OP_H = 2,      // psums[lb, lb+m/2) ^= psums[lb+m/2, lb+m)
    OP_FROZEN = 3, // frozen leaf or rate-0 node
    OP_INFO = 4,   // information leaf
    OP_R1 = 5,     // rate-1 node (list only; SC schedules expand it)
    OP_REP = 6,    // repetition node
    OP_SPC = 7,    // single-parity node (list only; SC schedules expand it)
    OP_SCSUB = 8,  // SC only: a whole subtree of size <= 32 decoded in one op by
                   // unabridged SC recursion; the next schedule word is its
                   // frozen mask (bit i = position lb+i frozen)
    OP_R1SC = 9,   // SC only: rate-1 node.  Next word = length of the expanded
                   // recursion that follows; when no input LLR is zero the
                   // recursion's result is the hard decision and it is skipped
    OP_GR1 = 10,   // lane schedules: a G op whose child is a rate-1 node.
                   // The g values are formed in registers; when none of them is
                   // zero (in any lane) their signs are the node's decisions and
                   // the next word's count of ops (the plain G op and the
                   // expanded recursion) is skipped; nothing is stored
};
constexpr int kScSubMax = 32;
// largest fused leaf (values held per lane): int8 / float
constexpr int kFuseMaxI8 = 8, kFuseMaxF32 = 4;

//   bit   28    (list schedules) fused leaf: the leaf's LLRs are not
//               materialised; the leaf op computes them in registers from
//               the parent segment (depth - 1) with F, or with G when
//   bit   29    is set (the F / G op of the parent is then omitted).  Leaves
//               of at most kFuseMax* values: fused_leaf; larger rate-1 /
//               single-parity right children (bit 29 set): r1spc_stats.
//               Lane schedules: the same two bits on an OP_SCSUB word
//               (lane_sub forms the subtree's LLRs from the parent's values)
constexpr uint32_t kOpFused = 1u << 28, kOpFusedG = 1u << 29;
//   bit   30    (list schedules) F / G op chained with the F op of its child:
//               both levels are computed in one sweep and stored, the child's
//               F op (dropped from the schedule) never reads its input back
constexpr uint32_t kOpChain = 1u << 30;
//   bits 28..29 (lane schedules) F / G: number of chained F ops this op
//               computes along with its own level (host.cu fuse_lane_chains)
constexpr int kOpChainShift = 28;
__host__ __device__ inline uint32_t op_pack(uint32_t op, int depth, int logm, int lb) {
    return op | (uint32_t(depth) << 4) | (uint32_t(logm) << 8) | (uint32_t(lb) << 12);
}
__host__ __device__ inline int op_code(uint32_t w) { return int(w & 15u); }
__host__ __device__ inline int op_depth(uint32_t w) { return int((w >> 4) & 15u); }
__host__ __device__ inline int op_logm(uint32_t w) { return int((w >> 8) & 15u); }
__host__ __device__ inline int op_lb(uint32_t w) { return int((w >> 12) & 0xffffu); }

// ---- per-code device tables -------------------------------------------
struct DevCode {
    int32_t n, stages, k, psize, crc_width, pad;
    const uint32_t* sched_list; // list-decoder schedule (pruned or full tree)
    const uint32_t* sched_sc;   // SC-rung schedule (R1/SPC expanded)
    const uint32_t* sched_lane; // the same without OP_SCSUB (frame-per-lane SC kernel)
    int32_t nops_list, nops_sc, nops_lane, pad2;
    // List-schedule variants (kernels.cu kSchedVariant picks one per kernel
    // instantiation): [0] = sched_list: big rate-1 / single-parity leaves
    // fused with their parent's G op; [1]: small fused leaves only; [2], [3]:
    // the same two with chained F ops (kOpChain, float).  Fixed point has
    // [0] and [1] ([2], [3] point at them).
    const uint32_t* sched_listv[4];
    int32_t nops_listv[4];
    // the same schedules decoded once on the host: {op word, depth, m, lb} per
    // op, one 16-byte load in the list kernels' op loop instead of the shifts
    // and masks of op_depth / op_logm / op_lb
    const uint4* sched_listx[4];
    const uint16_t* info_pos;   // psize open positions, ascending
    // CRC as an affine map over the decided codeword:
    // syndrome = crc_c0 ^ XOR_j crc_tab[j][byte_j(codeword)], zero <=> pass.
    const uint64_t* crc_tab;    // (n/8) x 256
    uint64_t crc_c0;
    // payload gather by codeword byte: open_mask[j] = the open positions
    // among 8j..8j+7 (bit i = position 8j+i); comp_tab[m * 256 + v] = the
    // bits of v selected by m in ascending position order, first one most
    // significant (a universal 64 KB table)
    const uint8_t* open_mask;   // ceil(n/8)
    const uint8_t* comp_tab;
};

// ---- launch parameters ------------------------------------------------
struct LaunchParams {
    const DevCode* codes;
    const void* llr;
    int64_t llr_stride;        // elements per frame
    const int64_t* llr_offset; // nullable: element offset of each frame (packed
                               // variable-length frames, pl_decode_packed)
    const int32_t* code_id;    // nullable
    const int32_t* frame_list; // nullable: frames [0, nframes) in order
    const int32_t* frame_count;// device count for frame_list (nullable)
    int64_t nframes;           // used when frame_list == nullptr
    unsigned long long* work;  // work-claim counter (zeroed before launch)
    int32_t* fail_list;        // nullable: CRC-failed frames appended here
    int32_t* fail_count;
    uint8_t* payload;
    int64_t payload_stride;
    uint8_t* codeword;         // nullable
    int64_t codeword_stride;
    uint8_t* crc_ok;           // nullable
    uint8_t* esc;              // nullable
    float* metric;             // nullable
    void* gscratch;            // global spill for the large LLR segments
    int64_t gscratch_per_frame;// bytes per in-flight frame
    int32_t l;                 // list size of this pass (1 for SC)
    int32_t select_by_crc;
    int32_t seg_smem_max;      // segments with more elements live in gscratch
    int32_t nmax;              // largest n over the codes
    int32_t smem_per_warp;     // bytes (= fpw * smem_per_frame)
    int32_t smem_per_frame;    // bytes
    int32_t esc_level;         // value written to esc[] by this pass
    int32_t wpb;               // warps per block (1, 2 or 4)
    int32_t fpw;               // frames per warp (1, 2 or 4; >1 needs one code)
    int32_t team;              // >1: each block is a team of `team` warps decoding
                               // one frame (list passes, 32-lane kernels)
    int64_t count_lo, count_hi;// the launch decodes only if count_lo < frames <= count_hi
                               // (two launches with complementary ranges pick a
                               // plan on the device from the pass's frame count)
    int32_t seg_solo;          // >0: solo mode when the pass has <= solo_max frames:
    int32_t solo_max;          // warp 0 of each block decodes with the whole block's
                               // shared memory (segments <= seg_solo in smem)
    int32_t sc_keep;           // frame-per-lane SC pass: global depth segments of <= sc_keep
                               // values are loaded / stored L2::evict_last, larger ones
                               // (and the channel) evict_first; 0 = no cache hints
    int32_t sc_keep_hi;        // ... segments of <= sc_keep_hi values (> sc_keep) evict_normal
    int32_t sc_discard;        // frame-per-lane SC pass: discard.global.L2 the lines of a
                               // global depth segment after its last read (G op)
    int32_t list_discard;      // float list passes: the same for a frame's global depth
                               // pool after a G op
    uint32_t* lat_ns;          // nullable: per-frame device decode time, ns, summed over
                               // the passes the frame runs through (pl_frame_latency)
    uint32_t* path_alive;      // nullable (pl_list_paths): alive-slot mask of the final list
    float* path_metric;        // ... and the metric of every slot, path_stride per frame
    int32_t path_stride;
    int32_t sc_tr;             // frame-per-lane SC pass: the ops on a frame-major channel read it
                               // in coalesced tiles transposed through shared memory
    int32_t llr_il32;          // frame-per-lane SC pass: the channel is interleaved in groups
                               // of 32 frames (PL_LLR_INTERLEAVED32), one code, no frame list
    int32_t list_alt;          // float sub-warp list kernels: the instantiation with big fused
                               // leaves instead of chained F ops (codes of N <= 1024)
    int32_t out_by_idx;        // list passes at one frame per warp / team: outputs are indexed
                               // by the frame's position in frame_list (staging of a
                               // speculative FA rung), not by the frame id
};

constexpr int kMaxWarpsPerBlock = 4; // a block is 1, 2 or 4 independent warps
constexpr int kMaxTeam = 8;          // ... or a team of up to 8 warps on one frame

// Bytes of shared memory / global scratch one in-flight frame needs.
// sw: lanes per frame of the kernel (32 / frames per warp; team and SC kernels 32)
int64_t smem_bytes_per_frame(int nmax, int l, int elem_bytes, int seg_smem_max, int sw);
int64_t gscratch_bytes_per_frame(int nmax, int l, int elem_bytes, int seg_smem_max);
// Frames per warp of the sub-warp kernel of list size l (a list pass runs
// either that many or 1).
int frames_per_warp_max(int l);
bool frames_per_warp_ok(int l, int fpw); // a kernel exists for (l, fpw)

// Kernel launchers (kernels.cu).  Return cudaError_t of the launch.
cudaError_t launch_sc(const LaunchParams& p, int precision, int grid, cudaStream_t s);
cudaError_t launch_list(const LaunchParams& p, int precision, int grid, cudaStream_t s);
// Max resident blocks per SM for a kernel at the given dynamic smem.
int occupancy_sc(int precision, int smem_bytes, int wpb);
int occupancy_list(int precision, int l, int fpw, int smem_bytes, int wpb, bool team = false);
// Frame-per-lane SC kernel (32 frames per warp; SC / SSC and the first pass
// of PA / FA).  For it LaunchParams.smem_per_warp / gscratch_per_frame are
// the shared / global bytes of one 32-frame warp.
int64_t lane_smem_bytes_per_warp(int nmax, int elem_bytes, int seg_smem_max, bool stage);
int64_t lane_gscratch_bytes_per_warp(int nmax, int elem_bytes, int seg_smem_max);
cudaError_t launch_sc_lanes(const LaunchParams& p, int precision, int grid, cudaStream_t s);
int occupancy_sc_lanes(int precision, int smem_bytes, int wpb);
// Frame ids [0, n) bucketed by code id into `out` (counting sort, 3 small
// launches); *count_out = n.  hist: ncodes ints of scratch.
cudaError_t bucket_by_code(const int32_t* cid, int64_t n, int ncodes, int32_t* hist, int32_t* out,
                           int32_t* count_out, cudaStream_t s);
// Commit of the speculative FA rungs (host.cu run_decode): for every frame
// of `list` (positions [0, *count), only if *count <= count_hi) the staged
// result of the first rung whose CRC passed, else of the last rung, goes to
// the real outputs.  nst rungs; rung j staged at position idx:
// st_payload + (j * cap + idx) * payload_stride etc.; levels[j] = its esc value.
struct CommitParams {
    const DevCode* codes;
    const int32_t* code_id;     // nullable
    const int32_t* list;
    const int32_t* count;
    int64_t count_hi;
    int32_t nst, cap;
    int32_t levels[4];
    const uint8_t* st_payload;
    const uint8_t* st_codeword; // nullable
    const uint8_t* st_crc;
    const float* st_metric;
    uint8_t* payload;
    uint8_t* codeword;          // nullable
    uint8_t* crc_ok;            // nullable
    uint8_t* esc;               // nullable
    float* metric;              // nullable
    int64_t payload_stride, codeword_stride;
};
cudaError_t launch_commit(const CommitParams& p, int blocks, cudaStream_t s);
// Exhaustive device check of the packed int8 f/g against the scalar kernels.
cudaError_t kernel_selftest(unsigned long long* mismatches);
#ifdef PLB_OPTIME
cudaError_t read_optime(unsigned long long* out, bool reset); // profiling build only
#endif

} // namespace plb
