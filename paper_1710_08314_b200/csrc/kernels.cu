// sm_100a kernels of the batched polar decoder.
//
// Mapping: a sub-warp of SW lanes (SW = 32, 16 or 8) decodes
// one frame at a time, so a warp carries 32/SW frames in lockstep.  A
// persistent grid of warps claims frames from an atomic counter (frames
// differ in cost under adaptive decoding).  Inside a sub-warp the lanes are
// spread over (list path, LLR element) pairs, and every fork / sort /
// slot-assignment step is sub-warp-synchronous (shuffles, ballots, match, no
// CTA barrier).  Per-path bookkeeping lives in registers with lane == slot:
// lane s holds the path metric of slot s.  Frames of one code walk the same
// op schedule with the same alive count at every op (the alive trace is
// data-independent), so sub-warps stay in lockstep; SW < 32 is
// used for small L, where the per-op control work, not the element work,
// dominates.
//
// LLR storage follows the reference's depth-segment stack (sc_decoder.hpp:
// 18-20, list_decoder.hpp:45) with lazy path copies: every depth d >= 1 has
// a pool of l buffers of n>>d values and each slot points at one buffer per
// depth (bufidx[slot][d]).  Duplicating a path (list_decoder.hpp:402-423)
// copies a 16-byte pointer row instead of up to L*n LLRs.  An F or G step at
// depth d rewrites the depth-(d+1) segment of EVERY alive path and no path
// ever reads the old contents, so the writer of rank r simply takes buffer r:
// no reference counts, no copy-on-write.  Depth 0 is the channel frame, read
// in place from HBM.  Small segments live in shared memory, large ones in a
// per-frame global scratch (L2-resident).  Partial sums are bit-packed, one
// n-bit row per slot, LSB-first within 32-bit words; h is a word XOR.
//
// Bit-exactness: f/g/h, the penalty sums (sequential, index
// order), the halving REP fold, the (value,index) two-smallest order, the
// stable (metric, emission-index) ranking, the slot assignment and int8 /
// int16 normalisation all reproduce list_decoder.hpp / sc_decoder.hpp
// exactly, for float, int8 and int16 LLRs.
//
// Kernel families in this translation unit: decode_kernel<R, KV, SW> (list
// passes at L = 2^(KV-1) and the warp-per-frame SC pass, KV = 0), its
// opt-in team variant (a block of warps per frame), sc_lanes_kernel<R> (the
// default SC pass: one frame per lane, lanes.cuh), the frame bucketing
// kernels for multi-code batches, and the int8 SWAR self-test.  The device
// primitives they share (sub-warp collectives, Arith, SWAR f/g, sorting
// networks, vector access, L2 policies) are in primitives.cuh.
#include <algorithm>
#include <cstdint>

#include "polar_dev.h"

namespace plb {
namespace {

#include "primitives.cuh"

// ---- per-frame shared-memory area ----------------------------------------
// (followed by the bufidx rows, [slot][depth] -> buffer index in the depth
// pool, 16 bytes per slot of the pass's list size).  Arrays indexed by slot
// or rank hold NS = SW entries (a sub-warp of SW lanes decodes L <= SW
// paths): the 16-lane kernels (L = 4, 8) use a 592-byte area instead of
// 1 040, which leaves room for more depth pools in shared memory (cfg1
// +1.8%).
template <int NS>
struct alignas(16) FixedS {
    uint8_t alive_list[NS];  // rank -> slot, ascending
    uint8_t freetab[NS];     // k -> k-th free slot, ascending
    uint8_t dsrc[NS], dtgt[NS]; // k-th duplicate of a fork: source, target
    uint32_t met_s[NS];      // metric by slot (fork hand-over)
    uint64_t pool[16];       // generic address of each depth pool
    uint32_t alive_w;        // alive-slot mask (read by the helper warps of a team)
    uint32_t pad_[3];
    union {
        struct {
            int32_t st_i1[NS], st_i2[NS], st_w[NS]; // per-rank node statistics
            uint32_t st_a1[NS], st_a2[NS];
        };
        // OP_SCSUB: per-level LLRs of the subtree, [level][lane], levels
        // 0..4 (the leaf level of a 32-subtree is never read back; SC pass,
        // never live together with a node's statistics; 32-lane kernels)
        uint32_t scv[5 * (NS == 32 ? 32 : 1)];
    };
};
static_assert(sizeof(FixedS<8>) % 16 == 0 && sizeof(FixedS<16>) % 16 == 0 && sizeof(FixedS<32>) % 16 == 0,
              "fixed area alignment");
// bytes of the fixed area of an SW-lane kernel
__host__ __device__ constexpr int fixed_bytes(int sw) {
    return sw >= 32 ? int(sizeof(FixedS<32>)) : sw >= 16 ? int(sizeof(FixedS<16>)) : int(sizeof(FixedS<8>));
}

__host__ __device__ inline int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) ++r;
    return r;
}
__host__ __device__ inline int align16(int v) { return (v + 15) & ~15; }

// Shared-memory layout of one frame: Fixed | bufidx | psum rows | depth pools that
// fit (segment <= segmax values); larger segments go to the frame's global
// scratch.  want_d selects which depth's pool offset to return.
struct LayoutQ {
    int32_t rw, psum_off, smem_total, gmem_total, pool_off, pool_in_smem;
};
// Word stride between the psum rows of two slots: 16-byte aligned with a
// 4-bank skew for n >= 128 (vector copies, and the same word of different
// slots falls into different banks), odd below.
__host__ __device__ inline int row_stride(int rw) { return rw >= 4 ? rw + 4 : (rw | 1); }

__host__ __device__ inline LayoutQ layout_query(int n, int l, int esz, int segmax, int want_d, int sw) {
    LayoutQ q{};
    int off = fixed_bytes(sw) + align16(16 * l);
    q.rw = n >= 32 ? n / 32 : 1;
    q.psum_off = off;
    off = align16(off + 4 * l * row_stride(q.rw));
    int goff = 0;
    const int stages = ilog2(n);
    #pragma unroll 1
    for (int d = 1; d <= stages; ++d) {
        const int seg = n >> d;
        const int bytes = align16(l * seg * esz);
        if (seg <= segmax) {
            if (d == want_d) {
                q.pool_off = off;
                q.pool_in_smem = 1;
            }
            off += bytes;
        } else {
            if (d == want_d) {
                q.pool_off = goff;
                q.pool_in_smem = 0;
            }
            // whole 128-byte L2 lines per global pool (discard.global.L2 of a
            // dead pool must not touch a neighbour's)
            goff += (bytes + 127) & ~127;
        }
    }
    q.smem_total = off;
    q.gmem_total = goff;
    return q;
}

// ---- frame decode context (one sub-warp) ---------------------------------
template <typename R, int SW>
struct Ctx {
    using A = Arith<R>;
    using M = typename A::M;

    Sub<SW> sw;
    int lane; // == sw.lane
    int n, l;
    unsigned lmask;
    const R* chan;
    FixedS<SW>* fx;
    uint32_t* ps;
    int rw;
    unsigned alive; // sub-warp-uniform alive-slot mask
    int myrank;     // rank of slot `lane` among the alive slots
    M metric;       // lane s: metric of slot s
    // element loops (F/G, H) run over a team of warps when team > 1: thread
    // tt0 of tstride; otherwise tt0 = lane, tstride = SW
    int tt0, tstride, team;
    bool discard; // float: discard.global.L2 dead global depth pools (LaunchParams::list_discard)

    __device__ __forceinline__ R* pool(int d) const { return reinterpret_cast<R*>(fx->pool[d]); }
    __device__ __forceinline__ uint8_t* bix() const { return reinterpret_cast<uint8_t*>(fx + 1); }
    // the frame's channel: a register pair in the int8 / int16 kernels; the
    // float kernels read it from fx->pool[0] (measured: cfg0 +0.9%, cfg1
    // -0.4% if both do)
    __device__ __forceinline__ R* channel() const {
        if constexpr (sizeof(R) == 4) return pool(0);
        else return const_cast<R*>(chan);
    }
    __device__ __forceinline__ R* llr(int p, int d) const {
        if (d == 0) return channel();
        return pool(d) + int(bix()[p * 16 + d]) * (n >> d);
    }
    __device__ __forceinline__ uint32_t* row(int p) const { return ps + p * row_stride(rw); }
    __device__ __forceinline__ bool is_alive() const { return (alive >> lane) & 1u; }

    __device__ void set_alive(unsigned a) {
        alive = a;
        myrank = __popc(alive & sw.lt());
        if (is_alive()) fx->alive_list[myrank] = uint8_t(lane);
        if (lane == 0) fx->alive_w = a;
        __syncwarp();
    }

    // int8 metrics: pull the smallest alive metric back to 0
    // (list_decoder.hpp:447-455).
    __device__ void normalize() {
        if constexpr (A::kFixed) {
            const int v = is_alive() ? int(metric) : A::kMax;
            const int mn = int(sw.red_min(unsigned(v)));
            if (is_alive()) metric -= mn;
        }
    }
};

// ---- f / g over all alive paths ----------------------------------------
// One body for F and G (is_g is uniform), two vector widths per type (G = 1
// for narrow nodes, G = 16 bytes otherwise): the decode loop's hot code must
// stay inside the instruction cache.
// o = f(a, b) or g(a, b, bits) on G values (bits: partial sum i in bit i)
template <typename R, int G>
__device__ __forceinline__ Vec<R, G> fg_compute(const Vec<R, G>& a, const Vec<R, G>& b, uint32_t bits,
                                                bool is_g) {
    using A = Arith<R>;
    Vec<R, G> o;
    if constexpr (sizeof(R) == 1 && G >= 4) {
        constexpr int W = G / 4;
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(&a.raw);
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(&b.raw);
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o.raw);
        if (is_g) {
#pragma unroll
            for (int w = 0; w < W; ++w) ow[w] = g_swar(aw[w], bw[w], (bits >> (4 * w)) & 15u);
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w) ow[w] = f_swar(aw[w], bw[w]);
        }
    } else if (is_g) {
#pragma unroll
        for (int i = 0; i < G; ++i) o.v[i] = A::g(a.v[i], b.v[i], (bits >> i) & 1u);
    } else if constexpr (sizeof(R) == 2 && G >= 2) {
        // int16 f: two values per 32-bit word
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(&a.raw);
        const uint32_t* bw = reinterpret_cast<const uint32_t*>(&b.raw);
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o.raw);
#pragma unroll
        for (int w = 0; w < G / 2; ++w) ow[w] = f_swar16(aw[w], bw[w]);
    } else {
#pragma unroll
        for (int i = 0; i < G; ++i) o.v[i] = A::f(a.v[i], b.v[i]);
    }
    return o;
}

template <typename R, int G>
__device__ __forceinline__ void fg_item(const R* in, R* out, const uint32_t* prow, int h,
                                        int c, int lb, bool is_g) {
    const Vec<R, G> a = vld<R, G>(in + c * G);
    const Vec<R, G> b = vld<R, G>(in + h + c * G);
    const int pos = lb + c * G;
    const uint32_t bits = is_g ? prow[pos >> 5] >> (pos & 31) : 0u;
    vst<R, G>(out + c * G, fg_compute<R, G>(a, b, bits, is_g));
}

template <typename R, int SW, int G>
__device__ __forceinline__ void fg_run(Ctx<R, SW>& cx, int d, int h, int lb, int na, bool is_g) {
    const int cp = h / G; // items per path, power of two
    const int lg = __ffs(cp) - 1;
    R* const outp = cx.pool(d + 1);
    R* const inp = d == 0 ? cx.channel() : cx.pool(d);
    const int seg = cx.n >> d;
    const int total = na << lg;
    #pragma unroll 1
    for (int t = cx.tt0; t < total; t += cx.tstride) {
        const int r = t >> lg;
        const int p = cx.fx->alive_list[r];
        const R* in = d == 0 ? inp : inp + int(cx.bix()[p * 16 + d]) * seg;
        fg_item<R, G>(in, outp + r * h, cx.row(p), h, t & (cp - 1), lb, is_g);
    }
}

// A chained op (kOpChain, float kernels with kChainKernel): the F / G op at
// depth d and the F op of its left child in one sweep.  An item is one chunk
// of the depth-(d+2) segment of a path: its two depth-(d+1) chunks (c and
// c + h/2) come from four input chunks (all four loads in flight), and both
// levels go to the buffers of the path's rank.  The child's F op (absent
// from the chained schedule) never reads the depth-(d+1) pool back, and its
// item loop, buffer lookups and dispatch are gone.
template <typename R, int SW, int G>
__device__ __forceinline__ void fg_run_chain(Ctx<R, SW>& cx, int d, int h, int lb, int na, bool is_g) {
    const int hh = h >> 1;
    const int cp2 = hh / G; // items per path, power of two
    const int lg = __ffs(cp2) - 1;
    R* const out1 = cx.pool(d + 1);
    R* const out2 = cx.pool(d + 2);
    R* const inp = d == 0 ? cx.channel() : cx.pool(d);
    const int seg = cx.n >> d;
    const int total = na << lg;
    #pragma unroll 1
    for (int t = cx.tt0; t < total; t += cx.tstride) {
        const int r = t >> lg, c = (t & (cp2 - 1)) * G;
        const int p = cx.fx->alive_list[r];
        const R* in = d == 0 ? inp : inp + int(cx.bix()[p * 16 + d]) * seg;
        const Vec<R, G> a0 = vld<R, G>(in + c), a1 = vld<R, G>(in + c + hh);
        const Vec<R, G> b0 = vld<R, G>(in + h + c), b1 = vld<R, G>(in + h + c + hh);
        uint32_t bits0 = 0, bits1 = 0;
        if (is_g) {
            const uint32_t* prow = cx.row(p);
            const int pos0 = lb + c, pos1 = lb + c + hh;
            bits0 = prow[pos0 >> 5] >> (pos0 & 31);
            bits1 = prow[pos1 >> 5] >> (pos1 & 31);
        }
        const Vec<R, G> r0 = fg_compute<R, G>(a0, b0, bits0, is_g);
        const Vec<R, G> r1 = fg_compute<R, G>(a1, b1, bits1, is_g);
        vst<R, G>(out1 + r * h + c, r0);
        vst<R, G>(out1 + r * h + c + hh, r1);
        vst<R, G>(out2 + r * hh + c, fg_compute<R, G>(r0, r1, 0u, false));
    }
}

// U items per lane in flight (all loads issued before the first compute):
// the L = 32 float kernel waits on L2 / DRAM for its depth pools, and one
// item per trip leaves a single load pair in flight per lane
template <typename R, int SW, int G, int U>
__device__ __forceinline__ void fg_run_batched(Ctx<R, SW>& cx, int d, int h, int lb, int na, bool is_g) {
    const int cp = h / G;
    const int lg = __ffs(cp) - 1;
    R* const outp = cx.pool(d + 1);
    R* const inp = d == 0 ? cx.channel() : cx.pool(d);
    const int seg = cx.n >> d;
    const int total = na << lg;
    #pragma unroll 1
    for (int t0 = cx.tt0; t0 < total; t0 += U * cx.tstride) {
        Vec<R, G> a[U], b[U];
        uint32_t bits[U];
        int ro[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * cx.tstride;
            const int tt = t < total ? t : t0; // tail: re-read item t0, store nothing
            const int r = tt >> lg, c = tt & (cp - 1);
            const int p = cx.fx->alive_list[r];
            const R* in = d == 0 ? inp : inp + int(cx.bix()[p * 16 + d]) * seg;
            a[u] = vld<R, G>(in + c * G);
            b[u] = vld<R, G>(in + h + c * G);
            const int pos = lb + c * G;
            bits[u] = is_g ? cx.row(p)[pos >> 5] >> (pos & 31) : 0u;
            ro[u] = t < total ? r * h + c * G : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (ro[u] >= 0) vst<R, G>(outp + ro[u], fg_compute<R, G>(a[u], b[u], bits[u], is_g));
    }
}

#ifndef PLB_FG_UNROLL
#define PLB_FG_UNROLL 2
#endif
#ifndef PLB_FG_UNROLL_MINKV
#define PLB_FG_UNROLL_MINKV 6
#endif
template <int UB = 1, bool CHK = false, typename R, int SW>
__device__ __forceinline__ void fg_elems(Ctx<R, SW>& cx, int d, int m, int lb, int na, bool is_g,
                                         bool chain = false) {
    constexpr int VE = 16 / int(sizeof(R));
    const int h = m >> 1;
    if constexpr (CHK) {
        if (chain) { // (host.cu chain_list_ops: h >= 2 * VE)
            fg_run_chain<R, SW, VE>(cx, d, h, lb, na, is_g);
            return;
        }
    }
    if constexpr (UB > 1) {
        if (h >= VE) {
            fg_run_batched<R, SW, VE, UB>(cx, d, h, lb, na, is_g);
            return;
        }
    }
    if (h >= VE) fg_run<R, SW, VE>(cx, d, h, lb, na, is_g);
    else if (sizeof(R) == 1 && h >= 4) fg_run<R, SW, 4>(cx, d, h, lb, na, is_g); // one SWAR word
    else fg_run<R, SW, 1>(cx, d, h, lb, na, is_g);
}

// Team barrier around an element op: the control warp's shared-state writes
// before it, the element results after it (team > 1 only).
template <typename R, int SW>
__device__ __forceinline__ void team_sync(const Ctx<R, SW>& cx) {
    if (cx.team > 1) __syncthreads();
    else __syncwarp();
}

template <int UB = 1, bool CHK = false, typename R, int SW>
__device__ void op_fg(Ctx<R, SW>& cx, int d, int m, int lb, int na, bool is_g, bool chain = false) {
    // the child segment of the path of rank r goes to buffer r (see header)
    if (cx.is_alive()) {
        cx.bix()[cx.lane * 16 + d + 1] = uint8_t(cx.myrank);
        if constexpr (CHK)
            if (chain) cx.bix()[cx.lane * 16 + d + 2] = uint8_t(cx.myrank);
    }
    if (cx.team > 1) __syncthreads();
    fg_elems<UB, CHK>(cx, d, m, lb, na, is_g, chain);
    team_sync(cx);
    if constexpr (sizeof(R) == 4 && SW == 32) {
        // after a G op the depth-d pool is dead (its next use is a write by
        // the parent's next op): drop its L2 lines without write-back when
        // it lives in global scratch, so dead LLRs never reach DRAM (the
        // float list passes write 2x what they read).  Float 32-lane kernels
        // (L >= 16) only: cfg4 L=32 / 16 +1.5%, L = 4 / 8 unchanged
        if (is_g && d > 0 && cx.discard && __isGlobal(cx.pool(d))) {
            const char* base = reinterpret_cast<const char*>(cx.pool(d));
            const int lines = (cx.l * (cx.n >> d) * int(sizeof(R))) >> 7;
            #pragma unroll 1
            for (int i = cx.lane; i < lines; i += SW)
                asm volatile("discard.global.L2 [%0], 128;" :: "l"(base + (size_t(i) << 7)) : "memory");
        }
    }
}

// psums[lb, lb+h) ^= psums[lb+h, lb+2h) for every alive path
template <typename R, int SW>
__device__ __forceinline__ void h_elems(Ctx<R, SW>& cx, int m, int lb, int na) {
    const int h = m >> 1;
    if (h >= 32) {
        const int W = h >> 5, lg = __ffs(W) - 1;
        const int total = na << lg;
        #pragma unroll 1
        for (int t = cx.tt0; t < total; t += cx.tstride) {
            uint32_t* w = cx.row(cx.fx->alive_list[t >> lg]) + (lb >> 5) + (t & (W - 1));
            w[0] ^= w[W];
        }
    } else if (cx.tt0 < na) {
        uint32_t* w = cx.row(cx.fx->alive_list[cx.tt0]) + (lb >> 5);
        const int s = lb & 31;
        const uint32_t mk = (1u << h) - 1u;
        *w ^= ((*w >> (s + h)) & mk) << s;
    }
}

template <typename R, int SW>
__device__ void op_h(Ctx<R, SW>& cx, int m, int lb, int na) {
    if (cx.team > 1) __syncthreads();
    h_elems(cx, m, lb, na);
    team_sync(cx);
}

// write `bit` over the span [lb, lb+m) of a psum row (whole sub-warp)
template <int SW>
__device__ __forceinline__ void span_fill(uint32_t* row, int lb, int m, int bit, int lane) {
    if (m >= 32) {
        #pragma unroll 1
        for (int w = lane; w < (m >> 5); w += SW) row[(lb >> 5) + w] = bit ? FULL : 0u;
    } else if (lane == 0) {
        const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
        uint32_t* w = row + (lb >> 5);
        *w = bit ? (*w | mk) : (*w & ~mk);
    }
}
// same from a single lane (m < 32)
__device__ __forceinline__ void span_fill_lane(uint32_t* row, int lb, int m, int bit) {
    const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
    uint32_t* w = row + (lb >> 5);
    *w = bit ? (*w | mk) : (*w & ~mk);
}

// Halving fold of the REP node's LLRs (sc_decoder.hpp:116-125,
// list_decoder.hpp:282-289) for every alive path; the result of rank r goes
// to st_a1[r].  For m > SW the first halvings run in the rank's depth-(d+1)
// buffer, whose contents are dead at a leaf.
#ifndef PLB_VLEAF_MINKV
#define PLB_VLEAF_MINKV 2 // float list kernels (KV >= this: L >= 2) with the batched leaf loops
                          // (cfg4 L=8 +6%, cfg0 / cfg3 +1%, L=2 rungs +0.6%;
                          // `profiles/r02_sweep_big_leaf.log`)
#endif
#ifndef PLB_VLEAF_VF
#define PLB_VLEAF_VF 1 // float list kernels: vectors per trip in the per-path leaf loops
                       // (2 / 4 in the L = 32 kernel: 111 / 126 registers, cfg4 L=32 -8% / -10%)
#endif
#ifndef PLB_VLEAF_R1
#define PLB_VLEAF_R1 1
#endif
#ifndef PLB_VLEAF_PEN
#define PLB_VLEAF_PEN 1
#endif
template <bool VLEAF = false, typename R, int SW>
__device__ void rep_fold(Ctx<R, SW>& cx, int d, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    if (m <= SW) {
        const int lgm = __ffs(m) - 1;
        const int per = SW >> lgm;
        #pragma unroll 1
        for (int r0 = 0; r0 < na; r0 += per) {
            const int r = r0 + (cx.lane >> lgm), i = cx.lane & (m - 1);
            const bool ok = r < na;
            M v = ok ? A::val(cx.llr(cx.fx->alive_list[r], d)[i]) : M(0);
            for (int off = m >> 1; off >= 1; off >>= 1) {
                const M o = __shfl_down_sync(FULL, v, off, m);
                if (i < off) v = A::sat(v, o);
            }
            if (ok && i == 0) cx.fx->st_a1[r] = mbits<M>(v);
        }
    } else if constexpr (sizeof(R) == 4 && VLEAF) {
        // float, m > SW: one halving level at a time for all paths together
        // (level len: S[i] = S[i] + S[i + len/2], i < len/2 — the same sums
        // as the per-path loop below, in the same tree), so a level costs one
        // round trip to the depth-(d+1) buffers instead of one per path
        const int h = m >> 1;
        R* const S0 = cx.pool(d + 1);
        {
            const int q = h >> 2, lgq = __ffs(q) - 1; // float4 items per path
            #pragma unroll 1
            for (int t = cx.lane; t < (na << lgq); t += SW) {
                const int r = t >> lgq, c = (t & (q - 1)) << 2;
                const R* L = cx.llr(cx.fx->alive_list[r], d);
                const Vec<R, 4> a = vld<R, 4>(L + c), b = vld<R, 4>(L + h + c);
                vst<R, 4>(S0 + r * h + c, fg_compute<R, 4>(a, b, 0u, true)); // g with u = 0: a + b
            }
            __syncwarp();
        }
        #pragma unroll 1
        for (int len = h; len > 1; len >>= 1) {
            const int hh = len >> 1, lgh = __ffs(hh) - 1;
            #pragma unroll 1
            for (int t = cx.lane; t < (na << lgh); t += SW) {
                R* S = S0 + (t >> lgh) * h;
                const int i = t & (hh - 1);
                S[i] = A::store(A::sat(A::val(S[i]), A::val(S[i + hh])));
            }
            __syncwarp();
        }
        if (cx.lane < na) cx.fx->st_a1[cx.lane] = mbits<M>(A::val(S0[cx.lane * h]));
    } else {
        #pragma unroll 1
        for (int r = 0; r < na; ++r) {
            const R* L = cx.llr(cx.fx->alive_list[r], d);
            R* S = cx.pool(d + 1) + r * (m >> 1);
            const int h = m >> 1;
            #pragma unroll 1
            for (int i = cx.lane; i < h; i += SW) S[i] = A::store(A::sat(A::val(L[i]), A::val(L[i + h])));
            __syncwarp();
            #pragma unroll 1
            for (int len = h; len > SW; len >>= 1) {
                const int hh = len >> 1;
                #pragma unroll 1
                for (int i = cx.lane; i < hh; i += SW) S[i] = A::store(A::sat(A::val(S[i]), A::val(S[i + hh])));
                __syncwarp();
            }
            M v = A::val(S[cx.lane]);
            for (int off = SW / 2; off >= 1; off >>= 1) {
                const M o = __shfl_down_sync(FULL, v, off, SW);
                if (cx.lane < off) v = A::sat(v, o);
            }
            if (cx.lane == 0) cx.fx->st_a1[r] = mbits<M>(v);
            __syncwarp();
        }
    }
    __syncwarp();
}

// ---- list decoder: candidate ranking and slot assignment ----------------
enum ApplyKind { AK_BIT = 0, AK_BCAST = 1, AK_FLIPS = 2 };

// fork_apply (list_decoder.hpp:339-387) for ncand candidates held as
// candidate i = lane + SW*k in register k; candidate i belongs to the path of
// rank i >> lgb and is that path's candidate number i & (2^lgb - 1) at a node
// of type `code` (its decision is decoded from the node statistics after the
// ranking, so only the metrics travel through the sort).
template <typename R, int SW, int CPL, int MAXW>
__device__ void fork_apply(Ctx<R, SW>& cx, const typename Arith<R>::M (&cm)[CPL],
                           const int (&csrc)[CPL], const int (&caux)[CPL], int ncand,
                           int code, int lgb, int lb, int m, int lgrun) {
    using A = Arith<R>;
    using M = typename A::M;
    using K = typename A::Key;
    const int lane = cx.lane;
    // 1. stable order by (metric, emission index): a sub-warp bitonic sort of
    //    the unique keys leaves the candidate of rank r in lane r (register 0)
    K key[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = lane + SW * k;
        key[k] = i < ncand ? A::make_key(cm[k], i) : A::kKeyMax;
    }
    if constexpr (CPL == 1) {
        // two network widths per kernel: MAXW = min(SW, 4L) and MAXW/2
        if (MAXW > 4 && ncand <= MAXW / 2) key[0] = sort_runs<K, (MAXW > 4 ? MAXW / 2 : 4)>(key[0], lane, lgrun);
        else key[0] = sort_runs<K, MAXW>(key[0], lane, lgrun);
    } else if constexpr (CPL == 2) {
        // 4L <= 2 SW: keep = L <= SW/2, so the best SW/2 suffice
        if (ncand > SW) key[0] = top_half2<K, SW>(key[0], key[1], lane, lgrun);
        else key[0] = sort_runs<K, SW>(key[0], lane, lgrun);
    } else {
        // only the best keep <= SW are needed, in order
        int nreg = (ncand + SW - 1) / SW;
        if constexpr (!A::kFixed && SW == 32) {
            // L = 32 float, all paths alive: every path's smallest candidate
            // (the head of its sorted run) has a metric <= T = the largest of
            // them, so >= L candidates do and none with a larger metric can
            // be kept.  Survivors (99% of the 128-candidate R1 forks keep <= 64,
            // measured at cfg4) are compacted in emission order into two
            // registers through the node-statistics area (the float path
            // carries its decisions in registers, the statistics are spent):
            // cfg4 L=32 +5% (the 64-candidate REP / SPC forks: -1%, not done).
            if (ncand > 2 * SW && __popc(cx.alive) == cx.l && lgrun > 0) {
                uint32_t hb = 0;
#pragma unroll
                for (int k = 0; k < CPL; ++k)
                    if ((lane & ((1 << lgrun) - 1)) == 0 && lane + SW * k < ncand)
                        hb = max(hb, uint32_t(key[k] >> 32));
                const uint32_t t = __reduce_max_sync(FULL, hb);
                unsigned bal[CPL];
                int cnt = 0;
#pragma unroll
                for (int k = 0; k < CPL; ++k) {
                    bal[k] = __ballot_sync(FULL, lane + SW * k < ncand && uint32_t(key[k] >> 32) <= t);
                    cnt += __popc(bal[k]);
                }
                if (cnt <= 2 * SW) {
                    K* stage = reinterpret_cast<K*>(cx.fx->st_i1);
                    int base = 0;
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        if ((bal[k] >> lane) & 1u) stage[base + __popc(bal[k] & lanemask_lt())] = key[k];
                        base += __popc(bal[k]);
                    }
                    __syncwarp();
                    key[0] = lane < cnt ? stage[lane] : A::kKeyMax;
                    key[1] = lane + SW < cnt ? stage[SW + lane] : A::kKeyMax;
#pragma unroll
                    for (int k = 2; k < CPL; ++k) key[k] = A::kKeyMax;
                    __syncwarp();
                    nreg = cnt > SW ? 2 : 1;
                    lgrun = 0;
                }
            }
        }
        top_regs<K, CPL, SW>(key, lane, nreg, lgrun);
    }
    const int keep = min(cx.l, ncand);
    const bool kept = lane < keep;
    const int ci = kept ? A::key_idx(key[0]) : 0;
    const M cmet = A::key_val(key[0]);
    // the ranked candidate's source path and decision (list_decoder.hpp:
    // 240-333): ca = the bit (info leaf, REP) or the first flip, cb = the
    // second flip (R1 / SPC; -1 = none)
    int src, ca, cb = -1;
    if constexpr (A::kFixed) {
        // issue-bound fixed-point kernels: decoded from the node statistics
        const int cr = ci >> lgb, j = ci & ((1 << lgb) - 1);
        src = cx.fx->alive_list[cr];
        if (code == OP_INFO) {
            ca = j;
        } else if (code == OP_REP) {
            ca = cx.fx->st_w[cr] ^ j;
        } else {
            // R1: none, i1, i2, i1&i2.  SPC: broken parity -> i1, i2;
            // intact -> none, i1&i2.
            const int jj = code == OP_R1 ? j : (cx.fx->st_w[cr] ? j + 1 : j * 3);
            const int i1 = cx.fx->st_i1[cr], i2 = cx.fx->st_i2[cr];
            ca = jj == 0 ? -1 : jj == 2 ? i2 : i1;
            if (jj == 3) cb = i2;
        }
    } else {
        // latency-bound float kernels: emitted before the ranking (off its
        // critical path), fetched from the emitting lane
        int aux = 0;
        src = 0;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int sv = cx.sw.shfl(csrc[k], ci & (SW - 1));
            const int av = cx.sw.shfl(caux[k], ci & (SW - 1));
            if (ci / SW == k) {
                src = sv;
                aux = av;
            }
        }
        ca = int(int16_t(aux & 0xffff));
        cb = aux >> 16;
    }
    if (!kept) src = 64 + lane;
    const int kind = code == OP_INFO ? AK_BIT : code == OP_REP ? AK_BCAST : AK_FLIPS;
    // 2. slot assignment: the first use of a slot stays in place, the others
    //    take the free slots in ascending order, in rank order
    const unsigned same = cx.sw.match(src);
    const bool first = kept && (__ffs(same) - 1) == lane;
    const unsigned surv = cx.sw.red_or(kept ? (1u << src) : 0u);
    const bool dup = kept && !first;
    const unsigned dupm = cx.sw.ballot(dup);
    int tgt = src;
    {
        const unsigned freem = cx.lmask & ~surv;
        if ((freem >> lane) & 1u) cx.fx->freetab[__popc(freem & cx.sw.lt())] = uint8_t(lane);
        __syncwarp();
        if (dup) {
            const int k = __popc(dupm & cx.sw.lt());
            tgt = cx.fx->freetab[k];
            cx.fx->dsrc[k] = uint8_t(src);
            cx.fx->dtgt[k] = uint8_t(tgt);
            // 3. duplicate: the LLR pointer row ...
            *reinterpret_cast<uint4*>(cx.bix() + tgt * 16) =
                *reinterpret_cast<const uint4*>(cx.bix() + src * 16);
        }
        __syncwarp();
        // ... and the decided partial sums incl. the node span (which holds
        // the source's hard decisions for R1/SPC); words past the decided
        // prefix are don't-care, so whole 16-byte chunks are copied, all
        // duplicates at once
        const int nw = min(cx.rw, (lb + m + 31) >> 5);
        const int nd = __popc(dupm);
        if (cx.rw >= 4) {
            const int n4 = (nw + 3) >> 2;
            const int lg = n4 > 1 ? 32 - __clz(n4 - 1) : 0; // ceil(log2(n4))
            #pragma unroll 1
            for (int t = lane; t < (nd << lg); t += SW) {
                const int k = t >> lg, q = t & ((1 << lg) - 1);
                if (q < n4)
                    reinterpret_cast<uint4*>(cx.row(cx.fx->dtgt[k]))[q] =
                        reinterpret_cast<const uint4*>(cx.row(cx.fx->dsrc[k]))[q];
            }
        } else if (lane < nd) {
            for (int w = 0; w < cx.rw; ++w) cx.row(cx.fx->dtgt[lane])[w] = cx.row(cx.fx->dsrc[lane])[w];
        }
        __syncwarp();
    }
    // 4. apply decisions (list_decoder.hpp:425-445)
    if (kind == AK_BIT) {
        if (kept) span_fill_lane(cx.row(tgt), lb, 1, ca);
    } else if (kind == AK_BCAST) {
        if (m < 32) {
            if (kept) span_fill_lane(cx.row(tgt), lb, m, ca);
        } else {
            #pragma unroll 1
            for (int r = 0; r < keep; ++r) {
                const int t = cx.sw.shfl(tgt, r);
                const int bit = cx.sw.shfl(ca, r);
                span_fill<SW>(cx.row(t), lb, m, bit, lane);
            }
        }
    } else if (kept) {
        uint32_t* tr = cx.row(tgt);
        if (ca >= 0) tr[(lb + ca) >> 5] ^= 1u << ((lb + ca) & 31);
        if (cb >= 0) tr[(lb + cb) >> 5] ^= 1u << ((lb + cb) & 31);
    }
    if (kept) cx.fx->met_s[tgt] = mbits<M>(cmet);
    const unsigned nal = cx.sw.red_or(kept ? (1u << tgt) : 0u);
    __syncwarp();
    if ((nal >> lane) & 1u) cx.metric = mfrom<M>(cx.fx->met_s[lane]);
    if constexpr (A::kFixed) {
        // normalisation (list_decoder.hpp:447-455): the smallest alive metric
        // is the rank-0 candidate's, no reduction needed
        const M mn = cx.sw.shfl(cmet, 0);
        if ((nal >> lane) & 1u) cx.metric -= mn;
    }
    cx.set_alive(nal);
}

// frozen leaf / rate-0 node (list_decoder.hpp:227-238)
template <bool VLEAF = false, typename R, int SW>
__device__ void list_frozen(Ctx<R, SW>& cx, int d, int m, int lb, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    M pen = M(0);
    if (A::kFixed && m >= 32) {
        // saturating sums of non-negative terms are order-free in int8
        #pragma unroll 1
        for (int r = 0; r < na; ++r) {
            const R* L = cx.llr(cx.fx->alive_list[r], d);
            int s = 0;
            #pragma unroll 1
            for (int i = cx.lane; i < m; i += SW) s += max(0, -int(A::val(L[i])));
            s = int(cx.sw.red_add(unsigned(s)));
            if (cx.lane == r) pen = M(min(s, A::kMax));
        }
    } else if (cx.lane < na) {
        const R* L = cx.llr(cx.fx->alive_list[cx.lane], d);
        if (sizeof(R) == 4 && VLEAF && PLB_VLEAF_PEN && m >= 8) {
            // float: PLB_VLEAF_VF vectors in flight per trip; the penalty
            // is still summed one value at a time in index order
            #pragma unroll 1
            for (int i = 0; i < m; i += 4 * PLB_VLEAF_VF) {
                Vec<R, 4> q[PLB_VLEAF_VF];
#pragma unroll
                for (int u = 0; u < PLB_VLEAF_VF; ++u)
                    if (i + 4 * u < m) q[u] = vld<R, 4>(L + i + 4 * u);
#pragma unroll
                for (int u = 0; u < PLB_VLEAF_VF; ++u)
                    if (i + 4 * u < m)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const M v = A::val(q[u].v[j]);
                            if (v < M(0)) pen = A::sat(pen, -v);
                        }
            }
        } else {
            #pragma unroll 1
            for (int i = 0; i < m; ++i) {
                const M v = A::val(L[i]);
                if (v < M(0)) pen = A::sat(pen, -v); // sequential: float order matters
            }
        }
    }
    const M pr = cx.sw.shfl(pen, cx.myrank & (SW - 1));
    if (cx.is_alive()) cx.metric = A::sat(cx.metric, pr);
    if (m >= 32) {
        const int W = m >> 5;
        #pragma unroll 1
        for (int t = cx.lane; t < na * W; t += SW)
            cx.row(cx.fx->alive_list[t / W])[(lb >> 5) + (t % W)] = 0u;
    } else if (cx.lane < na) {
        span_fill_lane(cx.row(cx.fx->alive_list[cx.lane]), lb, m, 0);
    }
    __syncwarp();
    cx.normalize();
}

// Per-path statistics of an R1 / SPC node: hard decisions written into the
// path's own psum span, the two smallest magnitudes under the (value, index)
// order (select.hpp:18-68) -> st_i1/st_a1, st_i2/st_a2, parity -> st_w.
// gf (a big fused leaf, kOpFused | kOpFusedG on a node of more than the
// fused_leaf sizes): the node is a right child whose parent's G op was
// dropped from the schedule; its LLRs are formed here, from the parent
// segment (depth d - 1) and the left sibling's decisions, and never stored
// -- nothing reads a leaf's LLRs after its statistics.
template <bool VLEAF = false, bool BF = false, typename R, int SW>
__device__ void r1spc_stats(Ctx<R, SW>& cx, int d, int m, int lb, int na, bool gf_arg = false) {
    const bool gf = BF && gf_arg; // (folds away in the kernels without big fused leaves)
    using A = Arith<R>;
    using M = typename A::M;
    using K = typename A::Key;
    // One pass over all paths: lp lanes per path (na is a power of two, C22).
    const int lp = min(m, SW / na);
    const int lglp = __ffs(lp) - 1;
    const int E = m >> lglp;
    const int r = cx.lane >> lglp, l0 = cx.lane & (lp - 1);
    const bool ok = r < na;
    const int p = cx.fx->alive_list[ok ? r : 0];
    if (E == 1) {
        // one value per lane (lp == m): every path's hard bits in one ballot
        M v = M(0);
        if (ok) {
            if (gf) {
                const R* pa = cx.llr(p, d - 1);
                const int up = lb - m + l0;
                v = A::val(A::g(pa[l0], pa[m + l0], (cx.row(p)[up >> 5] >> (up & 31)) & 1u));
            } else {
                v = A::val(cx.llr(p, d)[l0]);
            }
        }
        const unsigned hb = cx.sw.ballot(ok && v < M(0));
        const uint32_t mk = m >= 32 ? FULL : ((1u << m) - 1u);
        const uint32_t gb = (hb >> (cx.lane & ~(lp - 1))) & mk;
        K k1 = ok ? A::make_key(A::mag(v), l0) : A::kKeyMax, k2 = A::kKeyMax;
        for (int off = 1; off < lp; off <<= 1) {
            const K o1 = shfl_xor_k(k1, off), o2 = shfl_xor_k(k2, off);
            const K n1 = kmin(k1, o1);
            k2 = kmin(kmax(k1, o1), kmin(k2, o2));
            k1 = n1;
        }
        if (ok && l0 == 0) {
            uint32_t* w = cx.row(p) + (lb >> 5);
            const int sh = lb & 31;
            *w = (*w & ~(mk << sh)) | (gb << sh);
            cx.fx->st_i1[r] = A::key_idx(k1);
            cx.fx->st_i2[r] = A::key_idx(k2);
            cx.fx->st_a1[r] = mbits<M>(A::key_val(k1));
            cx.fx->st_a2[r] = mbits<M>(A::key_val(k2));
            cx.fx->st_w[r] = __popc(gb) & 1;
        }
        __syncwarp();
        return;
    }
    // lane l0 of a group takes the E = m/lp consecutive values
    // [l0*E, (l0+1)*E) of its path (vector loads), builds their hard bits
    // locally and ORs them into the path's (cleared) psum span.
    const int i0 = l0 * E;
    // (gf: L = the parent's left half at this lane's values, L + m its right
    // half, ub0 = the position of the left sibling's decision for value i0)
    const R* L = (gf ? cx.llr(p, d - 1) : cx.llr(p, d)) + i0;
    const uint32_t* urow = cx.row(p);
    const int ub0 = lb - m + i0;
    uint32_t* span = cx.row(p) + (lb >> 5);
    const int base = m < 32 ? (lb & 31) : 0; // span bit of value 0 within span[0]
    if (ok && l0 == 0) {
        if (m >= 32) {
            #pragma unroll 1
            for (int w = 0; w < (m >> 5); ++w) span[w] = 0u;
        } else {
            *span &= ~(((1u << m) - 1u) << base);
        }
    }
    __syncwarp();
    K k1 = A::kKeyMax, k2 = A::kKeyMax;
    uint32_t acc = 0;
    int par = 0;
    bool swar = false;
    if constexpr (sizeof(R) == 1) swar = E >= 4 && m <= 512;
    if (ok && swar) {
        // int8, four values per word: hard bits from the sign bits, |v| by
        // VABSDIFF4, the two smallest (|v| << 9 | index) keys per 16-bit lane
        // by VIMNMX.U16x2 (index < 512: the (value, index) order of
        // select.hpp:18-68 in 16 bits)
        uint32_t q1 = FULL, q2 = FULL;
        #pragma unroll 1
        for (int k = 0; k < E; k += 4) {
            uint32_t w = *reinterpret_cast<const uint32_t*>(L + k);
            if (gf)
                w = g_swar(w, *reinterpret_cast<const uint32_t*>(L + m + k),
                           (urow[(ub0 + k) >> 5] >> ((ub0 + k) & 31)) & 15u);
            acc |= ((((w >> 7) & 0x01010101u) * 0x01020408u) >> 24) << (k & 31);
            const uint32_t a4 = __vabsdiffu4(w ^ 0x80808080u, 0x80808080u);
            const uint32_t ix = uint32_t(i0 + k) * 0x00010001u + 0x00010000u;
            const uint32_t ka = prmt(a4, 0, 0x4140) * 512u + ix;
            const uint32_t kb = prmt(a4, 0, 0x4342) * 512u + ix + 0x00020002u;
            uint32_t n1 = __vminu2(q1, ka);
            q2 = __vminu2(q2, __vmaxu2(q1, ka));
            q1 = n1;
            n1 = __vminu2(q1, kb);
            q2 = __vminu2(q2, __vmaxu2(q1, kb));
            q1 = n1;
            if (((k + 4) & 31) == 0 || k + 4 >= E) {
                const int pos = base + i0 + (k & ~31);
                if (acc) atomicOr(span + (pos >> 5), acc << (pos & 31));
                par ^= __popc(acc);
                acc = 0;
            }
        }
        const uint32_t x = q1 & 0xffffu, y = q1 >> 16;
        const uint32_t e1 = min(x, y), e2 = min(max(x, y), min(q2 & 0xffffu, q2 >> 16));
        k1 = K(((e1 >> 9) << 16) | (e1 & 511u));
        k2 = K(((e2 >> 9) << 16) | (e2 & 511u));
    } else if (sizeof(R) == 4 && VLEAF && PLB_VLEAF_R1 && ok && E >= 4 * PLB_VLEAF_VF) {
        // float (VLEAF): PLB_VLEAF_VF vectors per trip, keys in index order
        #pragma unroll 1
        for (int k = 0; k < E; k += 4 * PLB_VLEAF_VF) {
            Vec<R, 4> q[PLB_VLEAF_VF];
#pragma unroll
            for (int u = 0; u < PLB_VLEAF_VF; ++u) q[u] = vld<R, 4>(L + k + 4 * u);
            if (gf) {
#pragma unroll
                for (int u = 0; u < PLB_VLEAF_VF; ++u) {
                    const int up = ub0 + k + 4 * u;
                    q[u] = fg_compute<R, 4>(q[u], vld<R, 4>(L + m + k + 4 * u), urow[up >> 5] >> (up & 31), true);
                }
            }
#pragma unroll
            for (int u = 0; u < PLB_VLEAF_VF; ++u)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const M v = A::val(q[u].v[j]);
                    acc |= uint32_t(v < M(0)) << ((k + 4 * u + j) & 31);
                    const K kv = A::make_key(A::mag(v), i0 + k + 4 * u + j);
                    const K n1 = kmin(k1, kv);
                    k2 = kmin(k2, kmax(k1, kv));
                    k1 = n1;
                }
            if (((k + 4 * PLB_VLEAF_VF) & 31) == 0 || k + 4 * PLB_VLEAF_VF >= E) {
                const int pos = base + i0 + (k & ~31);
                if (acc) atomicOr(span + (pos >> 5), acc << (pos & 31));
                par ^= __popc(acc);
                acc = 0;
            }
        }
    } else if (ok) {
        #pragma unroll 1
        for (int k = 0; k < E; k += 4) {
            M v[4];
            if (E >= 4) {
                Vec<R, 4> q = vld<R, 4>(L + k);
                if (gf) q = fg_compute<R, 4>(q, vld<R, 4>(L + m + k), urow[(ub0 + k) >> 5] >> ((ub0 + k) & 31), true);
                #pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = A::val(q.v[j]);
            } else {
                #pragma unroll
                for (int j = 0; j < 4; ++j)
                    v[j] = j >= E ? M(0)
                           : gf   ? A::val(A::g(L[j], L[m + j], (urow[(ub0 + j) >> 5] >> ((ub0 + j) & 31)) & 1u))
                                  : A::val(L[j]);
            }
            #pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j < E) {
                    acc |= uint32_t(v[j] < M(0)) << ((k + j) & 31);
                    const K kv = A::make_key(A::mag(v[j]), i0 + k + j);
                    const K n1 = kmin(k1, kv);
                    k2 = kmin(k2, kmax(k1, kv));
                    k1 = n1;
                }
            }
            if (((k + 4) & 31) == 0 || k + 4 >= E) {
                const int pos = base + i0 + (k & ~31);
                if (acc) atomicOr(span + (pos >> 5), acc << (pos & 31));
                par ^= __popc(acc);
                acc = 0;
            }
        }
    }
    for (int off = 1; off < lp; off <<= 1) {
        const K o1 = shfl_xor_k(k1, off), o2 = shfl_xor_k(k2, off);
        const K n1 = kmin(k1, o1);
        k2 = kmin(kmax(k1, o1), kmin(k2, o2));
        k1 = n1;
        par ^= __shfl_xor_sync(FULL, par, off);
    }
    if (ok && l0 == 0) {
        cx.fx->st_i1[r] = A::key_idx(k1);
        cx.fx->st_i2[r] = A::key_idx(k2);
        cx.fx->st_a1[r] = mbits<M>(A::key_val(k1));
        cx.fx->st_a2[r] = mbits<M>(A::key_val(k2));
        cx.fx->st_w[r] = par & 1;
    }
    __syncwarp();
}

// repetition node (list_decoder.hpp:276-305): after the fold, pen_w = the
// sum of the magnitudes that disagree with the fold's decision, sequential
// in index order (float order matters; int8 is order-free) -> st_a2, st_w.
template <bool VLEAF = false, typename R, int SW>
__device__ void rep_pen(Ctx<R, SW>& cx, int d, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    if (A::kFixed && m >= 32) {
        #pragma unroll 1
        for (int r = 0; r < na; ++r) {
            const R* L = cx.llr(cx.fx->alive_list[r], d);
            const bool w = mfrom<M>(cx.fx->st_a1[r]) < M(0);
            int s = 0;
            #pragma unroll 1
            for (int i = cx.lane; i < m; i += SW) {
                const int v = int(A::val(L[i]));
                if (w ? (v > 0) : (v < 0)) s += abs(v);
            }
            s = int(cx.sw.red_add(unsigned(s)));
            if (cx.lane == 0) {
                cx.fx->st_w[r] = w;
                cx.fx->st_a2[r] = mbits<M>(M(min(s, A::kMax)));
            }
        }
    } else if (cx.lane < na) {
        const R* L = cx.llr(cx.fx->alive_list[cx.lane], d);
        const bool w = mfrom<M>(cx.fx->st_a1[cx.lane]) < M(0);
        M pen = M(0);
        if (sizeof(R) == 4 && VLEAF && PLB_VLEAF_PEN && m >= 8) {
            // float: PLB_VLEAF_VF vectors in flight per trip, summed in index order
            #pragma unroll 1
            for (int i = 0; i < m; i += 4 * PLB_VLEAF_VF) {
                Vec<R, 4> q[PLB_VLEAF_VF];
#pragma unroll
                for (int u = 0; u < PLB_VLEAF_VF; ++u)
                    if (i + 4 * u < m) q[u] = vld<R, 4>(L + i + 4 * u);
#pragma unroll
                for (int u = 0; u < PLB_VLEAF_VF; ++u)
                    if (i + 4 * u < m)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const M v = A::val(q[u].v[j]);
                            if (w ? (v > M(0)) : (v < M(0))) pen = A::sat(pen, A::mag(v));
                        }
            }
        } else {
            #pragma unroll 1
            for (int i = 0; i < m; ++i) {
                const M v = A::val(L[i]);
                if (w ? (v > M(0)) : (v < M(0))) pen = A::sat(pen, A::mag(v));
            }
        }
        cx.fx->st_w[cx.lane] = w;
        cx.fx->st_a2[cx.lane] = mbits<M>(pen);
    }
    __syncwarp();
}

// A leaf of m <= MF values fused with its parent's F or G (kOpFused): lane r
// < na computes the m LLRs of the path of rank r in registers from the
// parent segment (depth d-1) and takes the leaf's statistics in-lane, with
// the same kernels, orders and tie rules as the unfused ops (r1spc_stats,
// rep_fold/rep_pen, list_frozen; list_decoder.hpp:227-333).  The depth-d
// segment is never written: nothing reads a leaf's LLRs afterwards.
template <typename R, int SW>
__device__ void fused_leaf(Ctx<R, SW>& cx, int code, int d, int m, int lb, int na, bool is_g) {
    using A = Arith<R>;
    using M = typename A::M;
    using K = typename A::Key;
    constexpr int MF = sizeof(R) == 1 ? kFuseMaxI8 : kFuseMaxF32;
    const int r = cx.lane;
    M pen = M(0);
    if constexpr (sizeof(R) == 1) {
        // int8: the m <= 8 child values packed in one u64 (value i in byte
        // i), produced by the SWAR f / g, statistics in rolled loops (small
        // code: the decode loop must stay inside the instruction cache)
        if (r < na) {
            const int p = cx.fx->alive_list[r];
            const R* in = cx.llr(p, d - 1);
            uint32_t* row = cx.row(p);
            uint32_t bits = 0;
            if (is_g) {
                const int pos = lb - m; // the left sibling's decisions
                bits = row[pos >> 5] >> (pos & 31);
            }
            uint64_t pk = 0;
            if (m >= 4) {
                #pragma unroll 1
                for (int q = 0; q < m; q += 4) {
                    const uint32_t a4 = *reinterpret_cast<const uint32_t*>(in + q);
                    const uint32_t b4 = *reinterpret_cast<const uint32_t*>(in + m + q);
                    const uint32_t c4 = is_g ? g_swar(a4, b4, (bits >> q) & 15u) : f_swar(a4, b4);
                    pk |= uint64_t(c4) << (8 * q);
                }
            } else {
                #pragma unroll 1
                for (int i = 0; i < m; ++i) {
                    const R c = is_g ? A::g(in[i], in[m + i], (bits >> i) & 1u) : A::f(in[i], in[m + i]);
                    pk |= uint64_t(uint8_t(c)) << (8 * i);
                }
            }
            // statistics on the packed bytes (values past m are 0): byte
            // magnitudes by VABSDIFF4, sums by VABSDIFF4.ACC (SAD), the two
            // smallest (|v|, index) keys as 16-bit lanes through VIMNMX.U16x2
            const uint32_t lo = uint32_t(pk), hi = uint32_t(pk >> 32);
            const uint32_t mk = (1u << m) - 1u;
            const uint32_t hb = ((((lo >> 7) & 0x01010101u) * 0x01020408u) >> 24 |
                                 ((((hi >> 7) & 0x01010101u) * 0x01020408u) >> 24) << 4) & mk;
            const uint32_t alo = __vabsdiffu4(lo ^ 0x80808080u, 0x80808080u);
            const uint32_t ahi = __vabsdiffu4(hi ^ 0x80808080u, 0x80808080u);
            const uint32_t nlo = prmt(lo, 0, 0xba98), nhi = prmt(hi, 0, 0xba98); // 0xff: negative
            uint32_t* w = row + (lb >> 5);
            const int sh = lb & 31;
            if (code == OP_FROZEN) {
                // non-negative terms: the saturating sum is order-free
                const int s = int(__vsadu4(alo & nlo, 0u) + __vsadu4(ahi & nhi, 0u));
                pen = min(s, 127);
                *w &= ~(mk << sh);
            } else if (code == OP_INFO) {
                cx.fx->st_a1[r] = mbits<M>(int(int8_t(uint8_t(lo))));
            } else if (code == OP_REP) {
                // halving fold: value i of level len/2 = sat(i + i + len/2)
                uint32_t x = m == 8 ? g_swar(lo, hi, 0u) : lo;
                #pragma unroll 1
                for (int len = m == 8 ? 4 : m; len > 1; len >>= 1) x = g_swar(x, x >> (4 * len), 0u);
                const int f0 = int(int8_t(uint8_t(x)));
                const bool wn = f0 < 0;
                // magnitudes of the values that disagree with the fold
                const int s = int(__vsadu4(alo & (wn ? ~nlo : nlo), 0u) + __vsadu4(ahi & (wn ? ~nhi : nhi), 0u));
                cx.fx->st_w[r] = wn;
                cx.fx->st_a1[r] = mbits<M>(f0);
                cx.fx->st_a2[r] = mbits<M>(min(s, 127));
            } else {
                // keys (|v| << 3 | i), two per word; values past m -> 0xffff
                uint32_t k0 = prmt(alo, 0, 0x4140) * 8u + 0x00010000u;
                uint32_t k1 = prmt(alo, 0, 0x4342) * 8u + 0x00030002u;
                uint32_t k2 = prmt(ahi, 0, 0x4140) * 8u + 0x00050004u;
                uint32_t k3 = prmt(ahi, 0, 0x4342) * 8u + 0x00070006u;
                if (m < 2) k0 |= 0xffff0000u;
                if (m < 4) k1 = FULL;
                if (m < 8) k2 = k3 = FULL;
                const uint32_t mn01 = __vminu2(k0, k1), mx01 = __vmaxu2(k0, k1);
                const uint32_t mn23 = __vminu2(k2, k3), mx23 = __vmaxu2(k2, k3);
                const uint32_t a = __vminu2(mn01, mn23);                                   // per lane: smallest
                const uint32_t b = __vminu2(__vmaxu2(mn01, mn23), __vminu2(mx01, mx23));  // second
                const uint32_t alo16 = a & 0xffffu, ahi16 = a >> 16;
                const uint32_t e1 = min(alo16, ahi16);
                const uint32_t e2 = min(max(alo16, ahi16), min(b & 0xffffu, b >> 16));
                *w = (*w & ~(mk << sh)) | (hb << sh);
                cx.fx->st_i1[r] = int(e1 & 7u);
                cx.fx->st_i2[r] = int(e2 & 7u);
                cx.fx->st_a1[r] = mbits<M>(int(e1 >> 3));
                cx.fx->st_a2[r] = mbits<M>(int(e2 >> 3));
                cx.fx->st_w[r] = __popc(hb) & 1;
            }
        }
    } else if (r < na) {
        const int p = cx.fx->alive_list[r];
        const R* in = cx.llr(p, d - 1);
        uint32_t* row = cx.row(p);
        uint32_t bits = 0;
        if (is_g) {
            const int pos = lb - m; // the left sibling's decisions
            bits = row[pos >> 5] >> (pos & 31);
        }
        M v[MF];
        uint32_t hb = 0;
#pragma unroll
        for (int i = 0; i < MF; ++i) {
            if (i < m) {
                const R a = in[i], b = in[m + i];
                v[i] = A::val(is_g ? A::g(a, b, (bits >> i) & 1u) : A::f(a, b));
                hb |= uint32_t(v[i] < M(0)) << i;
            }
        }
        const uint32_t mk = (1u << m) - 1u;
        uint32_t* w = row + (lb >> 5);
        const int sh = lb & 31;
        if (code == OP_FROZEN) { // list_frozen: sequential penalty, zero span
#pragma unroll
            for (int i = 0; i < MF; ++i)
                if (i < m && v[i] < M(0)) pen = A::sat(pen, -v[i]);
            *w &= ~(mk << sh);
        } else if (code == OP_INFO) {
            cx.fx->st_a1[r] = mbits<M>(v[0]);
        } else if (code == OP_REP) { // rep_fold (halving) + rep_pen (sequential)
            M x[MF];
#pragma unroll
            for (int i = 0; i < MF; ++i) x[i] = i < m ? v[i] : M(0);
#pragma unroll
            for (int len = MF; len > 1; len >>= 1)
                if (len <= m)
#pragma unroll
                    for (int i = 0; i < len / 2; ++i) x[i] = A::sat(x[i], x[i + len / 2]);
            const bool wn = x[0] < M(0);
            M pw = M(0);
#pragma unroll
            for (int i = 0; i < MF; ++i)
                if (i < m && (wn ? (v[i] > M(0)) : (v[i] < M(0)))) pw = A::sat(pw, A::mag(v[i]));
            cx.fx->st_w[r] = wn;
            cx.fx->st_a1[r] = mbits<M>(x[0]);
            cx.fx->st_a2[r] = mbits<M>(pw);
        } else { // R1 / SPC: hard decisions, two smallest (value, index), parity
            K k1 = A::kKeyMax, k2 = A::kKeyMax;
#pragma unroll
            for (int i = 0; i < MF; ++i) {
                if (i < m) {
                    const K kv = A::make_key(A::mag(v[i]), i);
                    const K n1 = kmin(k1, kv);
                    k2 = kmin(k2, kmax(k1, kv));
                    k1 = n1;
                }
            }
            *w = (*w & ~(mk << sh)) | (hb << sh);
            cx.fx->st_i1[r] = A::key_idx(k1);
            cx.fx->st_i2[r] = A::key_idx(k2);
            cx.fx->st_a1[r] = mbits<M>(A::key_val(k1));
            cx.fx->st_a2[r] = mbits<M>(A::key_val(k2));
            cx.fx->st_w[r] = __popc(hb) & 1;
        }
    }
    __syncwarp();
    if (code == OP_FROZEN) {
        const M pr = cx.sw.shfl(pen, cx.myrank & (SW - 1));
        if (cx.is_alive()) cx.metric = A::sat(cx.metric, pr);
        cx.normalize();
    }
}

// A forking node: per-path statistics, candidates in emission order
// (ascending slot, then candidate number, list_decoder.hpp:240-333), one
// shared fork_apply, normalisation.  C = candidates per lane, fixed per
// kernel instantiation (4L <= SW*C).
template <typename R, int SW, int C, int MAXW, bool VLEAF = false, bool BF = false>
__device__ void list_fork_node(Ctx<R, SW>& cx, int code, int d, int m, int lb, int na, bool fused) {
    using A = Arith<R>;
    using M = typename A::M;
    constexpr int MF = sizeof(R) == 1 ? kFuseMaxI8 : kFuseMaxF32;
    if (fused && m <= MF) {
        // statistics already taken by fused_leaf
    } else if (code == OP_R1 || code == OP_SPC) {
        r1spc_stats<VLEAF, BF>(cx, d, m, lb, na, BF && fused);
    } else if (code == OP_REP) {
        rep_fold<VLEAF>(cx, d, m, na);
        rep_pen<VLEAF>(cx, d, m, na);
    } else { // INFO: the leaf LLR of rank r -> st_a1[r]
        if (cx.lane < na) cx.fx->st_a1[cx.lane] = mbits<M>(A::val(cx.llr(cx.fx->alive_list[cx.lane], d)[0]));
        __syncwarp();
    }
    const int lgb = code == OP_R1 ? 2 : 1; // candidates per path: 4 or 2
    M cm[C];
    int cs[C], cax[C]; // source slot, decision (a | b << 16): float kernels only
    if constexpr (A::kFixed) {
        // metrics only (fork_apply decodes the kept candidates' decisions)
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int i = cx.lane + SW * k, r = min(i >> lgb, na - 1), j = i & ((1 << lgb) - 1);
            const M base = cx.sw.shfl(cx.metric, int(cx.fx->alive_list[r]));
            const M a1 = mfrom<M>(cx.fx->st_a1[r]);
            if (code == OP_INFO) { // list_decoder.hpp:240-252
                cm[k] = A::sat(base, (j == 0) == (a1 < M(0)) ? A::mag(a1) : M(0));
            } else if (code == OP_REP) { // :276-305, preferred bit first
                const M pen_w = mfrom<M>(cx.fx->st_a2[r]);
                cm[k] = A::sat(base, j == 0 ? pen_w : A::sat(pen_w, A::mag(a1)));
            } else { // R1 :254-274, SPC :307-333 (jj as in fork_apply)
                const M a2 = mfrom<M>(cx.fx->st_a2[r]);
                const int jj = code == OP_R1 ? j : (cx.fx->st_w[r] ? j + 1 : j * 3);
                cm[k] = jj == 0 ? base : A::sat(base, jj == 1 ? a1 : jj == 2 ? a2 : A::sat(a1, a2));
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int i = cx.lane + SW * k, r = min(i >> lgb, na - 1), j = i & ((1 << lgb) - 1);
            const int p = cx.fx->alive_list[r];
            const M base = cx.sw.shfl(cx.metric, p);
            cs[k] = p;
            if (code == OP_INFO) { // list_decoder.hpp:240-252
                const M v = mfrom<M>(cx.fx->st_a1[r]);
                cm[k] = A::sat(base, (j == 0) == (v < M(0)) ? A::mag(v) : M(0));
                cax[k] = pack_aux(j, -1);
            } else if (code == OP_REP) { // :276-305, preferred bit first
                const int w = cx.fx->st_w[r];
                const M pen_w = mfrom<M>(cx.fx->st_a2[r]);
                cm[k] = j == 0 ? A::sat(base, pen_w)
                               : A::sat(base, A::sat(pen_w, A::mag(mfrom<M>(cx.fx->st_a1[r]))));
                cax[k] = pack_aux(w ^ j, -1);
            } else {
                const int i1 = cx.fx->st_i1[r], i2 = cx.fx->st_i2[r];
                const M a1 = mfrom<M>(cx.fx->st_a1[r]), a2 = mfrom<M>(cx.fx->st_a2[r]);
                const int jj = code == OP_R1 ? j : (cx.fx->st_w[r] ? j + 1 : j * 3);
                cm[k] = jj == 0 ? base : jj == 1 ? A::sat(base, a1) : jj == 2 ? A::sat(base, a2)
                                                                     : A::sat(base, A::sat(a1, a2));
                cax[k] = jj == 0 ? pack_aux(-1, -1) : jj == 1 ? pack_aux(i1, -1)
                                                    : jj == 2 ? pack_aux(i2, -1) : pack_aux(i1, i2);
            }
        }
    }
    // candidates of one path form a sorted run except at information leaves
    fork_apply<R, SW, C, MAXW>(cx, cm, cs, cax, na << lgb, code, lgb, lb, code == OP_INFO ? 1 : m,
                               code == OP_INFO ? 0 : lgb);
}

// ---- CRC syndrome of a decided codeword row ----------------
template <int SW>
__device__ uint64_t row_syndrome(const DevCode& C, const uint32_t* row, int lane) {
    uint64_t syn = 0;
    const int nbytes = (C.n + 7) >> 3;
    #pragma unroll 1
    for (int j = lane; j < nbytes; j += SW) {
        const uint32_t byte = (row[j >> 2] >> ((j & 3) * 8)) & 0xffu;
        syn ^= __ldg(C.crc_tab + (size_t(j) << 8) + byte);
    }
#pragma unroll
    for (int off = SW / 2; off >= 1; off >>= 1) syn ^= shfl_xor_k(syn, off);
    return syn ^ C.crc_c0;
}

// payload (MSB-first bytes of the open positions) + optional codeword
template <int SW>
__device__ void write_outputs(const LaunchParams& P, const DevCode& C, const uint32_t* row,
                              int frame, int lane) {
    uint8_t* pay = P.payload + int64_t(frame) * P.payload_stride;
    const int pb = (C.psize + 7) >> 3;
    #pragma unroll 1
    for (int q = lane; q < pb; q += SW) {
        uint32_t byte = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int j = 8 * q + b;
            if (j < C.psize) {
                const int pos = C.info_pos[j];
                byte |= ((row[pos >> 5] >> (pos & 31)) & 1u) << (7 - b);
            }
        }
        pay[q] = uint8_t(byte);
    }
    if (P.codeword) {
        uint8_t* cw = P.codeword + int64_t(frame) * P.codeword_stride;
        const int cb = (C.n + 7) >> 3;
        #pragma unroll 1
        for (int q = lane; q < cb; q += SW) {
            uint32_t byte = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int pos = 8 * q + b;
                if (pos < C.n) byte |= ((row[pos >> 5] >> (pos & 31)) & 1u) << (7 - b);
            }
            cw[q] = uint8_t(byte);
        }
    }
}

template <bool TEAM = false, typename R, int SW>
__device__ void setup_ctx(Ctx<R, SW>& cx, const LaunchParams& P, const DevCode& C,
                          unsigned char* sm, unsigned char* gs, int frame, const Sub<SW>& sw,
                          int l, int segmax) {
    cx.sw = sw;
    cx.lane = sw.lane;
    cx.n = C.n;
    cx.l = l;
    cx.lmask = l >= 32 ? FULL : ((1u << l) - 1u);
    if constexpr (sizeof(R) == 4 && SW == 32) cx.discard = P.list_discard != 0;
    cx.chan = frame_llr<R>(P, frame);
    cx.fx = reinterpret_cast<FixedS<SW>*>(sm);
    if constexpr (sizeof(R) == 4)
        if (cx.lane == 0) cx.fx->pool[0] = reinterpret_cast<uint64_t>(cx.chan);
    const LayoutQ q0 = layout_query(C.n, l, int(sizeof(R)), segmax, 0, SW);
    cx.ps = reinterpret_cast<uint32_t*>(sm + q0.psum_off);
    cx.rw = q0.rw;
    // (constants outside team kernels: the team code folds away)
    cx.team = TEAM ? P.team : 1;
    cx.tt0 = cx.lane;
    cx.tstride = TEAM ? 32 * P.team : SW;
    #pragma unroll 1
    for (int d = cx.lane + 1; d <= C.stages; d += SW) {
        const LayoutQ q = layout_query(C.n, l, int(sizeof(R)), segmax, d, SW);
        cx.fx->pool[d] = reinterpret_cast<uint64_t>((q.pool_in_smem ? sm : gs) + q.pool_off);
    }
    if (cx.lane == 0) *reinterpret_cast<uint4*>(cx.bix()) = make_uint4(0, 0, 0, 0);
    cx.metric = typename Arith<R>::M(0);
    __syncwarp();
    cx.set_alive(1u);
}

// ---- one frame, list decoding at list size P.l --------------------------
// Kernel variant KV (1..6) <-> list size 1, 2, 4, 8, 16, 32 on sub-warps of
// SW lanes: candidates per lane CW = ceil(4L / SW) and the widest ranking
// network MAXW = min(SW, 4L).
__host__ __device__ constexpr int kv_l(int kv) { return 1 << (kv - 1); }
// Float kernels that decode a chained schedule (DevCode::sched_listv[2..3]):
// those with register room for the chained loop's four loads in flight --
// the sub-warp kernels (L <= 8 at 2 / 4 frames per warp) and L = 32 (128
// registers).  The 32-lane kernels at L <= 16 spill with it (cfg4 L=16
// -1.5%) and keep the plain schedule and code.
#ifndef PLB_CHAIN_SUBWARP
#define PLB_CHAIN_SUBWARP 1
#endif
#ifndef PLB_BIGFUSE_SUBWARP
#define PLB_BIGFUSE_SUBWARP 0
#endif
#ifndef PLB_CHAIN_KERNELS
#define PLB_CHAIN_KERNELS 1
#endif
// (ALT: the second instantiation of the float sub-warp kernels, big fused
// leaves instead of chained F ops -- the better of the two for codes of
// N <= 1024, whose depth pools are shared-memory resident: N = 1024 rate
// 0.84 L = 8 / 4 +8% / +6%, N = 256 +8%, while N = 2048 / 4096 lose 8% / 21%
// without the chained ops, `profiles/r02b_sweeps.log` nsweep; host.cu picks
// per handle, LaunchParams::list_alt)
template <typename R, int KV, int SW, bool ALT = false>
constexpr bool kChainKernel = PLB_CHAIN_KERNELS && sizeof(R) == 4 && (KV == 6 || (PLB_CHAIN_SUBWARP && SW < 32 && !ALT));
// Kernels whose statistics pass can form a big rate-1 / single-parity leaf
// from its parent's segment (r1spc_stats gf): all but the float sub-warp
// kernels, which lose 7-10% to the extra code at their 64-register cap
// (cfg0 20.1 -> 19.7 with it, 18.1 with the code present and unused).
#ifndef PLB_BIGFUSE_KERNELS
#define PLB_BIGFUSE_KERNELS 1
#endif
#ifndef PLB_SCHEDX
#define PLB_SCHEDX 1
#endif
template <typename R, int KV, int SW, bool ALT = false>
constexpr bool kBigFuseKernel = PLB_BIGFUSE_KERNELS && (sizeof(R) != 4 || SW == 32 || PLB_BIGFUSE_SUBWARP || ALT);
// ... and the schedule variant (DevCode::sched_listv) a kernel reads
template <typename R, int KV, int SW, bool ALT = false>
constexpr int kSchedVariant = (kChainKernel<R, KV, SW, ALT> ? 2 : 0) + (kBigFuseKernel<R, KV, SW, ALT> ? 0 : 1);
__host__ __device__ constexpr int kv_cw(int kv, int sw) { return (4 * kv_l(kv) + sw - 1) / sw; }
__host__ __device__ constexpr int kv_maxw(int kv, int sw) { return 4 * kv_l(kv) < sw ? 4 * kv_l(kv) : sw; }

template <typename R, int KV, int SW, bool TEAM, bool ALT = false>
__device__ void list_frame(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                           unsigned char* gs, int frame, bool active, const Sub<SW>& sw, int segmax,
                           int oidx) {
    using A = Arith<R>;
    using M = typename A::M;
    constexpr int CW = kv_cw(KV, SW), MAXW = kv_maxw(KV, SW);
    // (the start time goes to memory, not a register live across the op loop:
    // lat = end - start in wrapping 32-bit ns)
    if (P.lat_ns && active && sw.lane == 0) P.lat_ns[frame] -= uint32_t(gtimer());
    Ctx<R, SW> cx;
    setup_ctx<TEAM>(cx, P, C, sm, gs, frame, sw, kv_l(KV), segmax); // P.l == kv_l(KV)
    const int lane = cx.lane;
    constexpr bool CHK = kChainKernel<R, KV, SW, ALT>;
    constexpr bool BFK = kBigFuseKernel<R, KV, SW, ALT>;
    // the fixed-point sub-warp kernels (the throughput passes) read the
    // host-decoded schedule: one 16-byte load per op instead of the field
    // shifts and masks, cfg1 19.31 -> 19.68 Gb/s.  The float kernels at their
    // 64-register cap lose 1-6% with it, and the 32-lane kernels run the
    // latency-bound small passes of the FA ladder, where the 4x larger
    // schedule misses the L1 more often (rungs 3-5% slower): both keep the
    // packed words (profiles/r02c_ab_schedx_*.log)
    constexpr bool SX = PLB_SCHEDX && sizeof(R) != 4 && SW < 32;
    constexpr int SV = kSchedVariant<R, KV, SW, ALT>;
    const uint32_t* sched = C.sched_listv[SV];
    const uint4* schedx = C.sched_listx[SV];
    const int nops = C.nops_listv[SV];
    #pragma unroll 1
    for (int oi = 0; oi < nops; ++oi) {
#ifdef PLB_OPTIME
        const long long ot0 = clock64();
#endif
        uint32_t op;
        int d, m, lb;
        if constexpr (SX) {
            const uint4 ox = __ldg(schedx + oi);
            op = ox.x;
            d = int(ox.y);
            m = int(ox.z);
            lb = int(ox.w);
        } else {
            op = __ldg(sched + oi);
            d = op_depth(op);
            m = 1 << op_logm(op);
            lb = op_lb(op);
        }
        const int code = op_code(op);
        const int na = __popc(cx.alive);
        const bool fused = (op & kOpFused) != 0;
        if (fused && m <= (sizeof(R) == 1 ? kFuseMaxI8 : kFuseMaxF32)) fused_leaf(cx, code, d, m, lb, na, (op & kOpFusedG) != 0);
        if (code <= OP_G) op_fg<(sizeof(R) == 4 && KV >= PLB_FG_UNROLL_MINKV) ? PLB_FG_UNROLL : 1, CHK>(cx, d, m, lb, na, code == OP_G, CHK && (op & kOpChain) != 0);
        else if (code == OP_H) op_h(cx, m, lb, na);
        else if (code == OP_FROZEN) {
            if (!fused) list_frozen<(sizeof(R) == 4 && KV >= PLB_VLEAF_MINKV)>(cx, d, m, lb, na);
        } else {
            list_fork_node<R, SW, CW, MAXW, (sizeof(R) == 4 && KV >= PLB_VLEAF_MINKV), BFK>(cx, code, d, m, lb, na, fused);
        }
#ifdef PLB_OPTIME
        // (profiling build only) cycles per op kind of the first frame
        __syncwarp();
        if (frame == 0 && lane == 0) {
            const int slot = code * 2 + (fused ? 1 : 0);
            atomicAdd(&g_optime[slot], (unsigned long long)(clock64() - ot0));
            atomicAdd(&g_optime[32 + slot], 1ull);
        }
#endif
    }
    // finish (list_decoder.hpp:457-502): stable order by (metric, slot)
    using K = typename A::Key;
    const K okey = cx.is_alive() ? A::make_key(cx.metric, lane) : A::kKeyMax;
    K best = okey;
#pragma unroll
    for (int off = SW / 2; off >= 1; off >>= 1) best = kmin(best, shfl_xor_k(best, off));
    int pick = A::key_idx(best);
    int crc_ok = 0;
    if (C.crc_width > 0) {
        if (SW == 32) {
            if (row_syndrome<SW>(C, cx.row(pick), lane) == 0) {
                crc_ok = 1;
            } else if (P.select_by_crc) {
                unsigned passm = 0;
                #pragma unroll 1
                for (unsigned mm = cx.alive & ~(1u << pick); mm; mm &= mm - 1) {
                    const int s = __ffs(mm) - 1;
                    if (row_syndrome<SW>(C, cx.row(s), lane) == 0) passm |= 1u << s;
                }
                if (passm) {
                    K bk = ((passm >> lane) & 1u) ? okey : A::kKeyMax;
#pragma unroll
                    for (int off = SW / 2; off >= 1; off >>= 1) bk = kmin(bk, shfl_xor_k(bk, off));
                    pick = A::key_idx(bk);
                    crc_ok = 1;
                }
            }
        } else {
            // the sub-warps of a warp hold different frames, so every
            // collective runs outside data-dependent branches: check every
            // slot (L <= 8 here), rank the passing ones, then pick as the
            // reference does
            unsigned passm = 0;
            #pragma unroll 1
            for (int s = 0; s < cx.l; ++s)
                if (row_syndrome<SW>(C, cx.row(s), lane) == 0 && ((cx.alive >> s) & 1u)) passm |= 1u << s;
            K bk = ((passm >> lane) & 1u) ? okey : A::kKeyMax;
#pragma unroll
            for (int off = SW / 2; off >= 1; off >>= 1) bk = kmin(bk, shfl_xor_k(bk, off));
            if ((passm >> pick) & 1u) {
                crc_ok = 1;
            } else if (P.select_by_crc && passm) {
                pick = A::key_idx(bk);
                crc_ok = 1;
            }
        }
    }
    const M pm = cx.sw.shfl(cx.metric, pick);
    if (active) {
        // (speculative rungs of the FA ladder write to a staging area indexed
        // by the frame's position in the pass's list, LaunchParams::out_by_idx)
        const int of = P.out_by_idx ? oidx : frame;
        write_outputs<SW>(P, C, cx.row(pick), of, lane);
        if (P.path_alive) {
            // ListDecoder<R>::alive / metric_of (list_decoder.hpp:91-93): the
            // final list, logical slot s in lane s
            if (lane < cx.l) P.path_metric[int64_t(frame) * P.path_stride + lane] = A::to_float(cx.metric);
            if (lane == 0) P.path_alive[frame] = cx.alive;
        }
        if (lane == 0) {
            if (P.crc_ok) P.crc_ok[of] = uint8_t(crc_ok);
            if (P.esc) P.esc[of] = uint8_t(P.esc_level);
            if (P.metric) P.metric[of] = A::to_float(pm);
            if (P.fail_list && C.crc_width > 0 && !crc_ok) P.fail_list[atomicAdd(P.fail_count, 1)] = frame;
            if (P.lat_ns) P.lat_ns[frame] += uint32_t(gtimer());
        }
    }
    __syncwarp();
}

// SC over a whole subtree of size m <= 32 (OP_SCSUB): lane i owns position
// lb + i; the LLRs of the node on the current root-to-leaf path at level k
// live in scv[k][lane] (a level-k node covering [p, p+s) keeps its values in
// lanes [p, p+s)), partial sums in one register bit per lane.  Visits the
// leaves in order exactly like sc_decoder.hpp:58-112: G into the right child
// whose subtree starts at leaf j, F down to the leaf, the hard (or frozen)
// decision, then the h combines of every node that leaf completes.
template <typename R>
__device__ void sc_sub(Ctx<R, 32>& cx, int d, int m, int lb, uint32_t fmask) {
    using A = Arith<R>;
    using M = typename A::M;
    const int lane = cx.lane;
    const int lgm = __ffs(m) - 1;
    M* V = reinterpret_cast<M*>(cx.fx->scv);
    const M v0 = lane < m ? A::val(cx.llr(0, d)[lane]) : M(0);
    V[lane] = v0;
    __syncwarp();
    uint32_t x = 0;
    int j = 0, k = 0; // next leaf; level of the node entered at leaf j
    M vk = v0;        // V[k][lane]
    #pragma unroll 1
    while (true) {
        // Descend from the node at level k covering [j, j + s).  Two exact
        // sub-node shortcuts: all frozen -> codeword 0; all information with
        // no zero input -> hard decisions (see the rate-1 argument in
        // host.cu emit_sc); otherwise F into the left child.
        int last, done; // last leaf and size of the node just completed
        #pragma unroll 1
        while (true) {
            const int s = m >> k;
            const uint32_t mk = s >= 32 ? FULL : ((1u << s) - 1u);
            const uint32_t fm = (fmask >> j) & mk;
            const bool mine = lane >= j && lane < j + s;
            done = s;
            last = j + s - 1;
            if (fm == mk) {
                if (mine) x = 0u;
                break;
            }
            if (fm == 0u && !__any_sync(FULL, mine && vk == M(0))) {
                if (mine) x = uint32_t(vk < M(0)); // the node's codeword
                break;
            }
            // (s == 1 is always one of the two cases above or a zero-LLR info
            // leaf, whose hard decision is 0)
            if (s == 1) {
                if (mine) x = 0u;
                break;
            }
            const int h = s >> 1;
            const M b = __shfl_down_sync(FULL, vk, h);
            const M fv = M(A::f(R(vk), R(b)));
            if (lane >= j && lane < j + h && k < 4) V[(k + 1) * 32 + lane] = fv;
            vk = fv;
            ++k;
            __syncwarp();
        }
        // h combines of every enclosing node completed by leaf `last`
        #pragma unroll 1
        for (int s = 2 * done; s <= m && ((last + 1) & (s - 1)) == 0; s <<= 1) {
            const int h = s >> 1;
            const uint32_t o = __shfl_down_sync(FULL, x, h);
            if (lane >= last + 1 - s && lane < last + 1 - h) x ^= o;
        }
        j = last + 1;
        if (j >= m) break;
        // G into the right child that starts at leaf j
        const int kk = lgm - __ffs(j);
        const int h = 1 << (__ffs(j) - 1);
        const M pv = V[kk * 32 + lane];
        const M a = __shfl_up_sync(FULL, pv, h);
        const uint32_t xb = __shfl_up_sync(FULL, x, h);
        const M gv = M(A::g(R(a), R(pv), xb));
        if (lane >= j && lane < j + h && kk < 4) V[(kk + 1) * 32 + lane] = gv;
        vk = gv;
        k = kk + 1;
        __syncwarp();
    }
    const uint32_t bits = __ballot_sync(FULL, lane < m && x);
    if (lane == 0) {
        const uint32_t mk = m >= 32 ? FULL : ((1u << m) - 1u);
        uint32_t* w = cx.row(0) + (lb >> 5);
        *w = (*w & ~(mk << (lb & 31))) | ((bits & mk) << (lb & 31));
    }
    __syncwarp();
}

// ---- one frame, successive cancellation (sc_decoder.hpp:37-125) ---------
template <typename R>
__device__ void sc_frame(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                         unsigned char* gs, int frame, const Sub<32>& sw) {
    using A = Arith<R>;
    using M = typename A::M;
    if (P.lat_ns && sw.lane == 0) P.lat_ns[frame] -= uint32_t(gtimer());
    Ctx<R, 32> cx;
    setup_ctx(cx, P, C, sm, gs, frame, sw, 1, P.seg_smem_max);
    const int lane = cx.lane;
    uint32_t* row = cx.row(0);
    const uint32_t* sched = C.sched_sc;
    const int nops = C.nops_sc;
    #pragma unroll 1
    for (int oi = 0; oi < nops; ++oi) {
        const uint32_t op = __ldg(sched + oi);
        const int code = op_code(op), d = op_depth(op), m = 1 << op_logm(op), lb = op_lb(op);
        switch (code) {
        case OP_F:
        case OP_G: op_fg(cx, d, m, lb, 1, code == OP_G); break;
        case OP_H: op_h(cx, m, lb, 1); break;
        case OP_FROZEN: span_fill<32>(row, lb, m, 0, lane); __syncwarp(); break;
        case OP_INFO:
            if (lane == 0) span_fill_lane(row, lb, 1, A::val(cx.llr(0, d)[0]) < M(0));
            __syncwarp();
            break;
        case OP_REP: {
            rep_fold(cx, d, m, 1);
            const int bit = mfrom<M>(cx.fx->st_a1[0]) < M(0);
            span_fill<32>(row, lb, m, bit, lane);
            __syncwarp();
            break;
        }
        case OP_SCSUB: sc_sub(cx, d, m, lb, __ldg(sched + ++oi)); break;
        case OP_R1SC: {
            const int skip = int(__ldg(sched + ++oi));
            const R* L = cx.llr(0, d);
            bool zero = false;
            #pragma unroll 1
            for (int i = lane; i < m; i += 32) zero |= A::val(L[i]) == M(0);
            if (__any_sync(FULL, zero)) break; // run the expanded recursion
            if (m >= 32) {
                #pragma unroll 1
                for (int w = 0; w < (m >> 5); ++w) {
                    const uint32_t hb = __ballot_sync(FULL, A::val(L[(w << 5) + lane]) < M(0));
                    if (lane == 0) row[(lb >> 5) + w] = hb;
                }
            } else {
                const uint32_t hb = __ballot_sync(FULL, lane < m && A::val(L[lane]) < M(0));
                if (lane == 0) {
                    const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
                    row[lb >> 5] = (row[lb >> 5] & ~mk) | ((hb << (lb & 31)) & mk);
                }
            }
            __syncwarp();
            oi += skip;
            break;
        }
        default: break;
        }
    }
    int crc_ok = 0;
    if (C.crc_width > 0) crc_ok = row_syndrome<32>(C, row, lane) == 0;
    write_outputs<32>(P, C, row, frame, lane);
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[frame] = uint8_t(crc_ok);
        if (P.esc) P.esc[frame] = 1;
        if (P.metric) P.metric[frame] = 0.0f; // DecodeResult default (decode_result.hpp:12)
        if (P.fail_list && C.crc_width > 0 && !crc_ok) P.fail_list[atomicAdd(P.fail_count, 1)] = frame;
        if (P.lat_ns) P.lat_ns[frame] += uint32_t(gtimer());
    }
    __syncwarp();
}

// A helper warp of a team (warps 1..team-1 of a block that decodes one
// frame, large list sizes): walks the same schedule as the control warp
// (warp 0, list_frame) and joins only the element ops (F/G, H), between the
// same two block barriers op_fg / op_h place around them.  All path
// bookkeeping stays with warp 0; the helpers read the alive list it
// publishes in shared memory.
template <typename R, int KV>
__device__ void team_helper(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                            int frame, int wib) {
    Ctx<R, 32> cx;
    cx.lane = threadIdx.x & 31;
    cx.n = C.n;
    cx.l = P.l;
    cx.chan = frame_llr<R>(P, frame);
    cx.fx = reinterpret_cast<FixedS<32>*>(sm);
    const LayoutQ q0 = layout_query(C.n, P.l, int(sizeof(R)), P.seg_smem_max, 0, 32);
    cx.ps = reinterpret_cast<uint32_t*>(sm + q0.psum_off);
    cx.rw = q0.rw;
    cx.team = P.team;
    cx.tt0 = wib * 32 + cx.lane;
    cx.tstride = 32 * P.team;
    constexpr bool CHK = kChainKernel<R, KV, 32>;
    const uint32_t* sched = C.sched_listv[kSchedVariant<R, KV, 32>];
    const int nops = C.nops_listv[kSchedVariant<R, KV, 32>];
    #pragma unroll 1
    for (int oi = 0; oi < nops; ++oi) {
        const uint32_t op = __ldg(sched + oi);
        const int code = op_code(op);
        if (code > OP_H) continue; // control ops: warp 0 alone
        const int d = op_depth(op), m = 1 << op_logm(op), lb = op_lb(op);
        __syncthreads();
        const int na = __popc(cx.fx->alive_w);
        if (code == OP_H) h_elems(cx, m, lb, na);
        else fg_elems<1, CHK>(cx, d, m, lb, na, code == OP_G, CHK && (op & kOpChain) != 0);
        __syncthreads();
    }
}

#ifndef PLB_MINBLOCKS
#define PLB_MINBLOCKS 8
#endif
// register budget of the L = 32 kernels, whose occupancy shared memory
// limits anyway (minimum resident 256-thread blocks: 2 -> up to 128
// registers; measured cfg4 L=32 1.17 -> 1.24 Gb/s.  L = 16 is register-
// limited and keeps 64: 3.15 vs 2.79 Gb/s with 128)
#ifndef PLB_MINBLOCKS_BIGL
#define PLB_MINBLOCKS_BIGL 2
#endif

// KV = 0: SC pass; KV = 1..6: list pass at L = 1, 2, 4, 8, 16, 32.  A warp
// holds 32/SW frames (SW < 32 only for single-code batches).
template <typename R, int KV, int SW, bool TEAM = false, bool ALT = false>
__global__ void __launch_bounds__(kMaxTeam * 32, KV >= 6 ? PLB_MINBLOCKS_BIGL
                                                         : PLB_MINBLOCKS * kMaxWarpsPerBlock / kMaxTeam)
decode_kernel(const LaunchParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int FPW = 32 / SW;
    const int wl = threadIdx.x & 31, wib = threadIdx.x >> 5;
    Sub<SW> sw;
    sw.id = wl / SW;
    sw.base = sw.id * SW;
    sw.lane = wl - sw.base;
    if constexpr (TEAM && KV > 0 && SW == 32) {
        {
            // one frame per block: warp 0 controls, the others help
            __shared__ long long s_claim;
            const long long count = P.frame_list ? (long long)(*P.frame_count) : (long long)P.nframes;
            if (count <= P.count_lo || count > P.count_hi) return;
            unsigned char* gs = static_cast<unsigned char*>(P.gscratch) + int64_t(blockIdx.x) * P.gscratch_per_frame;
            for (;;) {
                if (threadIdx.x == 0) s_claim = (long long)atomicAdd(P.work, 1ull);
                __syncthreads();
                const long long idx = s_claim;
                __syncthreads(); // all read before the next claim overwrites
                if (idx >= count) break;
                const int frame = P.frame_list ? P.frame_list[idx] : int(idx);
                const int cid = P.code_id ? P.code_id[frame] : 0;
                const DevCode C = P.codes[cid];
                if (wib == 0) list_frame<R, KV, 32, true>(P, C, smem_raw, gs, frame, true, sw, P.seg_smem_max, int(idx));
                else team_helper<R, KV>(P, C, smem_raw, frame, wib);
            }
            return;
        }
    }
    const long long count = P.frame_list ? (long long)(*P.frame_count) : (long long)P.nframes;
    if (count <= P.count_lo || count > P.count_hi) return;
    // Solo mode for passes with few frames (the upper FA rungs: a few
    // hundred frames or less, where a frame's latency, not the throughput,
    // sets the pass time): warp 0 of each block decodes with the shared
    // memory of the whole block, so more depth segments stay out of the L2.
    const bool solo = P.seg_solo > 0 && count <= P.solo_max;
    if (solo && wib != 0) return;
    const int64_t gw = solo ? int64_t(blockIdx.x) : int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
    unsigned char* sm = solo ? smem_raw + sw.id * (P.smem_per_warp * P.wpb / FPW)
                             : smem_raw + wib * P.smem_per_warp + sw.id * P.smem_per_frame;
    unsigned char* gs = static_cast<unsigned char*>(P.gscratch) + (gw * FPW + sw.id) * P.gscratch_per_frame;
    const int segmax = solo ? P.seg_solo : P.seg_smem_max;
    for (;;) {
        unsigned long long i0 = 0;
        if (wl == 0) i0 = atomicAdd(P.work, (unsigned long long)FPW);
        const long long idx0 = (long long)__shfl_sync(FULL, i0, 0);
        if (idx0 >= count) break;
        const long long mine = idx0 + sw.id;
        const bool active = mine < count;
        const long long idx = active ? mine : idx0; // idle sub-warps shadow frame idx0
        const int frame = P.frame_list ? P.frame_list[idx] : int(idx);
        const int cid = P.code_id ? P.code_id[frame] : 0;
        if constexpr (FPW > 1) {
            // The sub-warps run in lockstep only on one code.  Multi-code
            // batches arrive bucketed by code (code_bucket), so a warp's
            // frames straddle two codes only at bucket edges: then the warp
            // decodes them one after the other, every sub-warp on the same
            // frame and sub-warp 0 writing.
            const bool same = __all_sync(FULL, cid == __shfl_sync(FULL, cid, 0));
            #pragma unroll 1
            for (int j = 0; j < (same ? 1 : FPW); ++j) {
                const int fj = same ? frame : __shfl_sync(FULL, frame, j * SW);
                const int cj = same ? cid : __shfl_sync(FULL, cid, j * SW);
                const bool aj = same ? active : (__shfl_sync(FULL, int(active), j * SW) && sw.id == 0);
                list_frame<R, KV, SW, false, ALT>(P, P.codes[cj], sm, gs, fj, aj, sw, segmax, fj);
            }
        } else {
            const DevCode C = P.codes[cid];
            if constexpr (KV > 0) list_frame<R, KV, SW, false, ALT>(P, C, sm, gs, frame, active, sw, segmax, int(idx));
            else sc_frame<R>(P, C, sm, gs, frame, sw);
        }
    }
}

// Bucket frames by code id (counting sort; order inside a bucket is
// arbitrary): hist[c] = frames of code c, then exclusive offsets, then each
// frame takes a slot of its bucket.  Lets multi-code batches use the
// several-frames-per-warp kernels (lockstep needs one code per warp).
__global__ void code_hist_kernel(const int32_t* cid, int64_t n, int32_t* hist) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(hist + cid[i], 1);
}
__global__ void code_scan_kernel(int32_t* hist, int ncodes, int32_t* count_out, int64_t n) {
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int c = 0; c < ncodes; ++c) {
            const int32_t v = hist[c];
            hist[c] = acc;
            acc += v;
        }
        *count_out = int32_t(n);
    }
}
__global__ void code_scatter_kernel(const int32_t* cid, int64_t n, int32_t* cursor, int32_t* out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[atomicAdd(cursor + cid[i], 1)] = int32_t(i);
}

#include "lanes.cuh"

// Exhaustive check of the packed int8 f/g against the scalar kernels: every
// (a, b) pair in [-127, 127]^2, in every byte position, next to
// pseudo-random neighbours, under all 16 partial-sum patterns.
// int16 f on packed pairs against the scalar kernel: every a in
// [-32767, 32767] against 512 pseudo-random b (incl. 0, +-1, +-32767), in
// both 16-bit lanes, with swapped operands in the other lane.
__global__ void selftest16_kernel(unsigned long long* bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 65535) return;
    using A = Arith<int16_t>;
    const int a = t - 32767;
    unsigned long long nbad = 0;
    uint32_t h = 0x9e3779b9u * uint32_t(t + 1);
    for (int j = 0; j < 512; ++j) {
        h ^= h << 13;
        h ^= h >> 17;
        h ^= h << 5;
        const int b = j < 5 ? (j == 0 ? 0 : j == 1 ? 1 : j == 2 ? -1 : j == 3 ? 32767 : -32767)
                            : int(h % 65535u) - 32767;
        const uint32_t x = uint32_t(uint16_t(int16_t(a))) | (uint32_t(uint16_t(int16_t(b))) << 16);
        const uint32_t y = uint32_t(uint16_t(int16_t(b))) | (uint32_t(uint16_t(int16_t(a))) << 16);
        const uint32_t r = f_swar16(x, y);
        nbad += int16_t(r & 0xffffu) != A::f(int16_t(a), int16_t(b));
        nbad += int16_t(r >> 16) != A::f(int16_t(b), int16_t(a));
    }
    if (nbad) atomicAdd(bad, nbad);
}

__global__ void selftest_kernel(unsigned long long* bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 255 * 255) return;
    const int a = t / 255 - 127, b = t % 255 - 127;
    unsigned long long nbad = 0;
    uint32_t h = 0x9e3779b9u * uint32_t(t + 1);
    for (int pos = 0; pos < 4; ++pos) {
        uint32_t wa = 0, wb = 0;
        int8_t va[4], vb[4];
        for (int j = 0; j < 4; ++j) {
            h ^= h << 13;
            h ^= h >> 17;
            h ^= h << 5;
            va[j] = int8_t(j == pos ? a : int(h % 255u) - 127);
            vb[j] = int8_t(j == pos ? b : int((h >> 8) % 255u) - 127);
            wa |= uint32_t(uint8_t(va[j])) << (8 * j);
            wb |= uint32_t(uint8_t(vb[j])) << (8 * j);
        }
        const uint32_t fo = f_swar(wa, wb);
        for (int j = 0; j < 4; ++j)
            nbad += int8_t(fo >> (8 * j)) != Arith<int8_t>::f(va[j], vb[j]);
        for (uint32_t s4 = 0; s4 < 16; ++s4) {
            const uint32_t go = g_swar(wa, wb, s4);
            for (int j = 0; j < 4; ++j)
                nbad += int8_t(go >> (8 * j)) != Arith<int8_t>::g(va[j], vb[j], (s4 >> j) & 1u);
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

// kernel of a pass: kv = 0 (SC) or 1..6 (list at L = 1..32), frames/warp fpw
template <typename R>
void (*kernel_for(int kv, int fpw, bool team = false, bool alt = false))(LaunchParams) {
    // team kernels (one frame per block, opt-in) at L = 16 / 32
    if (team) return kv == 5 ? decode_kernel<R, 5, 32, true> : decode_kernel<R, 6, 32, true>;
    if constexpr (sizeof(R) == 4) {
        // float sub-warp kernels: the big-fused-leaf instantiation (kChainKernel)
        if (alt && fpw == 4) return kv == 1 ? decode_kernel<R, 1, 8, false, true> : decode_kernel<R, 2, 8, false, true>;
        if (alt && fpw == 2) return kv == 3 ? decode_kernel<R, 3, 16, false, true> : decode_kernel<R, 4, 16, false, true>;
    }
    // (8-lane sub-warps measured slower than 16-lane ones at L = 4 and 8)
    if (fpw == 4) return kv == 1 ? decode_kernel<R, 1, 8> : decode_kernel<R, 2, 8>;
    if (fpw == 2) return kv == 3 ? decode_kernel<R, 3, 16> : decode_kernel<R, 4, 16>;
    switch (kv) {
    case 0: return decode_kernel<R, 0, 32>;
    case 1: return decode_kernel<R, 1, 32>;
    case 2: return decode_kernel<R, 2, 32>;
    case 3: return decode_kernel<R, 3, 32>;
    case 4: return decode_kernel<R, 4, 32>;
    case 5: return decode_kernel<R, 5, 32>;
    default: return decode_kernel<R, 6, 32>;
    }
}

int kv_of(int l, bool list) {
    if (!list) return 0;
    int kv = 1;
    while ((1 << (kv - 1)) < l && kv < 6) ++kv;
    return kv;
}

template <typename R>
cudaError_t launch(const LaunchParams& p, int kv, int grid, cudaStream_t s) {
    const bool team = p.team > 1;
    const int smem = team ? p.smem_per_frame : p.smem_per_warp * p.wpb;
    auto kern = kernel_for<R>(kv, p.fpw, team, p.list_alt != 0);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, (team ? p.team : p.wpb) * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <typename R>
int occupancy(int kv, int fpw, int smem, int wpb, bool team = false) {
    auto kern = kernel_for<R>(kv, fpw, team);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, wpb * 32, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nb;
}

} // namespace

int64_t smem_bytes_per_frame(int nmax, int l, int elem_bytes, int seg_smem_max, int sw) {
    return layout_query(nmax, l, elem_bytes, seg_smem_max, 0, sw).smem_total;
}
int64_t gscratch_bytes_per_frame(int nmax, int l, int elem_bytes, int seg_smem_max) {
    return layout_query(nmax, l, elem_bytes, seg_smem_max, 0, 32).gmem_total;
}
int frames_per_warp_max(int l) { return l <= 2 ? 4 : l <= 8 ? 2 : 1; }
bool frames_per_warp_ok(int l, int fpw) { return fpw == 1 || fpw == frames_per_warp_max(l); }

// precision: 0 float, 1 int8, 2 int16 (PL_F32 / PL_I8 / PL_I16)
cudaError_t launch_sc(const LaunchParams& p, int precision, int grid, cudaStream_t s) {
    return precision == 0   ? launch<float>(p, 0, grid, s)
           : precision == 1 ? launch<int8_t>(p, 0, grid, s)
                            : launch<int16_t>(p, 0, grid, s);
}
cudaError_t launch_list(const LaunchParams& p, int precision, int grid, cudaStream_t s) {
    const int kv = kv_of(p.l, true);
    return precision == 0   ? launch<float>(p, kv, grid, s)
           : precision == 1 ? launch<int8_t>(p, kv, grid, s)
                            : launch<int16_t>(p, kv, grid, s);
}
int occupancy_sc(int precision, int smem, int wpb) {
    return precision == 0   ? occupancy<float>(0, 1, smem, wpb)
           : precision == 1 ? occupancy<int8_t>(0, 1, smem, wpb)
                            : occupancy<int16_t>(0, 1, smem, wpb);
}

int64_t lane_smem_bytes_per_warp(int nmax, int elem_bytes, int seg_smem_max, bool stage) {
    return lane_layout(nmax, elem_bytes, seg_smem_max, 0, stage).smem_total;
}
int64_t lane_gscratch_bytes_per_warp(int nmax, int elem_bytes, int seg_smem_max) {
    return lane_layout(nmax, elem_bytes, seg_smem_max, 0, false).gmem_total;
}
cudaError_t launch_sc_lanes(const LaunchParams& p, int precision, int grid, cudaStream_t s) {
    const int smem = p.smem_per_warp * p.wpb;
    void (*kern)(LaunchParams) = precision == 0   ? sc_lanes_kernel<float>
                                 : precision == 1 ? sc_lanes_kernel<int8_t>
                                                  : sc_lanes_kernel<int16_t>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, p.wpb * 32, smem, s>>>(p);
    return cudaGetLastError();
}
int occupancy_sc_lanes(int precision, int smem, int wpb) {
    void (*kern)(LaunchParams) = precision == 0   ? sc_lanes_kernel<float>
                                 : precision == 1 ? sc_lanes_kernel<int8_t>
                                                  : sc_lanes_kernel<int16_t>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, wpb * 32, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nb;
}
int occupancy_list(int precision, int l, int fpw, int smem, int wpb, bool team) {
    const int kv = kv_of(l, true);
    return precision == 0   ? occupancy<float>(kv, fpw, smem, wpb, team)
           : precision == 1 ? occupancy<int8_t>(kv, fpw, smem, wpb, team)
                            : occupancy<int16_t>(kv, fpw, smem, wpb, team);
}

// one warp per listed frame: the staged result of the lowest passing rung
// (decoders.hpp:70-82: the first list size whose CRC passes, else the last)
__global__ void commit_kernel(const CommitParams p) {
    const long long count = *p.count;
    if (count > p.count_hi) return;
    const int lane = threadIdx.x & 31;
    const long long w0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long idx = w0; idx < count; idx += nw) {
        const int frame = p.list[idx];
        int j = 0;
        while (j + 1 < p.nst && !p.st_crc[(long long)j * p.cap + idx]) ++j;
        const long long sidx = (long long)j * p.cap + idx;
        // (the bytes write_outputs wrote: those of the frame's own code)
        const DevCode& C = p.codes[p.code_id ? p.code_id[frame] : 0];
        const int pb = (C.psize + 7) >> 3, cb = (C.n + 7) >> 3;
        const uint8_t* sp = p.st_payload + sidx * p.payload_stride;
        uint8_t* dp = p.payload + (long long)frame * p.payload_stride;
        for (int q = lane; q < pb; q += 32) dp[q] = sp[q];
        if (p.codeword) {
            const uint8_t* sc = p.st_codeword + sidx * p.codeword_stride;
            uint8_t* dc = p.codeword + (long long)frame * p.codeword_stride;
            for (int q = lane; q < cb; q += 32) dc[q] = sc[q];
        }
        if (lane == 0) {
            if (p.crc_ok) p.crc_ok[frame] = p.st_crc[sidx];
            if (p.esc) p.esc[frame] = uint8_t(p.levels[j]);
            if (p.metric) p.metric[frame] = p.st_metric[sidx];
        }
    }
}
cudaError_t launch_commit(const CommitParams& p, int blocks, cudaStream_t s) {
    commit_kernel<<<blocks, 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t bucket_by_code(const int32_t* cid, int64_t n, int ncodes, int32_t* hist, int32_t* out,
                           int32_t* count_out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(hist, 0, size_t(ncodes) * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    const int grid = int(std::min<int64_t>((n + 255) / 256, 1184));
    code_hist_kernel<<<grid, 256, 0, s>>>(cid, n, hist);
    code_scan_kernel<<<1, 32, 0, s>>>(hist, ncodes, count_out, n);
    code_scatter_kernel<<<grid, 256, 0, s>>>(cid, n, hist, out);
    return cudaGetLastError();
}

#ifdef PLB_OPTIME
cudaError_t read_optime(unsigned long long* out, bool reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out, g_optime, sizeof(g_optime));
    if (e == cudaSuccess && reset) {
        static const unsigned long long z[64] = {};
        e = cudaMemcpyToSymbol(g_optime, z, sizeof(z));
    }
    return e;
}
#endif

cudaError_t kernel_selftest(unsigned long long* mismatches) {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    cudaMemset(d, 0, sizeof(unsigned long long));
    selftest_kernel<<<(255 * 255 + 255) / 256, 256>>>(d);
    selftest16_kernel<<<(65535 + 255) / 256, 256>>>(d);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(mismatches, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e;
}

} // namespace plb
