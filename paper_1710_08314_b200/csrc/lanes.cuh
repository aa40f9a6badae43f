// The frame-per-lane SC kernel (SC / SSC and the first pass of PA / FA):
// 32 frames per warp, one per lane, in lockstep over the SC schedule.
//
// A fragment of kernels.cu: included inside namespace plb::{anonymous} after
// the list decoder (it shares Arith, Vec, fg_compute and the schedules).
#pragma once

// ==== frame-per-lane SC kernel (SC / SSC and the first pass of PA / FA) ====
// A warp decodes 32 frames, one per lane, in lockstep over the SC schedule
// of their (common) code: the op sequence of SC decoding is data-independent
// except for the rate-1 shortcut, which the warp takes only when no lane has
// a zero input (the expanded recursion is exact for every lane, so running
// it for all is correct).  One warp instruction then advances 32 frames, and
// the small nodes that cost the warp-per-frame kernel a whole warp step per
// value are plain per-lane loops.  Per-warp storage, lane-interleaved so
// every access is conflict-free / coalesced:
//   * partial sums: word w of lane l at ps[w * 32 + l] (shared memory);
//   * depth-d LLR segment (n >> d values per frame): chunks of
//     V = min(VE, n >> d) values, chunk c of lane l at ((c * 32) + l) * V
//     (VE = 16 bytes of values); small segments in shared memory, large ones
//     in the warp's global scratch;
//   * depth 0 is the channel, read in place (frame-major).
// (stage_off: the area of the shared-memory depth pools, at least
// kLaneStageBytes long: the staging tile of the transposed channel reads,
// lane_fg0_tr -- every shared-memory pool is dead during an op on the channel
// when the depth-1 pool is global)
// 32 frames x TC chunks of 16 bytes (one half at a time) + the 32 frames'
// channel pointers; TC = 8 (a 128-byte line per frame), 4 for int8 (its
// pools' area is half the size: 1-byte values)
template <typename R>
constexpr int kLaneTileChunks = sizeof(R) == 1 ? 4 : 8;
template <typename R>
constexpr int kLaneStageBytes = 32 * kLaneTileChunks<R> * 16 + 32 * 8;
struct LaneQ {
    int32_t rw, psum_off, smem_total, gmem_total, pool_off, pool_in_smem, stage_off, stage_bytes;
};
__host__ __device__ inline LaneQ lane_layout(int n, int esz, int segmax, int want_d, bool stage) {
    LaneQ q{};
    int off = 16 * 8; // pool pointer table
    q.rw = n >= 32 ? n / 32 : 1;
    q.psum_off = off;
    off += 4 * q.rw * 32;
    int goff = 0;
    const int stages = ilog2(n);
    q.stage_off = off;
    #pragma unroll 1
    for (int d = 1; d <= stages; ++d) {
        const int bytes = align16((n >> d) * 32 * esz);
        if ((n >> d) <= segmax) {
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
            goff += bytes;
        }
    }
    (void)stage; // (the tile lives inside the pools' area: no growth -- three 64 KB blocks keep
                 // the SM's shared-memory carve-out at 196 KB and 60 KB of L1 for the channel)
    q.stage_bytes = off - q.stage_off;
    q.smem_total = off;
    q.gmem_total = goff;
    return q;
}

template <typename R>
struct LaneCtx {
    static constexpr int VE = 16 / int(sizeof(R));
    int lane, n;
    int segmax, keep, keep_hi; // depth segments > segmax values live in global scratch
    bool discard;     // drop dead global segments from the L2 (LaunchParams::sc_discard)
    bool il;          // the channel is lane-interleaved like the depth pools (LaunchParams::llr_il32)
    unsigned char* stage;     // staging tile of lane_fg0_tr (nullptr: off)
    const R* chan;      // this lane's frame
    uint32_t* ps;       // this lane's psum words, stride 32
    const uint64_t* pt; // pool pointer table
    __device__ __forceinline__ R* pool(int d) const { return reinterpret_cast<R*>(pt[d]); }
    // first value of chunk c at depth d (chunk = min(VE, n >> d) values)
    __device__ __forceinline__ const R* chunk(int d, int c) const {
        const int v = min(VE, n >> d);
        return d == 0 ? chan + c * (il ? 32 * v : v) : pool(d) + (c * 32 + lane) * v;
    }
    // chunk k of depth d is at base + k * stride (loop-invariant form of chunk())
    __device__ __forceinline__ const R* chunk_base(int d, int& stride) const {
        const int v = min(VE, n >> d);
        stride = d == 0 && !il ? v : 32 * v;
        return d == 0 ? chan : pool(d) + lane * v;
    }
    __device__ __forceinline__ uint32_t& word(int w) const { return ps[w * 32]; }
    // L2 eviction class of depth d's global segment: <= keep values
    // evict_last, <= keep_hi evict_normal, larger ones and the channel
    // evict_first
    __device__ __forceinline__ uint64_t policy(int d) const {
        const int seg = n >> d;
        return l2_policy(d == 0 ? 0 : seg <= keep ? 2 : seg <= keep_hi ? 1 : 0);
    }
    __device__ void fill(int lb, int m, int bit) const {
        if (m >= 32) {
            #pragma unroll 1
            for (int w = 0; w < (m >> 5); ++w) word((lb >> 5) + w) = bit ? FULL : 0u;
        } else {
            const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
            uint32_t& x = word(lb >> 5);
            x = bit ? (x | mk) : (x & ~mk);
        }
    }
};

// sign bits of the G values of a vector (value i -> bit i)
template <typename R, int G>
__device__ __forceinline__ uint32_t vec_signs(const Vec<R, G>& x) {
    uint32_t s = 0;
    if constexpr (sizeof(R) == 1 && G >= 4) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x.raw);
#pragma unroll
        for (int k = 0; k < G / 4; ++k)
            s |= ((((w[k] >> 7) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
    } else {
#pragma unroll
        for (int i = 0; i < G; ++i) s |= uint32_t(Arith<R>::val(x.v[i]) < typename Arith<R>::M(0)) << i;
    }
    return s;
}
template <typename R, int G>
__device__ __forceinline__ bool vec_has_zero(const Vec<R, G>& x) {
    if constexpr (sizeof(R) == 1 && G >= 4) {
        // a zero byte: (w - 0x01..) & ~w & 0x80.. is non-zero exactly then
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x.raw);
        uint32_t z = 0;
#pragma unroll
        for (int k = 0; k < G / 4; ++k) z |= (w[k] - 0x01010101u) & ~w[k] & 0x80808080u;
        return z != 0u;
    } else {
        bool z = false;
#pragma unroll
        for (int i = 0; i < G; ++i) z |= Arith<R>::val(x.v[i]) == typename Arith<R>::M(0);
        return z;
    }
}

#ifndef PLB_LANE_U
#define PLB_LANE_U 4 // float: chunks per trip of the plain F / G loop
#endif
#ifndef PLB_LANE_MINB
#define PLB_LANE_MINB 4 // float: resident 4-warp blocks the register budget allows
#endif
// U chunks per iteration: 2U loads in flight per lane (the pools of the
// upper depths live in global memory), U * VE <= 32 partial-sum bits.
// HIN / HOUT: the input / output depth is in global memory and takes an L2
// eviction hint (pin / pout).
// disc: the input segment is a global depth pool read for the last time (a G
// op): its L2 lines are dropped without write-back once consumed
// (discard.global.L2), so dead LLRs of 32-frame warps never reach DRAM.
template <typename R, int U, bool HIN, bool HOUT>
__device__ __forceinline__ void lane_fg_chunks(const LaneCtx<R>& c, int d, int nc, int lb, bool is_g,
                                               R* out, uint64_t pin, uint64_t pout, bool disc) {
    constexpr int VE = LaneCtx<R>::VE;
    int cs;
    const R* in = c.chunk_base(d, cs);
    const R* in_b = in + nc * cs;
    R* o = out + c.lane * VE;
    #pragma unroll 1
    for (int k = 0; k < nc; k += U) {
        Vec<R, VE> a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (HIN) {
                a[u] = vld_hint<R, VE>(in + (k + u) * cs, pin);
                b[u] = vld_hint<R, VE>(in_b + (k + u) * cs, pin);
            } else {
                a[u] = vld<R, VE>(in + (k + u) * cs);
                b[u] = vld<R, VE>(in_b + (k + u) * cs);
            }
        }
        const int pos = lb + k * VE;
        const uint32_t bits = is_g ? c.word(pos >> 5) >> (pos & 31) : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const Vec<R, VE> r = fg_compute<R, VE>(a[u], b[u], bits >> (u * VE), is_g);
            if constexpr (HOUT) vst_hint<R, VE>(o + (k + u) * 32 * VE, r, pout);
            else vst<R, VE>(o + (k + u) * 32 * VE, r);
        }
        // (the values were consumed above by every lane of the warp; chunk
        // rows are 512-byte aligned, lanes 0 / 8 / 16 / 24 start its lines)
        if (disc && (c.lane & 7) == 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                asm volatile("discard.global.L2 [%0], 128;" :: "l"(in + (k + u) * cs) : "memory");
                asm volatile("discard.global.L2 [%0], 128;" :: "l"(in_b + (k + u) * cs) : "memory");
            }
        }
    }
}
template <typename R, int U>
__device__ __forceinline__ void lane_fg_chunks_any(const LaneCtx<R>& c, int d, int nc, int lb, bool is_g,
                                                   R* out) {
    if constexpr (sizeof(R) != 4) {
        // fixed point: no hint / discard code at all (the int16 pass lost 10%
        // to the larger loop even with the hints switched off)
        lane_fg_chunks<R, U, false, false>(c, d, nc, lb, is_g, out, 0, 0, false);
        return;
    }
    // hints only on global depths (the channel is depth 0); uniform per op
    const bool gin = c.keep > 0 && (d == 0 || (c.n >> d) > c.segmax);
    const bool gout = c.keep > 0 && (c.n >> (d + 1)) > c.segmax;
    const bool disc = c.discard && is_g && d > 0 && (c.n >> d) > c.segmax;
    if (gin) {
        const uint64_t pin = c.policy(d);
        if (gout)
            lane_fg_chunks<R, U, true, true>(c, d, nc, lb, is_g, out, pin,
                                             c.policy(d + 1), disc);
        else lane_fg_chunks<R, U, true, false>(c, d, nc, lb, is_g, out, pin, 0, disc);
    } else {
        lane_fg_chunks<R, U, false, false>(c, d, nc, lb, is_g, out, 0, 0, disc);
    }
}

// A chained op (host.cu fuse_lane_chains): the F / G op at depth d and the
// J F ops below it in one sweep.  Output chunk group k of the deepest level
// needs the 2^J depth-(d+1) chunks k + t * q (q = nc >> J), i.e. 2 * 2^J
// input chunks; every level is stored (the G ops of the levels read them
// later), none is read back.  HINT: float only, L2 eviction hints on the
// global levels as in lane_fg_chunks.
template <typename R, int J, int U, bool HINT>
__device__ __forceinline__ void lane_fg_chain(const LaneCtx<R>& c, int d, int nc, int lb, bool is_g) {
    constexpr int VE = LaneCtx<R>::VE;
    constexpr int T = 1 << J;
    int cs;
    const R* in = c.chunk_base(d, cs);
    const R* in_b = in + nc * cs;
    const int q = nc >> J;
    R* o[J + 1];
    bool og[J + 1];
    uint64_t pol[J + 1];
#pragma unroll
    for (int j = 0; j <= J; ++j) {
        o[j] = c.pool(d + 1 + j) + c.lane * VE;
        og[j] = HINT && c.keep > 0 && (c.n >> (d + 1 + j)) > c.segmax;
        pol[j] = 0;
        if constexpr (HINT)
            if (og[j]) pol[j] = c.policy(d + 1 + j);
    }
    const bool gin = HINT && c.keep > 0 && (d == 0 || (c.n >> d) > c.segmax);
    uint64_t pin = 0;
    if constexpr (HINT)
        if (gin) pin = c.policy(d);
    const bool disc = HINT && c.discard && is_g && d > 0 && (c.n >> d) > c.segmax;
    #pragma unroll 1
    for (int k = 0; k < q; k += U) {
        Vec<R, VE> a[U][T], b[U][T];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int ci = k + u + t * q;
                if (HINT && gin) {
                    a[u][t] = vld_hint<R, VE>(in + ci * cs, pin);
                    b[u][t] = vld_hint<R, VE>(in_b + ci * cs, pin);
                } else {
                    a[u][t] = vld<R, VE>(in + ci * cs);
                    b[u][t] = vld<R, VE>(in_b + ci * cs);
                }
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int ci = k + u + t * q;
                const int pos = lb + ci * VE;
                const uint32_t bits = is_g ? c.word(pos >> 5) >> (pos & 31) : 0u;
                a[u][t] = fg_compute<R, VE>(a[u][t], b[u][t], bits, is_g);
                if (HINT && og[0]) vst_hint<R, VE>(o[0] + ci * 32 * VE, a[u][t], pol[0]);
                else vst<R, VE>(o[0] + ci * 32 * VE, a[u][t]);
            }
#pragma unroll
            for (int j = 1; j <= J; ++j) {
#pragma unroll
                for (int t = 0; t < (T >> j); ++t) {
                    const int ci = k + u + t * q;
                    a[u][t] = fg_compute<R, VE>(a[u][t], a[u][t + (T >> j)], 0u, false);
                    if (HINT && og[j]) vst_hint<R, VE>(o[j] + ci * 32 * VE, a[u][t], pol[j]);
                    else vst<R, VE>(o[j] + ci * 32 * VE, a[u][t]);
                }
            }
        }
        if (HINT && disc && (c.lane & 7) == 0) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const int ci = k + u + t * q;
                    asm volatile("discard.global.L2 [%0], 128;" :: "l"(in + ci * cs) : "memory");
                    asm volatile("discard.global.L2 [%0], 128;" :: "l"(in_b + ci * cs) : "memory");
                }
        }
    }
}

// The ops on the frame-major channel, transposed through shared memory: a
// lane reading its own frame touches 64 scattered bytes per trip (32 lines
// per warp load: the pass loses 12-15% to it against an interleaved
// channel, PL_LLR_INTERLEAVED32).  Here the warp reads tiles of 8 chunks
// (one 128-byte line) per frame and half -- 8 lanes per frame, 4 frames per
// load, fully coalesced -- into a swizzled staging tile (slot j of frame f
// at j ^ (f & 7): conflict-free both ways), then every lane takes its own
// frame's 8 + 8 chunks back, computes and stores to the depth-1 pool as the
// plain loop does.
// TC: chunks per frame and half of one tile (8: a 128-byte line; 4 where the
// pools' area is smaller, int8)
template <typename R, int TC>
__device__ __forceinline__ void lane_fg0_tr(const LaneCtx<R>& c, int m, int lb, bool is_g) {
    constexpr int VE = LaneCtx<R>::VE;
    constexpr bool HINT = sizeof(R) == 4;
    constexpr int FPL = 32 / TC;                  // frames per warp load
    constexpr int SH = TC == 8 ? 0 : TC == 4 ? 1 : 2; // swizzle: slot j of frame f at j ^ ((f >> SH) & (TC - 1))
    const int h = m >> 1, nc = h / VE;
    const bool hint = HINT && c.keep > 0;
    const uint64_t pin = hint ? l2_policy(0) : 0, pout = hint ? c.policy(1) : 0;
    R* const o = c.pool(1) + c.lane * VE;
    uint4* const tile = reinterpret_cast<uint4*>(c.stage);
    // (the pools' area is dead during an op on the channel: the tile, then
    // the 32 frames' channel pointers)
    uint64_t* const chans = reinterpret_cast<uint64_t*>(c.stage + 32 * TC * 16);
    const int fq = c.lane / TC, j = c.lane % TC, sw = (c.lane >> SH) & (TC - 1);
    __syncwarp();
    chans[c.lane] = reinterpret_cast<uint64_t>(c.chan);
    __syncwarp();
    #pragma unroll 1
    for (int t = 0; t < nc; t += TC) {
        // both halves' loads in flight together (2 * TC per lane), then one
        // half at a time through the tile
        Vec<R, VE> a[TC], b[TC];
#pragma unroll
        for (int i = 0; i < TC; ++i) {
            const R* src = reinterpret_cast<const R*>(chans[FPL * i + fq]) + (t + j) * VE;
            if (hint) {
                a[i] = vld_hint<R, VE>(src, pin);
                b[i] = vld_hint<R, VE>(src + h, pin);
            } else {
                a[i] = vld<R, VE>(src);
                b[i] = vld<R, VE>(src + h);
            }
        }
#pragma unroll
        for (int i = 0; i < TC; ++i) {
            const int f = FPL * i + fq;
            tile[f * TC + (j ^ ((f >> SH) & (TC - 1)))] = *reinterpret_cast<const uint4*>(&a[i].raw);
        }
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < TC; ++k2) *reinterpret_cast<uint4*>(&a[k2].raw) = tile[c.lane * TC + (k2 ^ sw)];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < TC; ++i) {
            const int f = FPL * i + fq;
            tile[f * TC + (j ^ ((f >> SH) & (TC - 1)))] = *reinterpret_cast<const uint4*>(&b[i].raw);
        }
        __syncwarp();
        uint32_t bw[4] = {0, 0, 0, 0}; // (up to 8 chunks of <= 16 values: 128 decisions)
        if (is_g) {
            const int pos = lb + t * VE;
#pragma unroll
            for (int w = 0; w < (TC * VE + 31) / 32; ++w) bw[w] = c.word((pos >> 5) + w) >> (w == 0 ? (pos & 31) : 0);
        }
#pragma unroll
        for (int k2 = 0; k2 < TC; ++k2) {
            Vec<R, VE> bb;
            *reinterpret_cast<uint4*>(&bb.raw) = tile[c.lane * TC + (k2 ^ sw)];
            const uint32_t ub = is_g ? bw[(k2 * VE) >> 5] >> ((k2 * VE) & 31) : 0u;
            const Vec<R, VE> r = fg_compute<R, VE>(a[k2], bb, ub, is_g);
            if (hint) vst_hint<R, VE>(o + (t + k2) * 32 * VE, r, pout);
            else vst<R, VE>(o + (t + k2) * 32 * VE, r);
        }
        __syncwarp();
    }
}

template <typename R>
__device__ void lane_fg(const LaneCtx<R>& c, int d, int m, int lb, bool is_g, int chain) {
    if constexpr (sizeof(R) == 4) {
        // (float only.  The fixed-point passes are issue / latency-bound, not
        // DRAM-bound: with the tile loop -- and 128 registers for it -- int8
        // went 6.7 -> 7.9 ms and int16 10.0 -> 12.6 ms; at their 80
        // registers they spill with it)
        if (d == 0 && c.stage && !chain) {
            lane_fg0_tr<R, kLaneTileChunks<R>>(c, m, lb, is_g);
            return;
        }
    }
    if constexpr (sizeof(R) == 4) if (chain) {
        // (float only: the fixed-point passes measured 5-25% slower with
        // chained levels, host.cu emits none for them)
        constexpr bool HINT = true;
        const int nc = (m >> 1) / LaneCtx<R>::VE;
        // one chained level: 4 * U loads in flight per lane
        if (nc >= 8) lane_fg_chain<R, 1, 4, HINT>(c, d, nc, lb, is_g);
        else if (nc >= 4) lane_fg_chain<R, 1, 2, HINT>(c, d, nc, lb, is_g);
        else lane_fg_chain<R, 1, 1, HINT>(c, d, nc, lb, is_g);
        return;
    }
    using A = Arith<R>;
    constexpr int VE = LaneCtx<R>::VE;
    constexpr int U = sizeof(R) == 4 ? PLB_LANE_U : (32 / VE < 4 ? 32 / VE : 4);
    const int h = m >> 1;
    R* const out = c.pool(d + 1);
    if (h >= VE) {
        const int nc = h / VE;
        if (nc >= U) lane_fg_chunks_any<R, U>(c, d, nc, lb, is_g, out);
        else lane_fg_chunks_any<R, 1>(c, d, nc, lb, is_g, out);
    } else {
        // the parent's m <= VE values are one contiguous chunk
        const R* p = c.chunk(d, 0);
        R* q = out + c.lane * h;
        const uint32_t bits = is_g ? c.word(lb >> 5) >> (lb & 31) : 0u;
        if constexpr (sizeof(R) == 1) {
            // int8 nodes of 16 / 8 / 4 values: SWAR words (the chunk is m-byte aligned)
            if (h == 2) {
                const uint32_t x = *reinterpret_cast<const uint32_t*>(p);
                const uint32_t o = is_g ? g_swar(x & 0xffffu, x >> 16, bits & 3u) : f_swar(x & 0xffffu, x >> 16);
                *reinterpret_cast<uint16_t*>(q) = uint16_t(o);
                return;
            }
            if (h == 8) {
                const uint4 x = *reinterpret_cast<const uint4*>(p);
                uint2 o;
                o.x = is_g ? g_swar(x.x, x.z, bits & 15u) : f_swar(x.x, x.z);
                o.y = is_g ? g_swar(x.y, x.w, (bits >> 4) & 15u) : f_swar(x.y, x.w);
                *reinterpret_cast<uint2*>(q) = o;
                return;
            }
            if (h == 4) {
                const uint2 x = *reinterpret_cast<const uint2*>(p);
                *reinterpret_cast<uint32_t*>(q) = is_g ? g_swar(x.x, x.y, bits & 15u) : f_swar(x.x, x.y);
                return;
            }
        }
        #pragma unroll 1
        for (int j = 0; j < h; ++j) q[j] = is_g ? A::g(p[j], p[h + j], (bits >> j) & 1u) : A::f(p[j], p[h + j]);
    }
}

template <typename R>
__device__ void lane_h(const LaneCtx<R>& c, int m, int lb) {
    const int h = m >> 1;
    if (h >= 32) {
        #pragma unroll 1
        for (int w = 0; w < (h >> 5); ++w) c.word((lb >> 5) + w) ^= c.word(((lb + h) >> 5) + w);
    } else {
        uint32_t& x = c.word(lb >> 5);
        const int s = lb & 31;
        const uint32_t mk = (1u << h) - 1u;
        x ^= ((x >> (s + h)) & mk) << s;
    }
}

// repetition node (sc_decoder.hpp:114-125): halving fold, bit = fold < 0.
// Chunk pairs are added elementwise first (into the dead depth-(d+1)
// segment), then the last chunk is folded in registers: the same additions
// in the same order as the reference's halving loop.
template <typename R>
__device__ int lane_rep(const LaneCtx<R>& c, int d, int m) {
    using A = Arith<R>;
    using M = typename A::M;
    constexpr int VE = LaneCtx<R>::VE;
    Vec<R, VE> x;
    int len = m;
    if (m > VE) {
        R* S = c.pool(d + 1) + c.lane * VE; // chunk k at S + k * 32 * VE
        int nc = m / VE;
        int cs;
        const R* in = c.chunk_base(d, cs);
        #pragma unroll 1
        for (int first = 1; nc > 1; first = 0) {
            const int hc = nc >> 1;
            #pragma unroll 1
            for (int k = 0; k < hc; ++k) {
                const Vec<R, VE> a = first ? vld<R, VE>(in + k * cs) : vld<R, VE>(S + k * 32 * VE);
                const Vec<R, VE> b = first ? vld<R, VE>(in + (k + hc) * cs) : vld<R, VE>(S + (k + hc) * 32 * VE);
                vst<R, VE>(S + k * 32 * VE, fg_compute<R, VE>(a, b, 0u, true)); // g with u = 0: sat(a + b)
            }
            nc = hc;
        }
        x = vld<R, VE>(S);
        len = VE;
    } else {
        const R* p = c.chunk(d, 0);
#pragma unroll
        for (int i = 0; i < VE; ++i) x.v[i] = i < m ? p[i] : R(0);
    }
    M v[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) v[i] = A::val(x.v[i]);
#pragma unroll
    for (int s = VE; s > 1; s >>= 1)
        if (s <= len)
#pragma unroll
            for (int i = 0; i < s / 2; ++i) v[i] = A::sat(v[i], v[i + s / 2]);
    return v[0] < M(0);
}

// rate-1 shortcut: true when this lane's m values hold no zero
template <typename R>
__device__ bool lane_r1_nozero(const LaneCtx<R>& c, int d, int m) {
    constexpr int VE = LaneCtx<R>::VE;
    bool zero = false;
    constexpr int NB = sizeof(R) == 4 ? 8 : 4; // chunks per trip (32 / 64 / 32 values)
    if (m >= NB * VE) {
        // NB chunks in flight per trip (the large rate-1 nodes read global
        // depth pools)
        int cs;
        const R* in = c.chunk_base(d, cs);
        #pragma unroll 1
        for (int k = 0; k < m / VE; k += NB) {
            Vec<R, VE> q[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) q[u] = vld<R, VE>(in + (k + u) * cs);
#pragma unroll
            for (int u = 0; u < NB; ++u) zero |= vec_has_zero<R, VE>(q[u]);
        }
    } else if (m >= VE) {
        int cs;
        const R* in = c.chunk_base(d, cs);
        #pragma unroll 1
        for (int k = 0; k < m / VE; ++k) zero |= vec_has_zero<R, VE>(vld<R, VE>(in + k * cs));
    } else if (sizeof(R) == 1 && m >= 4) { // int8 nodes of 4 / 8 values: whole words
        const uint32_t* p = reinterpret_cast<const uint32_t*>(c.chunk(d, 0));
        #pragma unroll 1
        for (int k = 0; k < (m >> 2); ++k) zero |= ((p[k] - 0x01010101u) & ~p[k] & 0x80808080u) != 0u;
    } else {
        const R* p = c.chunk(d, 0);
        #pragma unroll 1
        for (int i = 0; i < m; ++i) zero |= Arith<R>::val(p[i]) == typename Arith<R>::M(0);
    }
    return !zero;
}
template <typename R>
__device__ void lane_r1_hard(const LaneCtx<R>& c, int d, int m, int lb) {
    using A = Arith<R>;
    constexpr int VE = LaneCtx<R>::VE;
    constexpr int NB = sizeof(R) == 4 ? 8 : 4; // chunks per trip: whole partial-sum words
    if (m >= NB * VE) {
        // NB chunks' loads in flight together, then their words
        int cs;
        const R* in = c.chunk_base(d, cs);
        #pragma unroll 1
        for (int k = 0; k < m / VE; k += NB) {
            Vec<R, VE> q[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) q[u] = vld<R, VE>(in + (k + u) * cs);
#pragma unroll
            for (int w = 0; w < NB * VE / 32; ++w) {
                uint32_t acc = 0;
#pragma unroll
                for (int u = w * 32 / VE; u < (w + 1) * 32 / VE; ++u)
                    acc |= vec_signs<R, VE>(q[u]) << ((u * VE) & 31);
                c.word(((lb + k * VE) >> 5) + w) = acc;
            }
        }
    } else if (m >= VE) {
        uint32_t acc = 0;
        int cs;
        const R* in = c.chunk_base(d, cs);
        #pragma unroll 1
        for (int k = 0; k < m / VE; ++k) {
            const int pos = k * VE; // bit of the node
            acc |= vec_signs<R, VE>(vld<R, VE>(in + k * cs)) << (pos & 31);
            if (((pos + VE) & 31) == 0 || pos + VE >= m) {
                if (m >= 32) {
                    c.word((lb + (pos & ~31)) >> 5) = acc;
                } else {
                    const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
                    uint32_t& x = c.word(lb >> 5);
                    x = (x & ~mk) | ((acc << (lb & 31)) & mk);
                }
                acc = 0;
            }
        }
    } else {
        const R* p = c.chunk(d, 0);
        uint32_t acc = 0;
        if (sizeof(R) == 1 && m >= 4) { // sign bits of whole words
            #pragma unroll 1
            for (int k = 0; k < (m >> 2); ++k) {
                const uint32_t w = reinterpret_cast<const uint32_t*>(p)[k];
                acc |= ((((w >> 7) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
            }
        } else {
            #pragma unroll 1
            for (int i = 0; i < m; ++i) acc |= uint32_t(A::val(p[i]) < typename A::M(0)) << i;
        }
        const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
        uint32_t& x = c.word(lb >> 5);
        x = (x & ~mk) | ((acc << (lb & 31)) & mk);
    }
}

// OP_GR1: the G op at depth d whose child [lb + m/2, lb + m) is a
// rate-1 node.  The g values stay in registers: their signs go to the
// partial sums (rewritten by the expanded recursion if that runs) and the
// result says whether this lane saw no zero.  The input segment is neither
// stored to depth d + 1 nor dropped here (the plain G op still needs it when
// some lane has a zero).
template <typename R>
__device__ bool lane_gr1(const LaneCtx<R>& c, int d, int m, int lb) {
    constexpr int VE = LaneCtx<R>::VE;
    constexpr int NB = 32 / VE; // chunks per partial-sum word
    const int h = m >> 1, nc = h / VE;
    int cs;
    const R* in = c.chunk_base(d, cs);
    const R* in_b = in + nc * cs;
    const bool gin = c.keep > 0 && (d == 0 || (c.n >> d) > c.segmax);
    const uint64_t pin = gin ? c.policy(d) : 0;
    bool zero = false;
    #pragma unroll 1
    for (int k = 0; k < nc; k += NB) {
        Vec<R, VE> a[NB], b[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            if (gin) {
                a[u] = vld_hint<R, VE>(in + (k + u) * cs, pin);
                b[u] = vld_hint<R, VE>(in_b + (k + u) * cs, pin);
            } else {
                a[u] = vld<R, VE>(in + (k + u) * cs);
                b[u] = vld<R, VE>(in_b + (k + u) * cs);
            }
        }
        const uint32_t bits = c.word((lb + k * VE) >> 5);
        uint32_t acc = 0;
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const Vec<R, VE> r = fg_compute<R, VE>(a[u], b[u], bits >> (u * VE), true);
            zero |= vec_has_zero<R, VE>(r);
            acc |= vec_signs<R, VE>(r) << (u * VE);
        }
        c.word((lb + h + k * VE) >> 5) = acc;
    }
    return !zero;
}
// the input segment of a taken OP_GR1 is dead: drop its lines from the L2
template <typename R>
__device__ void lane_discard_seg(const LaneCtx<R>& c, int d, int m) {
    constexpr int VE = LaneCtx<R>::VE;
    if (!(c.discard && d > 0 && (c.n >> d) > c.segmax) || (c.lane & 7) != 0) return;
    int cs;
    const R* in = c.chunk_base(d, cs);
    #pragma unroll 1
    for (int k = 0; k < m / VE; ++k) asm volatile("discard.global.L2 [%0], 128;" :: "l"(in + k * cs) : "memory");
}

// ---- in-register subtrees (OP_SCSUB of the lane schedule) ----------------
// A subtree of M <= kLaneSubMax values is decoded by the unabridged SC
// recursion of sc_decoder.hpp:99-112 on registers: the lane loads its M
// LLRs once, every f / g level is straight-line code on values of the
// metric type (no depth-pool round trips, no per-op dispatch), and the
// node's partial sums (after its H steps) come back as M bits.  `mask`
// (uniform: one code per warp) marks the frozen positions.  R0 / REP / SPC /
// R1 sub-nodes decide exactly as their pruned forms do (sc_decoder.hpp:
// 80-94: rate-1 and single-parity run this very recursion; the repetition
// fold is the frozen descent's g chain; rate-0 leaves are all 0).
template <typename R>
__device__ __forceinline__ typename Arith<R>::M f_val(typename Arith<R>::M a, typename Arith<R>::M b) {
    if constexpr (sizeof(R) == 4) {
        return Arith<float>::f(a, b);
    } else {
        const int m = min(abs(a), abs(b));
        return ((a ^ b) < 0) ? -m : m;
    }
}
template <typename R>
__device__ __forceinline__ typename Arith<R>::M g_val(typename Arith<R>::M a, typename Arith<R>::M b,
                                                      uint32_t s) {
    if constexpr (sizeof(R) == 4) {
        return Arith<float>::g(a, b, s);
    } else {
        const int v = s ? b - a : a + b;
        return max(-Arith<R>::kMax, min(Arith<R>::kMax, v));
    }
}
template <typename R, int M>
__device__ __forceinline__ uint32_t sc_regs(const typename Arith<R>::M (&x)[M], uint32_t mask) {
    using MM = typename Arith<R>::M;
    if constexpr (M == 1) {
        return uint32_t(x[0] < MM(0)) & ~mask & 1u;
    } else {
        constexpr int H = M / 2;
        constexpr uint32_t ones = (1u << H) - 1u;
        MM t[H];
        uint32_t ul = 0;
        // an all-frozen left half decides 0 without its f values (uniform)
        if (M < 4 || (mask & ones) != ones) {
#pragma unroll
            for (int i = 0; i < H; ++i) t[i] = f_val<R>(x[i], x[i + H]);
            ul = sc_regs<R, H>(t, mask & ones);
        }
#pragma unroll
        for (int i = 0; i < H; ++i) t[i] = g_val<R>(x[i], x[i + H], (ul >> i) & 1u);
        const uint32_t ur = sc_regs<R, H>(t, mask >> H);
        return (ul ^ ur) | (ur << H);
    }
}
constexpr int kLaneSubMax = 16;

// fz (kOpFused [| kOpFusedG] on the op word): the subtree is fused with its
// parent's F (1) or G (2) op, which is absent from the schedule: the M LLRs
// are formed from the parent's 2M values (depth d - 1; G: with the left
// sibling's decisions, bits [lb - M, lb)) and never stored.
template <typename R, int M>
__device__ __forceinline__ void lane_sub(const LaneCtx<R>& c, int d, int lb, uint32_t mask, int fz) {
    using A = Arith<R>;
    using MM = typename A::M;
    constexpr int VE = LaneCtx<R>::VE;
    MM x[M];
    if (fz) {
        const bool is_g = fz == 2;
        const int up = lb - M;
        const uint32_t ub = is_g ? c.word(up >> 5) >> (up & 31) : 0u;
        if constexpr (M >= VE) {
            int cs;
            const R* in = c.chunk_base(d - 1, cs);
#pragma unroll
            for (int k = 0; k < M / VE; ++k) {
                const Vec<R, VE> q = fg_compute<R, VE>(vld<R, VE>(in + k * cs), vld<R, VE>(in + (k + M / VE) * cs),
                                                       ub >> (k * VE), is_g);
#pragma unroll
                for (int i = 0; i < VE; ++i) x[k * VE + i] = A::val(q.v[i]);
            }
        } else {
            // the parent's 2M <= VE values are one chunk
            const Vec<R, 2 * M> q = vld<R, 2 * M>(c.chunk(d - 1, 0));
#pragma unroll
            for (int i = 0; i < M; ++i)
                x[i] = A::val(is_g ? A::g(q.v[i], q.v[M + i], (ub >> i) & 1u) : A::f(q.v[i], q.v[M + i]));
        }
    } else if constexpr (M >= VE) {
        int cs;
        const R* in = c.chunk_base(d, cs);
#pragma unroll
        for (int k = 0; k < M / VE; ++k) {
            const Vec<R, VE> q = vld<R, VE>(in + k * cs);
#pragma unroll
            for (int i = 0; i < VE; ++i) x[k * VE + i] = A::val(q.v[i]);
        }
    } else {
        const Vec<R, M> q = vld<R, M>(c.chunk(d, 0));
#pragma unroll
        for (int i = 0; i < M; ++i) x[i] = A::val(q.v[i]);
    }
    uint32_t bits;
    bool hard = false;
    if (mask == 0u) {
        // rate-1 shortcut (uniform): no zero input in any lane -> hard decisions
        bool nz = true;
#pragma unroll
        for (int i = 0; i < M; ++i) nz &= x[i] != MM(0);
        hard = __all_sync(FULL, nz);
    }
    if (hard) {
        bits = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) bits |= uint32_t(x[i] < MM(0)) << i;
    } else {
        bits = sc_regs<R, M>(x, mask);
    }
    constexpr uint32_t mk0 = M >= 32 ? FULL : ((1u << M) - 1u);
    uint32_t& w = c.word(lb >> 5);
    const int s = lb & 31;
    w = (w & ~(mk0 << s)) | (bits << s);
}

template <typename R>
__device__ void lane_frame(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                           unsigned char* gs, int frame, bool active, int lane) {
    using A = Arith<R>;
    using M = typename A::M;
    if (P.lat_ns && active) P.lat_ns[frame] -= uint32_t(gtimer());
    LaneCtx<R> c;
    c.lane = lane;
    c.n = C.n;
    c.segmax = P.seg_smem_max;
    c.keep = P.sc_keep;
    c.keep_hi = P.sc_keep_hi;
    c.discard = P.sc_discard != 0;
    c.il = P.llr_il32 != 0;
    if (c.il) {
        // chunk 0 of this lane's frame inside its group of 32 (host.cu
        // accepts the layout only without a frame list: frame = 32 * g + lane)
        const int v = min(LaneCtx<R>::VE, C.n);
        c.chan = static_cast<const R*>(P.llr) + int64_t(frame >> 5) * C.n * 32 + (frame & 31) * v;
    } else {
        c.chan = frame_llr<R>(P, frame);
    }
    const LaneQ q0 = lane_layout(C.n, int(sizeof(R)), P.seg_smem_max, 0, P.sc_tr != 0);
    c.ps = reinterpret_cast<uint32_t*>(sm + q0.psum_off) + lane;
    uint64_t* pt = reinterpret_cast<uint64_t*>(sm);
    c.pt = pt;
    // transposed channel reads: frame-major channel, the depth-1 pool global,
    // at least one 8-chunk tile per half (lane_layout reserved the tile)
    c.stage = (P.sc_tr && !c.il && (C.n >> 1) > P.seg_smem_max && (C.n >> 1) / LaneCtx<R>::VE >= 8 &&
               q0.stage_bytes >= kLaneStageBytes<R>)
                  ? sm + q0.stage_off : nullptr;
    __syncwarp();
    if (lane >= 1 && lane <= C.stages) {
        const LaneQ q = lane_layout(C.n, int(sizeof(R)), P.seg_smem_max, lane, P.sc_tr != 0);
        pt[lane] = reinterpret_cast<uint64_t>((q.pool_in_smem ? sm : gs) + q.pool_off);
    }
    __syncwarp();
    const uint32_t* sched = C.sched_lane;
    const int nops = C.nops_lane;
    // the next schedule word is fetched one op ahead (the schedules carry a
    // padding word)
    uint32_t next = __ldg(sched);
    #pragma unroll 1
    for (int oi = 0; oi < nops; ++oi) {
        const uint32_t op = next;
        next = __ldg(sched + oi + 1);
        const int code = op_code(op), d = op_depth(op), m = 1 << op_logm(op), lb = op_lb(op);
        switch (code) {
        case OP_F:
        case OP_G: lane_fg(c, d, m, lb, code == OP_G, int(op >> kOpChainShift) & 3); break;
        case OP_H: lane_h(c, m, lb); break;
        case OP_FROZEN: c.fill(lb, m, 0); break;
        case OP_INFO: c.fill(lb, 1, A::val(*c.chunk(d, 0)) < M(0)); break;
        case OP_REP: c.fill(lb, m, lane_rep(c, d, m)); break;
        case OP_SCSUB: {
            const uint32_t mask = next; // the word after OP_SCSUB
            ++oi;
            next = __ldg(sched + oi + 1);
            const int fz = (op & kOpFused) ? ((op & kOpFusedG) ? 2 : 1) : 0;
            switch (m) {
            case 2: lane_sub<R, 2>(c, d, lb, mask, fz); break;
            case 4: lane_sub<R, 4>(c, d, lb, mask, fz); break;
            case 8: lane_sub<R, 8>(c, d, lb, mask, fz); break;
            default: lane_sub<R, 16>(c, d, lb, mask, fz); break;
            }
            break;
        }
        case OP_GR1: {
            const int skip = int(next); // the word after OP_GR1
            ++oi;
            if (__all_sync(FULL, lane_gr1(c, d, m, lb))) {
                lane_discard_seg(c, d, m);
                oi += skip;
            } // else: the plain G op and the expanded recursion follow
            next = __ldg(sched + oi + 1);
            break;
        }
        case OP_R1SC: {
            const int skip = int(next); // the word after OP_R1SC
            ++oi;
            const bool r1ok = __all_sync(FULL, lane_r1_nozero(c, d, m));
#ifdef PLB_OPTIME
            // (profiling build) rate-1 shortcut attempts / successes per node size
            if (lane == 0) {
                atomicAdd(&g_optime[op_logm(op)], 1ull);
                if (r1ok) atomicAdd(&g_optime[32 + op_logm(op)], 1ull);
            }
#endif
            if (r1ok) {
                lane_r1_hard(c, d, m, lb);
                oi += skip;
            } // else: every lane runs the expanded recursion that follows
            next = __ldg(sched + oi + 1);
            break;
        }
        default: break;
        }
    }
    // finish: CRC syndrome, payload, codeword, status (per lane).  Codes of
    // n >= 32 go word by word: the four table lookups of a partial-sum word
    // are independent loads (two words per trip: eight in flight), and the
    // outputs leave as 32-bit stores where the rows are 4-byte aligned (one
    // byte store per payload byte is a partial-sector write each).
    int crc_ok = 0;
    const int nwords = C.n >> 5;
    if (C.crc_width > 0) {
        uint64_t syn = C.crc_c0;
        if (nwords > 0) {
            #pragma unroll 2
            for (int w = 0; w < nwords; ++w) {
                const uint32_t x = c.word(w);
                const uint64_t* t = C.crc_tab + (size_t(w) << 10);
                const uint64_t t0 = __ldg(t + (x & 0xffu)), t1 = __ldg(t + 256 + ((x >> 8) & 0xffu));
                const uint64_t t2 = __ldg(t + 512 + ((x >> 16) & 0xffu)), t3 = __ldg(t + 768 + (x >> 24));
                syn ^= (t0 ^ t1) ^ (t2 ^ t3);
            }
        } else {
            const int nbytes = (C.n + 7) >> 3;
            #pragma unroll 1
            for (int j = 0; j < nbytes; ++j) {
                const uint32_t byte = (c.word(j >> 2) >> ((j & 3) * 8)) & 0xffu;
                syn ^= __ldg(C.crc_tab + (size_t(j) << 8) + byte);
            }
        }
        crc_ok = syn == 0;
    }
    if (active) {
        // payload (extract_payload, prune_tree.hpp:78-105): the open bits of
        // each codeword byte compacted by table (all-open bytes: a bit
        // reversal) and streamed out MSB-first
        uint8_t* pay = P.payload + int64_t(frame) * P.payload_stride;
        const bool al4 = ((reinterpret_cast<uintptr_t>(P.payload) | uintptr_t(P.payload_stride)) & 3u) == 0;
        uint32_t acc = 0, ow = 0;
        int nb = 0, qb = 0;
        // byte qb of the row: through a 32-bit word when the row is aligned
        auto emit = [&](uint32_t byte) {
            if (al4) {
                ow |= byte << ((qb & 3) * 8);
                if ((qb & 3) == 3) {
                    *reinterpret_cast<uint32_t*>(pay + (qb & ~3)) = ow;
                    ow = 0;
                }
            } else {
                pay[qb] = uint8_t(byte);
            }
            ++qb;
        };
        auto take = [&](uint32_t m, uint32_t v) {
            if (m == 0u) return; // uniform: one code per warp
            const uint32_t bits = m == 0xffu ? __brev(v) >> 24 : uint32_t(__ldg(C.comp_tab + (m << 8) + v));
            const int k = __popc(m);
            acc = (acc << k) | bits;
            nb += k;
            if (nb >= 8) {
                nb -= 8;
                emit((acc >> nb) & 0xffu);
            }
        };
        if (nwords > 0) {
            const uint32_t* om = reinterpret_cast<const uint32_t*>(C.open_mask); // (uploads are 16-byte aligned)
            #pragma unroll 1
            for (int w = 0; w < nwords; ++w) {
                const uint32_t mm = __ldg(om + w), x = c.word(w);
#pragma unroll
                for (int b = 0; b < 4; ++b) take((mm >> (8 * b)) & 0xffu, (x >> (8 * b)) & 0xffu);
            }
        } else {
            const int cbytes = (C.n + 7) >> 3;
            #pragma unroll 1
            for (int j = 0; j < cbytes; ++j)
                take(__ldg(C.open_mask + j), (c.word(j >> 2) >> ((j & 3) * 8)) & 0xffu);
        }
        if (nb > 0) emit((acc << (8 - nb)) & 0xffu);
        if (al4 && (qb & 3) != 0) {
#pragma unroll 1
            for (int b = 0; b < (qb & 3); ++b) pay[(qb & ~3) + b] = uint8_t(ow >> (8 * b));
        }
        if (P.codeword) {
            uint8_t* cw = P.codeword + int64_t(frame) * P.codeword_stride;
            const bool cal4 = ((reinterpret_cast<uintptr_t>(P.codeword) | uintptr_t(P.codeword_stride)) & 3u) == 0;
            if (nwords > 0 && cal4) {
                #pragma unroll 1
                for (int w = 0; w < nwords; ++w) // bits reversed inside every byte, byte order kept
                    reinterpret_cast<uint32_t*>(cw)[w] = __byte_perm(__brev(c.word(w)), 0u, 0x0123u);
            } else {
                const int cb = (C.n + 7) >> 3;
                #pragma unroll 1
                for (int qb2 = 0; qb2 < cb; ++qb2) {
                    const uint32_t bits = (c.word(qb2 >> 2) >> ((qb2 & 3) * 8)) & 0xffu;
                    const uint32_t byte = __brev(bits) >> 24;
                    cw[qb2] = uint8_t(C.n >= 8 ? byte : (byte & (0xffu << (8 - C.n))));
                }
            }
        }
        if (P.crc_ok) P.crc_ok[frame] = uint8_t(crc_ok);
        if (P.esc) P.esc[frame] = 1;
        if (P.metric) P.metric[frame] = 0.0f; // DecodeResult default (decode_result.hpp:12)
        if (P.lat_ns) P.lat_ns[frame] += uint32_t(gtimer());
    }
    // failed frames -> the next rung's list (warp-aggregated append)
    if (P.fail_list && C.crc_width > 0) {
        const bool f = active && !crc_ok;
        const unsigned fm = __ballot_sync(FULL, f);
        int base = 0;
        if (lane == 0 && fm) base = atomicAdd(P.fail_count, __popc(fm));
        base = __shfl_sync(FULL, base, 0);
        if (f) P.fail_list[base + __popc(fm & lanemask_lt())] = frame;
    }
    __syncwarp();
}

// resident blocks the register budget allows: float runs 16 warps per SM
// (DRAM-bound), the fixed-point passes 24 (host.cu plan_lanes)
template <typename R>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? PLB_LANE_MINB : 6) sc_lanes_kernel(const LaunchParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* sm = smem_raw + wib * P.smem_per_warp;
    const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
    // (for this kernel gscratch_per_frame is the scratch of one 32-frame warp)
    unsigned char* gs = static_cast<unsigned char*>(P.gscratch) + gw * P.gscratch_per_frame;
    const long long count = P.frame_list ? (long long)(*P.frame_count) : (long long)P.nframes;
    for (;;) {
        unsigned long long i0 = 0;
        if (lane == 0) i0 = atomicAdd(P.work, 32ull);
        const long long idx0 = (long long)__shfl_sync(FULL, i0, 0);
        if (idx0 >= count) break;
        const long long mine = idx0 + lane;
        const bool active = mine < count;
        const long long idx = active ? mine : idx0; // idle lanes shadow frame idx0
        const int frame = P.frame_list ? P.frame_list[idx] : int(idx);
        const int cid = P.code_id ? P.code_id[frame] : 0;
        // lockstep needs one code: one pass per distinct code of the warp
        // (multi-code batches arrive bucketed by code, so usually one)
        unsigned pending = FULL;
        while (pending) {
            const int cc = __shfl_sync(FULL, cid, __ffs(pending) - 1);
            const unsigned grp = __ballot_sync(FULL, cid == cc) & pending;
            pending &= ~grp;
            // lanes outside the group shadow a member's frame: packed frames of
            // another code may be shorter than this code's n (no reads past them)
            const bool in_grp = (grp >> lane) & 1u;
            const int fr = __shfl_sync(FULL, frame, __ffs(grp) - 1);
            lane_frame<R>(P, P.codes[cc], sm, gs, in_grp ? frame : fr, active && in_grp, lane);
        }
    }
}
