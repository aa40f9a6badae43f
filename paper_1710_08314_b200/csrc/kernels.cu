// sm_100a kernels of the batched polar decoder.
//
// Mapping: one warp decodes one frame at a time.  A
// persistent grid of warps claims frames from an atomic counter (frames
// differ in cost under adaptive decoding).  Inside a warp the lanes are
// spread over (list path, LLR element) pairs, so a node of width m with A
// alive paths keeps all 32 lanes busy once A*m/2 >= 32, and every fork /
// sort / slot-assignment step is warp-synchronous (shuffles, ballots, match,
// no CTA barrier).  Per-path bookkeeping lives in registers with lane ==
// slot: lane s holds the path metric of slot s.
//
// LLR storage follows the reference's depth-segment stack (sc_decoder.hpp:
// 18-20, list_decoder.hpp:45) but with lazy copies: every depth d >= 1 has
// a pool of l buffers of n>>d values and each slot points at one buffer per
// depth (bufidx[slot][d]).  Duplicating a path (list_decoder.hpp:402-423)
// copies 16 bytes of pointers instead of up to L*n LLRs; a path that is
// about to overwrite a depth whose buffer it shares takes a free buffer
// first ("own").  Depth 0 is the channel frame, read in place from HBM.
// Small segments live in shared memory, large ones in a per-warp global
// scratch (L2-resident).  Partial sums are bit-packed, one n-bit row per
// slot, LSB-first within 32-bit words; h becomes a word XOR.
//
// Bit-exactness: f/g/h, the penalty sums (sequential, index
// order), the halving REP fold, the (value,index) two-smallest order, the
// stable (metric, emission-index) ranking, the slot assignment and int8
// normalisation all reproduce list_decoder.hpp / sc_decoder.hpp exactly.
#include <cstdint>

#include "polar_dev.h"

namespace plb {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(FULL, uint32_t(v), src);
    uint32_t hi = __shfl_sync(FULL, uint32_t(v >> 32), src);
    return (uint64_t(hi) << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m, int w = 32) {
    uint32_t lo = __shfl_xor_sync(FULL, uint32_t(v), m, w);
    uint32_t hi = __shfl_xor_sync(FULL, uint32_t(v >> 32), m, w);
    return (uint64_t(hi) << 32) | lo;
}
__device__ __forceinline__ int pack_aux(int a, int b) {
    return int((uint32_t(a) & 0xffffu) | (uint32_t(b) << 16));
}
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a < b ? b : a; }

// ---- per-representation arithmetic (llr.hpp:36-69) -------------------
template <typename R>
struct Arith;

template <>
struct Arith<float> {
    using M = float; // path-metric type
    static constexpr bool kFixed = false;
    __device__ static M sat(M a, M b) { return a + b; }
    // |v| as a non-negative float: abs_llr(-0.0f) is -0.0f in the reference
    // but every use of a magnitude is an add to a non-negative metric or a
    // (value, index) comparison, where +-0 behave identically.
    __device__ static M mag(float v) { return fabsf(v); }
    __device__ static uint32_t key(M v) { return __float_as_uint(v); } // v >= +0
    __device__ static M from_key(uint32_t k) { return __uint_as_float(k); }
    __device__ static M val(float v) { return v; }
    __device__ static float f(float a, float b) {
        // min-sum (llr.hpp:55-59).  The sign comes from the sign bits, which
        // differs from `(a<0) != (b<0)` only when an operand is -0.0, and
        // then the magnitude is 0: the result is a zero either way.
        const float m = fminf(fabsf(a), fabsf(b));
        return __uint_as_float(__float_as_uint(m) |
                               ((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u));
    }
    __device__ static float g(float a, float b, uint32_t s) { return s ? b - a : a + b; }
    __device__ static float store(M v) { return v; }
    __device__ static float to_float(M v) { return v; }
};

template <>
struct Arith<int8_t> {
    using M = int;
    static constexpr bool kFixed = true;
    __device__ static M sat(M a, M b) { return max(-127, min(127, a + b)); }
    __device__ static M mag(int v) { return abs(v); }
    __device__ static uint32_t key(M v) { return uint32_t(v); } // v in [0, 127]
    __device__ static M from_key(uint32_t k) { return int(k); }
    __device__ static M val(int8_t v) { return int(v); }
    __device__ static int8_t f(int8_t a, int8_t b) {
        const int m = min(abs(int(a)), abs(int(b)));
        return int8_t(((a ^ b) < 0) ? -m : m);
    }
    __device__ static int8_t g(int8_t a, int8_t b, uint32_t s) {
        const int v = s ? int(b) - int(a) : int(a) + int(b);
        return int8_t(max(-127, min(127, v)));
    }
    __device__ static int8_t store(M v) { return int8_t(v); }
    __device__ static float to_float(M v) { return float(v); }
};

template <typename M>
__device__ __forceinline__ uint32_t mbits(M v);
template <>
__device__ __forceinline__ uint32_t mbits<float>(float v) { return __float_as_uint(v); }
template <>
__device__ __forceinline__ uint32_t mbits<int>(int v) { return uint32_t(v); }
template <typename M>
__device__ __forceinline__ M mfrom(uint32_t b);
template <>
__device__ __forceinline__ float mfrom<float>(uint32_t b) { return __uint_as_float(b); }
template <>
__device__ __forceinline__ int mfrom<int>(uint32_t b) { return int(b); }

// ---- vector access of G consecutive values ----------------------------
template <int B>
struct VT;
template <> struct VT<1> { using T = uint8_t; };
template <> struct VT<2> { using T = uint16_t; };
template <> struct VT<4> { using T = uint32_t; };
template <> struct VT<8> { using T = uint2; };
template <> struct VT<16> { using T = uint4; };

template <typename R, int G>
union Vec {
    typename VT<G * sizeof(R)>::T raw;
    R v[G];
};

template <typename R, int G>
__device__ __forceinline__ Vec<R, G> vld(const R* p) {
    Vec<R, G> x;
    x.raw = *reinterpret_cast<const typename VT<G * sizeof(R)>::T*>(p);
    return x;
}
template <typename R, int G>
__device__ __forceinline__ void vst(R* p, const Vec<R, G>& x) {
    *reinterpret_cast<typename VT<G * sizeof(R)>::T*>(p) = x.raw;
}

// ---- per-warp shared-memory area ---------------------------------------
struct alignas(16) Fixed {
    uint8_t bufidx[32 * 16]; // [slot][depth] -> buffer index in the depth pool
    uint8_t alive_list[32];  // rank -> slot, ascending
    int32_t ksrc[32];        // kept candidates by rank
    int32_t kaux[32];
    uint32_t kmet[32];
    uint32_t met_s[32];
    int32_t st_i1[32], st_i2[32], st_w[32]; // per-rank node statistics
    uint32_t st_a1[32], st_a2[32];
    uint64_t pool[16];       // generic address of each depth pool
};
static_assert(sizeof(Fixed) % 16 == 0, "fixed area alignment");

struct Layout {
    int32_t rw;        // psum row words
    int32_t psum_off;  // bytes, in shared memory
    int32_t pool_off[16];
    uint32_t in_smem;  // depths whose pool is in shared memory
    int32_t smem_total, gmem_total;
};

__host__ __device__ inline int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) ++r;
    return r;
}
__host__ __device__ inline int align16(int v) { return (v + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int n, int l, int esz, int segmax) {
    Layout L{};
    int off = int(sizeof(Fixed));
    L.rw = n >= 32 ? n / 32 : 1;
    L.psum_off = off;
    off = align16(off + 4 * l * L.rw);
    int goff = 0;
    const int stages = ilog2(n);
    for (int d = 1; d <= stages; ++d) {
        const int seg = n >> d;
        const int bytes = align16(l * seg * esz);
        if (seg <= segmax) {
            L.pool_off[d] = off;
            off += bytes;
            L.in_smem |= 1u << d;
        } else {
            L.pool_off[d] = goff;
            goff += bytes;
        }
    }
    L.smem_total = off;
    L.gmem_total = goff;
    return L;
}

// ---- warp decode context ----------------------------------------------
template <typename R>
struct Ctx {
    using A = Arith<R>;
    using M = typename A::M;

    int lane, n, stages, l;
    unsigned lmask;
    const R* chan;
    Fixed* fx;
    uint32_t* ps;
    int rw;
    unsigned alive; // warp-uniform alive-slot mask
    unsigned dirty; // depths whose buffers may be shared between slots
    M metric;       // lane s: metric of slot s

    __device__ __forceinline__ R* llr(int p, int d) const {
        if (d == 0) return const_cast<R*>(chan);
        R* base = reinterpret_cast<R*>(fx->pool[d]);
        return base + int(fx->bufidx[p * 16 + d]) * (n >> d);
    }
    __device__ __forceinline__ uint32_t* row(int p) const { return ps + p * rw; }
    __device__ __forceinline__ bool is_alive() const { return (alive >> lane) & 1u; }

    __device__ void rebuild_alive_list() {
        if (is_alive()) fx->alive_list[__popc(alive & lanemask_lt())] = uint8_t(lane);
        __syncwarp();
    }

    // Give every alive slot an exclusive buffer at depth d1 before it is
    // overwritten (lazy copy-on-write; contents are dead, nothing is copied).
    __device__ void own(int d1) {
        if (!((dirty >> d1) & 1u)) return;
        dirty &= ~(1u << d1);
        const bool al = is_alive();
        const int b = al ? int(fx->bufidx[lane * 16 + d1]) : 64 + lane;
        const unsigned same = __match_any_sync(FULL, b);
        const bool need = al && (__ffs(same) - 1) != lane;
        const unsigned needm = __ballot_sync(FULL, need);
        if (needm) {
            const unsigned used = __reduce_or_sync(FULL, al ? (1u << b) : 0u);
            const unsigned freem = ~used & lmask;
            if (need) {
                const int k = __popc(needm & lanemask_lt());
                fx->bufidx[lane * 16 + d1] = uint8_t(__fns(freem, 0, k + 1));
            }
        }
        __syncwarp();
    }

    // int8 metrics: pull the smallest alive metric back to 0
    // (list_decoder.hpp:447-455).
    __device__ void normalize() {
        if constexpr (A::kFixed) {
            const int v = is_alive() ? int(metric) : 127;
            const int mn = int(__reduce_min_sync(FULL, unsigned(v)));
            if (is_alive()) metric -= mn;
        }
    }
};

// ---- f / g over all alive paths ----------------------------------------
template <typename R, int G, bool IS_G>
__device__ __forceinline__ void fg_item(const R* in, R* out, const uint32_t* prow, int h,
                                        int c, int lb) {
    using A = Arith<R>;
    const Vec<R, G> a = vld<R, G>(in + c * G);
    const Vec<R, G> b = vld<R, G>(in + h + c * G);
    Vec<R, G> o;
    if constexpr (IS_G) {
        const int pos = lb + c * G;
        const uint32_t bits = prow[pos >> 5] >> (pos & 31);
#pragma unroll
        for (int i = 0; i < G; ++i) o.v[i] = A::g(a.v[i], b.v[i], (bits >> i) & 1u);
    } else {
#pragma unroll
        for (int i = 0; i < G; ++i) o.v[i] = A::f(a.v[i], b.v[i]);
    }
    vst<R, G>(out + c * G, o);
}

template <typename R, int G, bool IS_G>
__device__ void fg_run(Ctx<R>& cx, int d, int h, int lb, int na) {
    const int cp = h / G; // items per path, power of two
    const int lg = __ffs(cp) - 1;
    if (cp >= 32) {
        for (int r = 0; r < na; ++r) {
            const int p = cx.fx->alive_list[r];
            const R* in = cx.llr(p, d);
            R* out = cx.llr(p, d + 1);
            const uint32_t* prow = cx.row(p);
#pragma unroll 2
            for (int c = cx.lane; c < cp; c += 32) fg_item<R, G, IS_G>(in, out, prow, h, c, lb);
        }
    } else {
        const int total = na << lg;
        for (int t = cx.lane; t < total; t += 32) {
            const int p = cx.fx->alive_list[t >> lg];
            fg_item<R, G, IS_G>(cx.llr(p, d), cx.llr(p, d + 1), cx.row(p), h, t & (cp - 1), lb);
        }
    }
    __syncwarp();
}

template <typename R, bool IS_G>
__device__ void op_fg(Ctx<R>& cx, int d, int m, int lb, int na) {
    constexpr int VE = 16 / int(sizeof(R));
    const int h = m >> 1;
    const int G = h < VE ? h : VE;
    cx.own(d + 1);
    switch (G) {
    case 1: fg_run<R, 1, IS_G>(cx, d, h, lb, na); break;
    case 2: fg_run<R, 2, IS_G>(cx, d, h, lb, na); break;
    case 4: fg_run<R, 4, IS_G>(cx, d, h, lb, na); break;
    default:
        if constexpr (VE >= 8) {
            if (G == 8) fg_run<R, 8, IS_G>(cx, d, h, lb, na);
            else fg_run<R, 16, IS_G>(cx, d, h, lb, na);
        }
        break;
    }
}

// psums[lb, lb+h) ^= psums[lb+h, lb+2h) for every alive path
template <typename R>
__device__ void op_h(Ctx<R>& cx, int m, int lb, int na) {
    const int h = m >> 1;
    if (h >= 32) {
        const int W = h >> 5, lg = __ffs(W) - 1;
        const int total = na << lg;
        for (int t = cx.lane; t < total; t += 32) {
            uint32_t* w = cx.row(cx.fx->alive_list[t >> lg]) + (lb >> 5) + (t & (W - 1));
            w[0] ^= w[W];
        }
    } else if (cx.lane < na) {
        uint32_t* w = cx.row(cx.fx->alive_list[cx.lane]) + (lb >> 5);
        const int s = lb & 31;
        const uint32_t mk = (1u << h) - 1u;
        *w ^= ((*w >> (s + h)) & mk) << s;
    }
    __syncwarp();
}

// write `bit` over the span [lb, lb+m) of path p's psum row (whole warp)
__device__ __forceinline__ void span_fill_warp(uint32_t* row, int lb, int m, int bit, int lane) {
    if (m >= 32) {
        for (int w = lane; w < (m >> 5); w += 32) row[(lb >> 5) + w] = bit ? FULL : 0u;
    } else if (lane == 0) {
        const uint32_t mk = (m == 32 ? FULL : ((1u << m) - 1u)) << (lb & 31);
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
// to st_a1[r].  For m > 32 the first halvings run in the path's depth-(d+1)
// buffer, whose contents are dead at a leaf.
template <typename R>
__device__ void rep_fold(Ctx<R>& cx, int d, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    if (m <= 32) {
        const int lgm = __ffs(m) - 1;
        const int per = 32 >> lgm;
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
    } else {
        for (int r = 0; r < na; ++r) {
            const int p = cx.fx->alive_list[r];
            const R* L = cx.llr(p, d);
            // scratch: the depth-(d+1) buffer of this path (dead at a leaf).
            // A shared buffer is fine: paths are folded one after another.
            R* S = cx.llr(p, d + 1);
            const int h = m >> 1;
            for (int i = cx.lane; i < h; i += 32) S[i] = A::store(A::sat(A::val(L[i]), A::val(L[i + h])));
            __syncwarp();
            for (int len = h; len > 32; len >>= 1) {
                const int hh = len >> 1;
                for (int i = cx.lane; i < hh; i += 32) S[i] = A::store(A::sat(A::val(S[i]), A::val(S[i + hh])));
                __syncwarp();
            }
            M v = A::val(S[cx.lane]);
            for (int off = 16; off >= 1; off >>= 1) {
                const M o = __shfl_down_sync(FULL, v, off);
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
// candidate i = lane + 32k in register k.  aux = a | b << 16 (int16 each).
template <typename R, int CPL>
__device__ void fork_apply(Ctx<R>& cx, const typename Arith<R>::M (&cm)[CPL],
                           const int (&csrc)[CPL], const int (&caux)[CPL], int ncand,
                           int kind, int lb, int m) {
    using A = Arith<R>;
    using M = typename A::M;
    const int lane = cx.lane;
    // 1. stable rank by (metric, emission index)
    uint64_t key[CPL];
    int rank[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = lane + 32 * k;
        key[k] = i < ncand ? ((uint64_t(A::key(cm[k])) << 32) | uint32_t(i)) : ~0ull;
        rank[k] = 0;
    }
#pragma unroll
    for (int kk = 0; kk < CPL; ++kk) {
        const int lim = min(32, ncand - 32 * kk);
        for (int j = 0; j < lim; ++j) {
            const uint64_t kj = shfl64(key[kk], j);
#pragma unroll
            for (int k = 0; k < CPL; ++k) rank[k] += kj < key[k];
        }
    }
    const int keep = min(cx.l, ncand);
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = lane + 32 * k;
        if (i < ncand && rank[k] < keep) {
            cx.fx->kmet[rank[k]] = mbits<M>(cm[k]);
            cx.fx->ksrc[rank[k]] = csrc[k];
            cx.fx->kaux[rank[k]] = caux[k];
        }
    }
    __syncwarp();
    // 2. slot assignment: first use of a slot stays, others take the next
    //    free slot in ascending order
    const bool kept = lane < keep;
    const int src = kept ? cx.fx->ksrc[lane] : 64 + lane;
    const int aux = kept ? cx.fx->kaux[lane] : 0;
    const unsigned same = __match_any_sync(FULL, src);
    const bool first = kept && (__ffs(same) - 1) == lane;
    const unsigned surv = __reduce_or_sync(FULL, kept ? (1u << src) : 0u);
    const unsigned freem = cx.lmask & ~surv;
    const bool dup = kept && !first;
    const unsigned dupm = __ballot_sync(FULL, dup);
    int tgt = src;
    if (dup) tgt = int(__fns(freem, 0, __popc(dupm & lanemask_lt()) + 1));
    // 3. duplicates: pointer rows + decided partial sums (incl. the node
    //    span, which holds the source's hard decisions for R1/SPC)
    if (dupm) {
        cx.dirty = FULL;
        if (dup) {
            *reinterpret_cast<uint4*>(cx.fx->bufidx + tgt * 16) =
                *reinterpret_cast<const uint4*>(cx.fx->bufidx + src * 16);
        }
        const int nw = min(cx.rw, (lb + m + 31) >> 5);
        for (unsigned mm = dupm; mm; mm &= mm - 1) {
            const int dl = __ffs(mm) - 1;
            const int s = __shfl_sync(FULL, src, dl);
            const int t = __shfl_sync(FULL, tgt, dl);
            const uint32_t* sr = cx.row(s);
            uint32_t* tr = cx.row(t);
            for (int w = lane; w < nw; w += 32) tr[w] = sr[w];
        }
        __syncwarp();
    }
    // 4. apply decisions (list_decoder.hpp:425-445)
    const int ca = int(int16_t(aux & 0xffff)), cb = aux >> 16;
    if (kind == AK_BIT) {
        if (kept) span_fill_lane(cx.row(tgt), lb, 1, ca);
    } else if (kind == AK_BCAST) {
        if (m < 32) {
            if (kept) span_fill_lane(cx.row(tgt), lb, m, ca);
        } else {
            for (int r = 0; r < keep; ++r) {
                const int t = __shfl_sync(FULL, tgt, r);
                const int bit = __shfl_sync(FULL, ca, r);
                span_fill_warp(cx.row(t), lb, m, bit, lane);
            }
        }
    } else if (kept) {
        uint32_t* tr = cx.row(tgt);
        if (ca >= 0) tr[(lb + ca) >> 5] ^= 1u << ((lb + ca) & 31);
        if (cb >= 0) tr[(lb + cb) >> 5] ^= 1u << ((lb + cb) & 31);
    }
    if (kept) cx.fx->met_s[tgt] = cx.fx->kmet[lane];
    cx.alive = __reduce_or_sync(FULL, kept ? (1u << tgt) : 0u);
    __syncwarp();
    if (cx.is_alive()) cx.metric = mfrom<M>(cx.fx->met_s[lane]);
    cx.rebuild_alive_list();
}

// base metric of the path at rank r (all lanes participate)
template <typename R>
__device__ __forceinline__ typename Arith<R>::M base_of(const Ctx<R>& cx, int r) {
    const int p = cx.fx->alive_list[r];
    return __shfl_sync(FULL, cx.metric, p);
}

// frozen leaf / rate-0 node (list_decoder.hpp:227-238)
template <typename R>
__device__ void list_frozen(Ctx<R>& cx, int d, int m, int lb, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    M pen = M(0);
    if (cx.lane < na) {
        const R* L = cx.llr(cx.fx->alive_list[cx.lane], d);
        for (int i = 0; i < m; ++i) {
            const M v = A::val(L[i]);
            if (v < M(0)) pen = A::sat(pen, -v); // sequential: float order matters
        }
    }
    const int myrank = __popc(cx.alive & lanemask_lt());
    const M pr = __shfl_sync(FULL, pen, myrank & 31);
    if (cx.is_alive()) cx.metric = A::sat(cx.metric, pr);
    if (m >= 32) {
        const int W = m >> 5;
        for (int t = cx.lane; t < na * W; t += 32)
            cx.row(cx.fx->alive_list[t / W])[(lb >> 5) + (t % W)] = 0u;
    } else if (cx.lane < na) {
        span_fill_lane(cx.row(cx.fx->alive_list[cx.lane]), lb, m, 0);
    }
    __syncwarp();
    cx.normalize();
}

// information leaf (list_decoder.hpp:240-252)
template <typename R>
__device__ void list_info(Ctx<R>& cx, int d, int lb, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    const int ncand = 2 * na;
    if (ncand <= 32) {
        M cm[1];
        int cs[1], cax[1];
        const int i = cx.lane, r = min(i >> 1, na - 1), j = i & 1;
        const int p = cx.fx->alive_list[r];
        const M v = A::val(cx.llr(p, d)[0]);
        const M base = __shfl_sync(FULL, cx.metric, p);
        const bool hb = v < M(0);
        const M av = A::mag(v);
        cm[0] = A::sat(base, (j == 0) == hb ? av : M(0));
        cs[0] = p;
        cax[0] = pack_aux(j, -1);
        fork_apply<R, 1>(cx, cm, cs, cax, ncand, AK_BIT, lb, 1);
    } else {
        M cm[2];
        int cs[2], cax[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int i = cx.lane + 32 * k, r = min(i >> 1, na - 1), j = i & 1;
            const int p = cx.fx->alive_list[r];
            const M v = A::val(cx.llr(p, d)[0]);
            const M base = __shfl_sync(FULL, cx.metric, p);
            const bool hb = v < M(0);
            const M av = A::mag(v);
            cm[k] = A::sat(base, (j == 0) == hb ? av : M(0));
            cs[k] = p;
            cax[k] = pack_aux(j, -1);
        }
        fork_apply<R, 2>(cx, cm, cs, cax, ncand, AK_BIT, lb, 1);
    }
    cx.normalize();
}

// Per-path statistics of an R1 / SPC node: hard decisions written into the
// path's own psum span, the two smallest magnitudes under the (value, index)
// order (select.hpp:18-68) -> st_i1/st_a1, st_i2/st_a2, parity -> st_w.
template <typename R>
__device__ void r1spc_stats(Ctx<R>& cx, int d, int m, int lb, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    if (m < 32) {
        const int lgm = __ffs(m) - 1;
        const int per = 32 >> lgm;
        for (int r0 = 0; r0 < na; r0 += per) {
            const int r = r0 + (cx.lane >> lgm), i = cx.lane & (m - 1);
            const bool ok = r < na;
            const int p = cx.fx->alive_list[ok ? r : 0];
            const M v = ok ? A::val(cx.llr(p, d)[i]) : M(0);
            const unsigned hb = __ballot_sync(FULL, ok && v < M(0));
            uint64_t k1 = ok ? ((uint64_t(A::key(A::mag(v))) << 32) | uint32_t(i)) : ~0ull;
            uint64_t k2 = ~0ull;
            for (int off = 1; off < m; off <<= 1) {
                const uint64_t o1 = shfl_xor64(k1, off), o2 = shfl_xor64(k2, off);
                const uint64_t n1 = umin64(k1, o1);
                k2 = umin64(umax64(k1, o1), umin64(k2, o2));
                k1 = n1;
            }
            if (ok && i == 0) {
                const uint32_t bits = (hb >> (cx.lane & ~(m - 1))) & ((1u << m) - 1u);
                uint32_t* w = cx.row(p) + (lb >> 5);
                const uint32_t mk = ((1u << m) - 1u) << (lb & 31);
                *w = (*w & ~mk) | (bits << (lb & 31));
                cx.fx->st_i1[r] = int(uint32_t(k1));
                cx.fx->st_i2[r] = int(uint32_t(k2));
                cx.fx->st_a1[r] = mbits<M>(A::from_key(uint32_t(k1 >> 32)));
                cx.fx->st_a2[r] = mbits<M>(A::from_key(uint32_t(k2 >> 32)));
                cx.fx->st_w[r] = __popc(bits) & 1;
            }
        }
    } else {
        for (int r = 0; r < na; ++r) {
            const int p = cx.fx->alive_list[r];
            const R* L = cx.llr(p, d);
            uint32_t* w = cx.row(p) + (lb >> 5);
            uint64_t k1 = ~0ull, k2 = ~0ull;
            int par = 0;
            for (int k = 0; k < (m >> 5); ++k) {
                const int i = (k << 5) + cx.lane;
                const M v = A::val(L[i]);
                const unsigned hb = __ballot_sync(FULL, v < M(0));
                if (cx.lane == 0) w[k] = hb;
                par ^= __popc(hb) & 1;
                const uint64_t kv = (uint64_t(A::key(A::mag(v))) << 32) | uint32_t(i);
                if (kv < k1) {
                    k2 = k1;
                    k1 = kv;
                } else if (kv < k2) {
                    k2 = kv;
                }
            }
            for (int off = 1; off < 32; off <<= 1) {
                const uint64_t o1 = shfl_xor64(k1, off), o2 = shfl_xor64(k2, off);
                const uint64_t n1 = umin64(k1, o1);
                k2 = umin64(umax64(k1, o1), umin64(k2, o2));
                k1 = n1;
            }
            if (cx.lane == 0) {
                cx.fx->st_i1[r] = int(uint32_t(k1));
                cx.fx->st_i2[r] = int(uint32_t(k2));
                cx.fx->st_a1[r] = mbits<M>(A::from_key(uint32_t(k1 >> 32)));
                cx.fx->st_a2[r] = mbits<M>(A::from_key(uint32_t(k2 >> 32)));
                cx.fx->st_w[r] = par;
            }
        }
    }
    __syncwarp();
}

// rate-1 node (list_decoder.hpp:254-274): 4 candidates per path
template <typename R, int CPL>
__device__ void list_r1_cands(Ctx<R>& cx, int lb, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    M cm[CPL];
    int cs[CPL], cax[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = cx.lane + 32 * k, r = min(i >> 2, na - 1), j = i & 3;
        const M base = base_of(cx, r);
        const int i1 = cx.fx->st_i1[r], i2 = cx.fx->st_i2[r];
        const M a1 = mfrom<M>(cx.fx->st_a1[r]), a2 = mfrom<M>(cx.fx->st_a2[r]);
        cs[k] = cx.fx->alive_list[r];
        if (j == 0) {
            cm[k] = base;
            cax[k] = pack_aux(-1, -1);
        } else if (j == 1) {
            cm[k] = A::sat(base, a1);
            cax[k] = pack_aux(i1, -1);
        } else if (j == 2) {
            cm[k] = A::sat(base, a2);
            cax[k] = pack_aux(i2, -1);
        } else {
            cm[k] = A::sat(base, A::sat(a1, a2));
            cax[k] = pack_aux(i1, i2);
        }
    }
    fork_apply<R, CPL>(cx, cm, cs, cax, 4 * na, AK_FLIPS, lb, m);
}

// single-parity node (list_decoder.hpp:307-333): 2 candidates per path
template <typename R, int CPL>
__device__ void list_spc_cands(Ctx<R>& cx, int lb, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    M cm[CPL];
    int cs[CPL], cax[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = cx.lane + 32 * k, r = min(i >> 1, na - 1), j = i & 1;
        const M base = base_of(cx, r);
        const int i1 = cx.fx->st_i1[r], i2 = cx.fx->st_i2[r];
        const M a1 = mfrom<M>(cx.fx->st_a1[r]), a2 = mfrom<M>(cx.fx->st_a2[r]);
        cs[k] = cx.fx->alive_list[r];
        if (cx.fx->st_w[r]) { // parity broken: restore it through i1 or i2
            cm[k] = A::sat(base, j == 0 ? a1 : a2);
            cax[k] = pack_aux(j == 0 ? i1 : i2, -1);
        } else if (j == 0) {
            cm[k] = base;
            cax[k] = pack_aux(-1, -1);
        } else {
            cm[k] = A::sat(base, A::sat(a1, a2));
            cax[k] = pack_aux(i1, i2);
        }
    }
    fork_apply<R, CPL>(cx, cm, cs, cax, 2 * na, AK_FLIPS, lb, m);
}

// repetition node (list_decoder.hpp:276-305): 2 candidates per path
template <typename R, int CPL>
__device__ void list_rep_cands(Ctx<R>& cx, int d, int lb, int m, int na) {
    using A = Arith<R>;
    using M = typename A::M;
    // pen_w: sequential sum of the disagreeing magnitudes
    if (cx.lane < na) {
        const R* L = cx.llr(cx.fx->alive_list[cx.lane], d);
        const M s = mfrom<M>(cx.fx->st_a1[cx.lane]);
        const bool w = s < M(0);
        M pen = M(0);
        for (int i = 0; i < m; ++i) {
            const M v = A::val(L[i]);
            if (w ? (v > M(0)) : (v < M(0))) pen = A::sat(pen, A::mag(v));
        }
        cx.fx->st_w[cx.lane] = w;
        cx.fx->st_a2[cx.lane] = mbits<M>(pen);
    }
    __syncwarp();
    M cm[CPL];
    int cs[CPL], cax[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int i = cx.lane + 32 * k, r = min(i >> 1, na - 1), j = i & 1;
        const M base = base_of(cx, r);
        const int w = cx.fx->st_w[r];
        const M pen_w = mfrom<M>(cx.fx->st_a2[r]);
        const M s = mfrom<M>(cx.fx->st_a1[r]);
        cs[k] = cx.fx->alive_list[r];
        if (j == 0) {
            cm[k] = A::sat(base, pen_w);
            cax[k] = pack_aux(w, -1);
        } else {
            cm[k] = A::sat(base, A::sat(pen_w, A::mag(s)));
            cax[k] = pack_aux(w ^ 1, -1);
        }
    }
    fork_apply<R, CPL>(cx, cm, cs, cax, 2 * na, AK_BCAST, lb, m);
}

// ---- CRC syndrome of a decided codeword row ----------------
__device__ uint64_t row_syndrome(const DevCode& C, const uint32_t* row, int lane) {
    uint64_t syn = 0;
    const int nbytes = (C.n + 7) >> 3;
    for (int j = lane; j < nbytes; j += 32) {
        const uint32_t byte = (row[j >> 2] >> ((j & 3) * 8)) & 0xffu;
        syn ^= __ldg(C.crc_tab + (size_t(j) << 8) + byte);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) syn ^= shfl_xor64(syn, off);
    return syn ^ C.crc_c0;
}

// payload (MSB-first bytes of the open positions) + optional codeword
__device__ void write_outputs(const LaunchParams& P, const DevCode& C, const uint32_t* row,
                              int frame, int lane) {
    uint8_t* pay = P.payload + int64_t(frame) * P.payload_stride;
    const int pb = (C.psize + 7) >> 3;
    for (int q = lane; q < pb; q += 32) {
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
        for (int q = lane; q < cb; q += 32) {
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

template <typename R>
__device__ void setup_ctx(Ctx<R>& cx, const LaunchParams& P, const DevCode& C,
                          unsigned char* sm, unsigned char* gs, int frame, int lane, int l) {
    cx.lane = lane;
    cx.n = C.n;
    cx.stages = C.stages;
    cx.l = l;
    cx.lmask = l >= 32 ? FULL : ((1u << l) - 1u);
    cx.chan = static_cast<const R*>(P.llr) + int64_t(frame) * P.llr_stride;
    cx.fx = reinterpret_cast<Fixed*>(sm);
    const Layout Ly = make_layout(C.n, l, int(sizeof(R)), P.seg_smem_max);
    cx.ps = reinterpret_cast<uint32_t*>(sm + Ly.psum_off);
    cx.rw = Ly.rw;
    if (lane >= 1 && lane <= C.stages) {
        unsigned char* base = ((Ly.in_smem >> lane) & 1u) ? sm : gs;
        cx.fx->pool[lane] = reinterpret_cast<uint64_t>(base + Ly.pool_off[lane]);
    }
    if (lane == 0) *reinterpret_cast<uint4*>(cx.fx->bufidx) = make_uint4(0, 0, 0, 0);
    __syncwarp();
    cx.alive = 1u;
    cx.dirty = 0u;
    cx.metric = typename Arith<R>::M(0);
    if (lane == 0) cx.fx->alive_list[0] = 0;
    __syncwarp();
}

__device__ __forceinline__ long long claim(const LaunchParams& P, int lane) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(P.work, 1ull);
    return (long long)__shfl_sync(FULL, idx, 0);
}

// ---- one frame, list decoding at list size P.l --------------------------
template <typename R>
__device__ void list_frame(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                           unsigned char* gs, int frame, int lane) {
    using A = Arith<R>;
    using M = typename A::M;
    Ctx<R> cx;
    setup_ctx(cx, P, C, sm, gs, frame, lane, P.l);
    const uint32_t* sched = C.sched_list;
    const int nops = C.nops_list;
    for (int oi = 0; oi < nops; ++oi) {
        const uint32_t op = __ldg(sched + oi);
        const int code = op_code(op), d = op_depth(op), m = 1 << op_logm(op), lb = op_lb(op);
        const int na = __popc(cx.alive);
        switch (code) {
        case OP_F: op_fg<R, false>(cx, d, m, lb, na); break;
        case OP_G: op_fg<R, true>(cx, d, m, lb, na); break;
        case OP_H: op_h(cx, m, lb, na); break;
        case OP_FROZEN: list_frozen(cx, d, m, lb, na); break;
        case OP_INFO: list_info(cx, d, lb, na); break;
        case OP_R1:
            r1spc_stats(cx, d, m, lb, na);
            if (4 * na <= 32) list_r1_cands<R, 1>(cx, lb, m, na);
            else if (4 * na <= 64) list_r1_cands<R, 2>(cx, lb, m, na);
            else list_r1_cands<R, 4>(cx, lb, m, na);
            cx.normalize();
            break;
        case OP_SPC:
            r1spc_stats(cx, d, m, lb, na);
            if (2 * na <= 32) list_spc_cands<R, 1>(cx, lb, m, na);
            else list_spc_cands<R, 2>(cx, lb, m, na);
            cx.normalize();
            break;
        case OP_REP:
            rep_fold(cx, d, m, na);
            if (2 * na <= 32) list_rep_cands<R, 1>(cx, d, lb, m, na);
            else list_rep_cands<R, 2>(cx, d, lb, m, na);
            cx.normalize();
            break;
        default: break;
        }
    }
    // finish (list_decoder.hpp:457-502): stable order by (metric, slot)
    const bool al = cx.is_alive();
    const uint64_t okey = al ? ((uint64_t(A::key(cx.metric)) << 32) | uint32_t(lane)) : ~0ull;
    uint64_t best = okey;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) best = umin64(best, shfl_xor64(best, off));
    int pick = int(uint32_t(best));
    int crc_ok = 0;
    if (C.crc_width > 0) {
        if (row_syndrome(C, cx.row(pick), lane) == 0) {
            crc_ok = 1;
        } else if (P.select_by_crc) {
            unsigned passm = 0;
            for (unsigned mm = cx.alive & ~(1u << pick); mm; mm &= mm - 1) {
                const int s = __ffs(mm) - 1;
                if (row_syndrome(C, cx.row(s), lane) == 0) passm |= 1u << s;
            }
            if (passm) {
                uint64_t bk = ((passm >> lane) & 1u) ? okey : ~0ull;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) bk = umin64(bk, shfl_xor64(bk, off));
                pick = int(uint32_t(bk));
                crc_ok = 1;
            }
        }
    }
    const M pm = __shfl_sync(FULL, cx.metric, pick);
    write_outputs(P, C, cx.row(pick), frame, lane);
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[frame] = uint8_t(crc_ok);
        if (P.esc) P.esc[frame] = uint8_t(P.esc_level);
        if (P.metric) P.metric[frame] = A::to_float(pm);
        if (P.fail_list && C.crc_width > 0 && !crc_ok) P.fail_list[atomicAdd(P.fail_count, 1)] = frame;
    }
    __syncwarp();
}

// ---- one frame, successive cancellation (sc_decoder.hpp:37-125) ---------
template <typename R>
__device__ void sc_frame(const LaunchParams& P, const DevCode& C, unsigned char* sm,
                         unsigned char* gs, int frame, int lane) {
    using A = Arith<R>;
    using M = typename A::M;
    Ctx<R> cx;
    setup_ctx(cx, P, C, sm, gs, frame, lane, 1);
    uint32_t* row = cx.row(0);
    const uint32_t* sched = C.sched_sc;
    const int nops = C.nops_sc;
    for (int oi = 0; oi < nops; ++oi) {
        const uint32_t op = __ldg(sched + oi);
        const int code = op_code(op), d = op_depth(op), m = 1 << op_logm(op), lb = op_lb(op);
        switch (code) {
        case OP_F: op_fg<R, false>(cx, d, m, lb, 1); break;
        case OP_G: op_fg<R, true>(cx, d, m, lb, 1); break;
        case OP_H: op_h(cx, m, lb, 1); break;
        case OP_FROZEN: span_fill_warp(row, lb, m, 0, lane); __syncwarp(); break;
        case OP_INFO:
            if (lane == 0) span_fill_lane(row, lb, 1, A::val(cx.llr(0, d)[0]) < M(0));
            __syncwarp();
            break;
        case OP_REP: {
            rep_fold(cx, d, m, 1);
            const int bit = mfrom<M>(cx.fx->st_a1[0]) < M(0);
            span_fill_warp(row, lb, m, bit, lane);
            __syncwarp();
            break;
        }
        default: break;
        }
    }
    int crc_ok = 0;
    if (C.crc_width > 0) crc_ok = row_syndrome(C, row, lane) == 0;
    write_outputs(P, C, row, frame, lane);
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[frame] = uint8_t(crc_ok);
        if (P.esc) P.esc[frame] = 1;
        if (P.metric) P.metric[frame] = 0.0f; // DecodeResult default (decode_result.hpp:12)
        if (P.fail_list && C.crc_width > 0 && !crc_ok) P.fail_list[atomicAdd(P.fail_count, 1)] = frame;
    }
    __syncwarp();
}

template <typename R, bool LIST>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) decode_kernel(const LaunchParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = int64_t(blockIdx.x) * kWarpsPerBlock + wib;
    unsigned char* sm = smem_raw + wib * P.smem_per_warp;
    unsigned char* gs = static_cast<unsigned char*>(P.gscratch) + gw * P.gscratch_per_warp;
    const long long count = P.frame_list ? (long long)(*P.frame_count) : (long long)P.nframes;
    for (;;) {
        const long long idx = claim(P, lane);
        if (idx >= count) break;
        const int frame = P.frame_list ? P.frame_list[idx] : int(idx);
        const int cid = P.code_id ? P.code_id[frame] : 0;
        const DevCode C = P.codes[cid];
        if constexpr (LIST) list_frame<R>(P, C, sm, gs, frame, lane);
        else sc_frame<R>(P, C, sm, gs, frame, lane);
    }
}

template <typename R, bool LIST>
cudaError_t launch(const LaunchParams& p, int grid, cudaStream_t s) {
    const int smem = p.smem_per_warp * kWarpsPerBlock;
    auto kern = decode_kernel<R, LIST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kWarpsPerBlock * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <typename R, bool LIST>
int occupancy(int smem) {
    auto kern = decode_kernel<R, LIST>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kWarpsPerBlock * 32, smem) != cudaSuccess)
        return 0;
    return nb;
}

} // namespace

int64_t smem_bytes_per_warp(int nmax, int l, int elem_bytes, int seg_smem_max) {
    return make_layout(nmax, l, elem_bytes, seg_smem_max).smem_total;
}
int64_t gscratch_bytes_per_warp(int nmax, int l, int elem_bytes, int seg_smem_max) {
    return make_layout(nmax, l, elem_bytes, seg_smem_max).gmem_total;
}

cudaError_t launch_sc(const LaunchParams& p, int precision, int grid, cudaStream_t s) {
    return precision == 0 ? launch<float, false>(p, grid, s) : launch<int8_t, false>(p, grid, s);
}
cudaError_t launch_list(const LaunchParams& p, int precision, int grid, cudaStream_t s) {
    return precision == 0 ? launch<float, true>(p, grid, s) : launch<int8_t, true>(p, grid, s);
}
int occupancy_sc(int precision, int smem) {
    return precision == 0 ? occupancy<float, false>(smem) : occupancy<int8_t, false>(smem);
}
int occupancy_list(int precision, int smem) {
    return precision == 0 ? occupancy<float, true>(smem) : occupancy<int8_t, true>(smem);
}

} // namespace plb
