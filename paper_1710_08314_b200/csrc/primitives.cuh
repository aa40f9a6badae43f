// Device primitives of the sm_100a decoder kernels: sub-warp collectives,
// the reference's per-representation arithmetic (llr.hpp:36-69) and its
// int8 SWAR form, sorting networks, vector access and L2 cache policies.
//
// A fragment of kernels.cu: included inside namespace plb::{anonymous}
// (one translation unit, so every helper inlines into the kernels).
#pragma once
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }

__device__ __forceinline__ int pack_aux(int a, int b) {
    return int((uint32_t(a) & 0xffffu) | (uint32_t(b) << 16));
}

// ---- sub-warp collectives ----------------------------------------------
// All calls are made by all 32 lanes of the warp (every sub-warp executes
// the same control flow); results are per sub-warp.
template <int SW>
struct Sub {
    static constexpr unsigned kMask = SW == 32 ? FULL : ((1u << SW) - 1u);
    int lane; // lane within the sub-warp
    int base; // first warp lane of the sub-warp
    int id;   // sub-warp index

    __device__ __forceinline__ unsigned ballot(bool p) const {
        if constexpr (SW == 32) return __ballot_sync(FULL, p);
        else return (__ballot_sync(FULL, p) >> base) & kMask;
    }
    __device__ __forceinline__ bool any(bool p) const { return ballot(p) != 0u; }
    __device__ __forceinline__ unsigned lt() const { return lanemask_lt() >> base; }
    __device__ __forceinline__ uint32_t shfl(uint32_t v, int src) const { return __shfl_sync(FULL, v, src, SW); }
    __device__ __forceinline__ int shfl(int v, int src) const { return __shfl_sync(FULL, v, src, SW); }
    __device__ __forceinline__ float shfl(float v, int src) const { return __shfl_sync(FULL, v, src, SW); }
    __device__ __forceinline__ uint64_t shfl(uint64_t v, int src) const {
        const uint32_t lo = __shfl_sync(FULL, uint32_t(v), src, SW);
        const uint32_t hi = __shfl_sync(FULL, uint32_t(v >> 32), src, SW);
        return (uint64_t(hi) << 32) | lo;
    }
    // OR of slot masks (v < 2^SW): every sub-warp's mask in its own SW-bit
    // field of one warp-wide redux
    __device__ __forceinline__ unsigned red_or(unsigned v) const {
        if constexpr (SW == 32) return __reduce_or_sync(FULL, v);
        else return (__reduce_or_sync(FULL, v << base) >> base) & kMask;
    }
    __device__ __forceinline__ unsigned red_min(unsigned v) const {
        if constexpr (SW == 32) {
            return __reduce_min_sync(FULL, v);
        } else {
#pragma unroll
            for (int o = SW / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
            return v;
        }
    }
    __device__ __forceinline__ unsigned red_add(unsigned v) const {
        if constexpr (SW == 32) {
            return __reduce_add_sync(FULL, v);
        } else {
#pragma unroll
            for (int o = SW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
            return v;
        }
    }
    // lanes of this sub-warp holding the same v (v < 2^24)
    __device__ __forceinline__ unsigned match(int v) const {
        if constexpr (SW == 32) return __match_any_sync(FULL, v);
        else return (__match_any_sync(FULL, (v << 2) | id) >> base) & kMask;
    }
};

__device__ __forceinline__ uint32_t shfl_xor_k(uint32_t v, int m) { return __shfl_xor_sync(FULL, v, m); }
__device__ __forceinline__ uint64_t shfl_xor_k(uint64_t v, int m) {
    const uint32_t lo = __shfl_xor_sync(FULL, uint32_t(v), m);
    const uint32_t hi = __shfl_xor_sync(FULL, uint32_t(v >> 32), m);
    return (uint64_t(hi) << 32) | lo;
}

// ---- per-representation arithmetic (llr.hpp:36-69) -------------------
// Key: a totally ordered (value, index) pair in one integer, used for the
// stable candidate ranking and for the two-smallest selection.
template <typename R>
struct Arith;

template <>
struct Arith<float> {
    using M = float;      // path-metric type
    using Key = uint64_t; // float bits << 32 | index  (value >= +0)
    static constexpr bool kFixed = false;
    static constexpr int kMax = 0; // (fixed point only: no saturation)
    static constexpr Key kKeyMax = ~0ull;
    __device__ static M sat(M a, M b) { return a + b; }
    // |v| as a non-negative float: abs_llr(-0.0f) is -0.0f in the reference,
    // but every use of a magnitude is an add to a non-negative metric or a
    // (value, index) comparison, where +-0 behave identically.
    __device__ static M mag(float v) { return fabsf(v); }
    __device__ static Key make_key(M v, int idx) { return (uint64_t(__float_as_uint(v)) << 32) | uint32_t(idx); }
    __device__ static int key_idx(Key k) { return int(uint32_t(k)); }
    __device__ static M key_val(Key k) { return __uint_as_float(uint32_t(k >> 32)); }
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
    using Key = uint32_t; // value (0..127) << 16 | index
    static constexpr bool kFixed = true;
    static constexpr int kMax = 127; // symmetric range (llr.hpp:29-33)
    static constexpr Key kKeyMax = ~0u;
    __device__ static M sat(M a, M b) { return max(-127, min(127, a + b)); }
    __device__ static M mag(int v) { return abs(v); }
    __device__ static Key make_key(M v, int idx) { return (uint32_t(v) << 16) | uint32_t(idx); }
    __device__ static int key_idx(Key k) { return int(k & 0xffffu); }
    __device__ static M key_val(Key k) { return int(k >> 16); }
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

// int16 (llr.hpp:22-26): the int8 rules on [-32767, 32767], scalar f / g
template <>
struct Arith<int16_t> {
    using M = int;
    using Key = uint32_t; // value (0..32767) << 16 | index
    static constexpr bool kFixed = true;
    static constexpr int kMax = 32767;
    static constexpr Key kKeyMax = ~0u;
    __device__ static M sat(M a, M b) { return max(-kMax, min(kMax, a + b)); }
    __device__ static M mag(int v) { return abs(v); }
    __device__ static Key make_key(M v, int idx) { return (uint32_t(v) << 16) | uint32_t(idx); }
    __device__ static int key_idx(Key k) { return int(k & 0xffffu); }
    __device__ static M key_val(Key k) { return int(k >> 16); }
    __device__ static M val(int16_t v) { return int(v); }
    __device__ static int16_t f(int16_t a, int16_t b) {
        const int m = min(abs(int(a)), abs(int(b)));
        return int16_t(((a ^ b) < 0) ? -m : m);
    }
    __device__ static int16_t g(int16_t a, int16_t b, uint32_t s) {
        const int v = s ? int(b) - int(a) : int(a) + int(b);
        return int16_t(max(-kMax, min(kMax, v)));
    }
    __device__ static int16_t store(M v) { return int16_t(v); }
    __device__ static float to_float(M v) { return float(v); }
};

// ---- int8 f / g on four packed values (SWAR) ---------------------------
// Bit-exact with Arith<int8_t>::f / ::g for operands in [-127, 127]; checked
// exhaustively by pl_kernel_selftest.
// f: |x| = absdiff_u8(x ^ 0x80, 0x80); min(p, q) = (p + q - |p - q|) / 2
// (bytes <= 127: no carries); the result is negated (two's complement, no
// carry for m >= 1) where the operand signs differ and m != 0.
// PRMT with the selector's sign-replicate bit (__byte_perm masks it away)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ uint32_t f_swar(uint32_t a, uint32_t b) {
    const uint32_t aa = __vabsdiffu4(a ^ 0x80808080u, 0x80808080u);
    const uint32_t ab = __vabsdiffu4(b ^ 0x80808080u, 0x80808080u);
    const uint32_t m = (((aa + ab) - __vabsdiffu4(aa, ab)) >> 1) & 0x7f7f7f7fu;
    const uint32_t sp = (a ^ b) & (m + 0x7f7f7f7fu) & 0x80808080u;
    return (m ^ prmt(sp, 0, 0xba98)) + (sp >> 7);
}
// g in two 16x2 halves: sign-extend, b + (s ? -a : a), clamp to [-127, 127]
// (the reference clamps to the symmetric range, llr.hpp:61-69), repack.
// s4 = the four partial-sum bits, element i in bit i.
__device__ __forceinline__ uint32_t g_swar(uint32_t a, uint32_t b, uint32_t s4) {
    const uint32_t al = prmt(a, 0, 0x9180), ah = prmt(a, 0, 0xb3a2);
    const uint32_t bl = prmt(b, 0, 0x9180), bh = prmt(b, 0, 0xb3a2);
    const uint32_t t = ((s4 * 0x00204081u) & 0x01010101u) << 7; // bit 7 of byte i = s_i
    const uint32_t ml = prmt(t, 0, 0x9988), mh = prmt(t, 0, 0xbbaa);
    uint32_t vl = __vadd2(__vadd2(al ^ ml, bl), ml & 0x00010001u);
    uint32_t vh = __vadd2(__vadd2(ah ^ mh, bh), mh & 0x00010001u);
    vl = __vmins2(__vmaxs2(vl, 0xff81ff81u), 0x007f007fu);
    vh = __vmins2(__vmaxs2(vh, 0xff81ff81u), 0x007f007fu);
    return __byte_perm(vl, vh, 0x6420);
}

// int16 f on two packed values (16x2 SIMD): |x| = max(x, ~x + 1) per lane
// (VIADDMNMX.S16x2), the smaller magnitude by VIMNMX.U16x2, negated
// (two's complement per lane, no carry across lanes) where the operand
// signs differ.  Bit-exact with Arith<int16_t>::f for operands in
// [-32767, 32767] (pl_kernel_selftest); 10 instructions per 2 values
// instead of 19.
__device__ __forceinline__ uint32_t f_swar16(uint32_t a, uint32_t b) {
    const uint32_t aa = __vmaxs2(a, __vadd2(~a, 0x00010001u));
    const uint32_t ab = __vmaxs2(b, __vadd2(~b, 0x00010001u));
    const uint32_t m = __vminu2(aa, ab);
    const uint32_t mk = prmt((a ^ b) & 0x80008000u, 0, 0xBB99); // sign -> 0xffff per lane
    return __vadd2(m ^ mk, mk & 0x00010001u);
}

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

// ---- sub-warp sorting networks (ascending) -------------------------------
// Every network here uses ascending comparators only: a bitonic merge whose
// first stage compares mirrored lanes (lane ^ (size-1)) merges two ASCENDING
// runs, so runs that are already sorted need no direction flips and their
// phases are skipped.  The candidates of one path are emitted in ascending
// (metric, index) order for R1, SPC and REP nodes (their penalties are
// 0 <= a1 <= a2 <= a1+a2 resp. pen_w <= pen_w+|s|, list_decoder.hpp:254-333),
// which makes each path's 2 or 4 consecutive lanes a sorted run.
// compare-exchange with lane ^ m: lanes with `bit` clear keep the smaller key
template <typename K>
__device__ __forceinline__ K cex(K key, int m, int lane, int bit) {
    const K o = shfl_xor_k(key, m);
    return (lane & bit) == 0 ? kmin(key, o) : kmax(key, o);
}

// W keys, one per lane, made of sorted runs of 2^lgrun lanes (lgrun uniform;
// 0 = unsorted): lanes [0, W) of each aligned W-lane group sorted ascending.
template <typename K, int W>
__device__ __forceinline__ K sort_runs(K key, int lane, int lgrun) {
#pragma unroll
    for (int size = 2; size <= W; size <<= 1) {
        if (size <= (1 << lgrun)) continue;
        key = cex(key, size - 1, lane, size >> 1);
#pragma unroll
        for (int j = size >> 2; j > 0; j >>= 1) key = cex(key, j, lane, j);
    }
    return key;
}

// The W/2 smallest of 2W keys (two registers, sorted runs of 2^lgrun),
// ascending in lanes [0, W/2): sort W/2-lane runs in both registers, keep the
// W/2 smallest of each pair of runs (min against the other register's run
// reversed: a bitonic sequence), sort those, then the same step across the
// two halves.  14 compare stages at W = 16 from runs of 4, vs 25 for two full
// sorts and a merge.
template <typename K, int W>
__device__ __forceinline__ K top_half2(K a, K b, int lane, int lgrun) {
    // both registers through the same stages (one uniform branch per phase,
    // two independent chains)
#pragma unroll
    for (int size = 2; size <= W / 2; size <<= 1) {
        if (size <= (1 << lgrun)) continue;
        a = cex(a, size - 1, lane, size >> 1);
        b = cex(b, size - 1, lane, size >> 1);
#pragma unroll
        for (int j = size >> 2; j > 0; j >>= 1) {
            a = cex(a, j, lane, j);
            b = cex(b, j, lane, j);
        }
    }
    K c = kmin(a, shfl_xor_k(b, W / 2 - 1));
#pragma unroll
    for (int j = W / 4; j > 0; j >>= 1) c = cex(c, j, lane, j);
    c = cex(c, W - 1, lane, W / 2);
#pragma unroll
    for (int j = W / 4; j > 0; j >>= 1) c = cex(c, j, lane, j);
    return c;
}

// The W smallest of two ascending W-key lane sequences, ascending: the
// element-wise min of a and reversed b is a bitonic sequence holding exactly
// those keys; half-cleaners sort it.
template <typename K, int W>
__device__ __forceinline__ K merge_top(K a, K b, int lane) {
    K c = kmin(a, shfl_xor_k(b, W - 1));
#pragma unroll
    for (int j = W / 2; j > 0; j >>= 1) c = cex(c, j, lane, j);
    return c;
}

// The W smallest of W*C keys (register k of each lane), ascending in
// register 0: sort each register across the lanes, then merge pairwise.
// Registers from nreg on hold only kKeyMax and are skipped (uniform).
template <typename K, int C, int W>
__device__ __forceinline__ void top_regs(K (&key)[C], int lane, int nreg, int lgrun) {
#pragma unroll
    for (int k = 0; k < C; ++k)
        if (k < nreg) key[k] = sort_runs<K, W>(key[k], lane, lgrun);
#pragma unroll
    for (int w = 1; w < C; w <<= 1)
#pragma unroll
        for (int k = 0; k + w < C; k += 2 * w)
            if (k + w < nreg) key[k] = merge_top<K, W>(key[k], key[k + w], lane);
}

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

// L2 eviction-priority hints of the frame-per-lane SC pass (global memory only)
__device__ __forceinline__ uint64_t l2_policy(int cls) { // 2 evict_last, 1 evict_normal, 0 evict_first
    uint64_t p;
    if (cls == 2) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (cls == 1) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <typename R, int G>
__device__ __forceinline__ Vec<R, G> vld_hint(const R* ptr, uint64_t pol) {
    static_assert(G * sizeof(R) == 16, "16-byte vectors");
    Vec<R, G> x;
    uint4 v;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(ptr), "l"(pol));
    x.raw = *reinterpret_cast<const typename VT<16>::T*>(&v);
    return x;
}
template <typename R, int G>
__device__ __forceinline__ void vst_hint(R* ptr, const Vec<R, G>& x, uint64_t pol) {
    static_assert(G * sizeof(R) == 16, "16-byte vectors");
    const uint4 v = *reinterpret_cast<const uint4*>(&x.raw);
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

#ifdef PLB_OPTIME
__device__ unsigned long long g_optime[64]; // profiling build: cycles / count per op kind
#endif

// per-frame decode time (LaunchParams::lat_ns): the device's global timer
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// first channel LLR of a frame: fixed stride, or the packed layout's offset
template <typename R>
__device__ __forceinline__ const R* frame_llr(const LaunchParams& P, int frame) {
    return static_cast<const R*>(P.llr) + (P.llr_offset ? P.llr_offset[frame] : int64_t(frame) * P.llr_stride);
}
