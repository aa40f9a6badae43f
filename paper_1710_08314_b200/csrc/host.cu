// Host side of the C ABI (include/polar_b200.h): validation, decode tree
// and schedule construction, CRC syndrome tables, device residency of the
// per-code tables, and the per-kind launch sequence including the fully
// adaptive ladder (decoders.hpp:60-85) as stream-ordered rungs over
// compacted frame lists.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cctype>
#include <climits>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/polar_b200.h"
#include "polar_dev.h"

namespace {

thread_local std::string g_thread_err;

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- CRC engine (crc.cpp:86-154 semantics) ------------------------------
uint64_t bit_reverse(uint64_t v, int width) {
    uint64_t r = 0;
    for (int i = 0; i < width; ++i) {
        r = (r << 1) | (v & 1);
        v >>= 1;
    }
    return r;
}

struct Crc {
    pl_crc spec{};
    uint64_t table[256]{};
    uint64_t rpoly = 0, poly_top = 0, init_reg = 0;

    explicit Crc(const pl_crc& s) : spec(s) {
        if (s.width < 1 || s.width > 64)
            throw ConfigError("CRC width must be in [1, 64], got " + std::to_string(s.width));
        const uint64_t mask = s.width == 64 ? ~0ull : ((1ull << s.width) - 1);
        if ((s.poly & ~mask) || (s.init & ~mask) || (s.xorout & ~mask))
            throw ConfigError("CRC poly/init/xorout do not fit in " + std::to_string(s.width) +
                              " bits");
        if ((s.poly & 1) == 0) throw ConfigError("CRC poly must have its x^0 term set");
        if (s.reflect) {
            rpoly = bit_reverse(s.poly, s.width);
            init_reg = bit_reverse(s.init, s.width);
            for (int b = 0; b < 256; ++b) {
                uint64_t r = uint64_t(b);
                for (int i = 0; i < 8; ++i) r = (r >> 1) ^ ((r & 1) ? rpoly : 0);
                table[b] = r;
            }
        } else {
            poly_top = s.poly << (64 - s.width);
            init_reg = s.init << (64 - s.width);
            for (int b = 0; b < 256; ++b) {
                uint64_t r = uint64_t(b) << 56;
                for (int i = 0; i < 8; ++i) {
                    const bool top = r >> 63;
                    r <<= 1;
                    if (top) r ^= poly_top;
                }
                table[b] = r;
            }
        }
    }

    // bits one per byte, index order; whole bytes MSB-first through the table,
    // trailing bits folded one at a time
    uint64_t compute(const uint8_t* bits, size_t len) const {
        uint64_t reg = init_reg;
        const size_t nbytes = len / 8;
        auto byte_at = [&](size_t k) {
            unsigned v = 0;
            for (int j = 0; j < 8; ++j) v = (v << 1) | (bits[8 * k + j] & 1u);
            return v;
        };
        if (spec.reflect) {
            for (size_t k = 0; k < nbytes; ++k) reg = (reg >> 8) ^ table[(reg ^ byte_at(k)) & 0xFF];
            for (size_t i = nbytes * 8; i < len; ++i) {
                reg ^= uint64_t(bits[i] & 1u);
                const bool lo = reg & 1;
                reg >>= 1;
                if (lo) reg ^= rpoly;
            }
            return reg ^ spec.xorout;
        }
        for (size_t k = 0; k < nbytes; ++k)
            reg = (reg << 8) ^ table[((reg >> 56) ^ byte_at(k)) & 0xFF];
        for (size_t i = nbytes * 8; i < len; ++i) {
            reg ^= uint64_t(bits[i] & 1u) << 63;
            const bool top = reg >> 63;
            reg <<= 1;
            if (top) reg ^= poly_top;
        }
        return (reg >> (64 - spec.width)) ^ spec.xorout;
    }
};

pl_crc parse_crc(const std::string& text) {
    if (text == "32-GZIP") return pl_crc{32, 1, 0x04C11DB7, 0xFFFFFFFF, 0xFFFFFFFF};
    if (text == "16-CCITT") return pl_crc{16, 0, 0x1021, 0xFFFF, 0x0000};
    if (text == "8") return pl_crc{8, 0, 0x07, 0x00, 0x00};
    std::vector<std::string> f(1);
    for (char c : text) {
        if (c == ':') f.emplace_back();
        else f.back().push_back(c);
    }
    if (f.size() != 5)
        throw ParseError("CRC spec '" + text +
                         "': expected a preset name or width:poly:reflect:init:xorout");
    auto hex = [](const std::string& s, const char* what) {
        if (s.empty()) throw ParseError(std::string("CRC spec: empty ") + what + " field");
        size_t pos = 0;
        uint64_t v = 0;
        try {
            v = std::stoull(s, &pos, 16);
        } catch (const std::exception&) {
            throw ParseError("CRC spec: bad hex value '" + s + "' for " + what);
        }
        if (pos != s.size()) throw ParseError("CRC spec: bad hex value '" + s + "' for " + what);
        return v;
    };
    pl_crc c{};
    try {
        size_t pos = 0;
        c.width = std::stoi(f[0], &pos, 10);
        if (pos != f[0].size()) throw std::invalid_argument("");
    } catch (const std::exception&) {
        throw ParseError("CRC spec: bad width '" + f[0] + "'");
    }
    c.poly = hex(f[1], "poly");
    if (f[2] == "0") c.reflect = 0;
    else if (f[2] == "1") c.reflect = 1;
    else throw ParseError("CRC spec: reflect field must be 0 or 1, got '" + f[2] + "'");
    c.init = hex(f[3], "init");
    c.xorout = hex(f[4], "xorout");
    return c;
}

// ---- decode tree (prune_tree.cpp:38-71) --------------------------------
enum Kind : int { NK_BRANCH, NK_FROZEN, NK_INFO, NK_R0, NK_R1, NK_REP, NK_SPC };

struct Node {
    int kind, depth, lb, size, left, right;
};

void check_pruning(const pl_pruning& c) {
    if (c.rep_max < 0 || c.spc_max < 0 || (c.rep_max && c.rep_max < 2) || (c.spc_max && c.spc_max < 4))
        throw ConfigError("node size caps must be 0 (unlimited), >= 2 for repetition and >= 4 for "
                          "single-parity");
}

int build_tree(std::vector<Node>& out, const uint8_t* frozen, int lo, int size, int depth,
               const pl_pruning& c) {
    const int idx = int(out.size());
    out.push_back(Node{NK_BRANCH, depth, lo, size, -1, -1});
    int nfrozen = 0;
    for (int i = 0; i < size; ++i) nfrozen += frozen[lo + i] != 0;
    int kind = NK_BRANCH;
    if (size == 1) kind = nfrozen ? NK_FROZEN : NK_INFO;
    else if (c.repetition && nfrozen == size - 1 && !frozen[lo + size - 1] &&
             (c.rep_max == 0 || size <= c.rep_max))
        kind = NK_REP;
    else if (c.single_parity && nfrozen == 1 && frozen[lo] && (c.spc_max == 0 || size <= c.spc_max))
        kind = NK_SPC;
    else if (c.rate_zero && nfrozen == size) kind = NK_R0;
    else if (c.rate_one && nfrozen == 0) kind = NK_R1;
    out[size_t(idx)].kind = kind;
    if (kind == NK_BRANCH && size > 1) {
        const int l = build_tree(out, frozen, lo, size / 2, depth + 1, c);
        const int r = build_tree(out, frozen, lo + size / 2, size / 2, depth + 1, c);
        out[size_t(idx)].left = l;
        out[size_t(idx)].right = r;
    }
    return idx;
}

int ilog2i(int v) {
    int r = 0;
    while ((1 << r) < v) ++r;
    return r;
}

// list schedule: the walk of list_decoder.hpp:174-224.  A leaf child of at
// most fuse_max values replaces its parent's F (G) op: the leaf op computes
// its LLRs in registers (kOpFused), which skips a round trip through the
// depth pool and an op.
// big_r1: rate-1 / single-parity right children of any larger size are
// fused with the parent's G op as well (r1spc_stats forms their LLRs from the
// parent segment; 0 = off).
void emit_list(const std::vector<Node>& t, int ni, std::vector<uint32_t>& s, int fuse_max, bool big_r1) {
    const Node& nd = t[size_t(ni)];
    const int lg = ilog2i(nd.size);
    auto fusable = [&](int ci, bool right = false) {
        const Node& c = t[size_t(ci)];
        if (c.kind == NK_BRANCH) return false;
        if (c.size <= fuse_max) return true;
        return right && big_r1 && (c.kind == NK_R1 || c.kind == NK_SPC);
    };
    switch (nd.kind) {
    case NK_BRANCH:
        if (fusable(nd.left)) {
            emit_list(t, nd.left, s, fuse_max, big_r1);
            s.back() |= plb::kOpFused;
        } else {
            s.push_back(plb::op_pack(plb::OP_F, nd.depth, lg, nd.lb));
            emit_list(t, nd.left, s, fuse_max, big_r1);
        }
        if (fusable(nd.right, true)) {
            emit_list(t, nd.right, s, fuse_max, big_r1);
            s.back() |= plb::kOpFused | plb::kOpFusedG;
        } else {
            s.push_back(plb::op_pack(plb::OP_G, nd.depth, lg, nd.lb));
            emit_list(t, nd.right, s, fuse_max, big_r1);
        }
        s.push_back(plb::op_pack(plb::OP_H, nd.depth, lg, nd.lb));
        break;
    case NK_FROZEN:
    case NK_R0: s.push_back(plb::op_pack(plb::OP_FROZEN, nd.depth, lg, nd.lb)); break;
    case NK_INFO: s.push_back(plb::op_pack(plb::OP_INFO, nd.depth, lg, nd.lb)); break;
    case NK_R1: s.push_back(plb::op_pack(plb::OP_R1, nd.depth, lg, nd.lb)); break;
    case NK_REP: s.push_back(plb::op_pack(plb::OP_REP, nd.depth, lg, nd.lb)); break;
    case NK_SPC: s.push_back(plb::op_pack(plb::OP_SPC, nd.depth, lg, nd.lb)); break;
    }
}

// List schedules: an F / G op directly followed by the F op of its child
// (the left descent) takes that F along (kOpChain; the F op is dropped) when
// the child's output still holds whole 16-byte chunks (h / 2 >= ve values).
void chain_list_ops(std::vector<uint32_t>& s, int ve) {
    std::vector<uint32_t> out;
    out.reserve(s.size());
    for (size_t i = 0; i < s.size(); ++i) {
        const uint32_t w = s[i];
        const int code = plb::op_code(w);
        const bool plain = (w & (plb::kOpFused | plb::kOpFusedG)) == 0;
        if (plain && (code == plb::OP_F || code == plb::OP_G) && i + 1 < s.size()) {
            const uint32_t nx = s[i + 1];
            const int h = (1 << plb::op_logm(w)) >> 1;
            if (plb::op_code(nx) == plb::OP_F && (nx & (plb::kOpFused | plb::kOpFusedG)) == 0 &&
                plb::op_depth(nx) == plb::op_depth(w) + 1 && (h >> 1) >= ve) {
                out.push_back(w | plb::kOpChain);
                ++i;
                continue;
            }
        }
        out.push_back(w);
    }
    s.swap(out);
}

// a subtree of size <= 32 as one register-level SC op + its frozen mask
void emit_scsub(int depth, int m, int lb, const uint8_t* frozen, std::vector<uint32_t>& s) {
    uint32_t mask = 0;
    for (int i = 0; i < m; ++i)
        if (frozen[lb + i]) mask |= 1u << i;
    s.push_back(plb::op_pack(plb::OP_SCSUB, depth, ilog2i(m), lb));
    s.push_back(mask);
}

// unabridged recursion of sc_decoder.hpp:99-112
void emit_sc_subtree(int depth, int m, int base, int frozen_at, std::vector<uint32_t>& s,
                     int sub_max) {
    if (m <= sub_max && m >= 2) {
        uint32_t mask = 0;
        if (frozen_at >= base && frozen_at < base + m) mask = 1u << (frozen_at - base);
        s.push_back(plb::op_pack(plb::OP_SCSUB, depth, ilog2i(m), base));
        s.push_back(mask);
        return;
    }
    if (m == 1) {
        s.push_back(plb::op_pack(base == frozen_at ? plb::OP_FROZEN : plb::OP_INFO, depth, 0, base));
        return;
    }
    const int lg = ilog2i(m);
    s.push_back(plb::op_pack(plb::OP_F, depth, lg, base));
    emit_sc_subtree(depth + 1, m / 2, base, frozen_at, s, sub_max);
    s.push_back(plb::op_pack(plb::OP_G, depth, lg, base));
    emit_sc_subtree(depth + 1, m / 2, base + m / 2, frozen_at, s, sub_max);
    s.push_back(plb::op_pack(plb::OP_H, depth, lg, base));
}

// SC schedule: the walk of sc_decoder.hpp:58-94.  Branch subtrees of size
// <= 32 become one OP_SCSUB (unpruned SC recursion; the R0 / REP shortcuts
// inside them decide identically, the reference's own SSC == SC property,
// test_sc.cpp:39-74).  sub_max = 0: no OP_SCSUB (the frame-per-lane SC
// kernel walks every op per lane).
void emit_sc(const std::vector<Node>& t, int ni, std::vector<uint32_t>& s,
             const uint8_t* frozen, int sub_max = plb::kScSubMax, bool lane = false) {
    const Node& nd = t[size_t(ni)];
    const int lg = ilog2i(nd.size);
    // (lane schedules: a small rate-1 node is a subtree op with no frozen
    // position; the op takes the hard-decision shortcut itself)
    if ((nd.kind == NK_BRANCH || (lane && nd.kind == NK_R1)) && nd.size <= sub_max && nd.size >= 2) {
        emit_scsub(nd.depth, nd.size, nd.lb, frozen, s);
        return;
    }
    switch (nd.kind) {
    case NK_BRANCH:
        s.push_back(plb::op_pack(plb::OP_F, nd.depth, lg, nd.lb));
        emit_sc(t, nd.left, s, frozen, sub_max, lane);
        s.push_back(plb::op_pack(plb::OP_G, nd.depth, lg, nd.lb));
        emit_sc(t, nd.right, s, frozen, sub_max, lane);
        s.push_back(plb::op_pack(plb::OP_H, nd.depth, lg, nd.lb));
        break;
    case NK_FROZEN:
    case NK_R0: s.push_back(plb::op_pack(plb::OP_FROZEN, nd.depth, lg, nd.lb)); break;
    case NK_INFO: s.push_back(plb::op_pack(plb::OP_INFO, nd.depth, lg, nd.lb)); break;
    case NK_R1: {
        // Rate-1 shortcut: f keeps the sign product with magnitude min(|a|,|b|)
        // and, given the left child's hard decisions, g adds magnitudes, so
        // with no zero input LLR no zero ever appears and the unabridged
        // recursion returns exactly hard(L).  Zero inputs run the recursion.
        s.push_back(plb::op_pack(plb::OP_R1SC, nd.depth, lg, nd.lb));
        const size_t at = s.size();
        s.push_back(0);
        emit_sc_subtree(nd.depth, nd.size, nd.lb, -1, s, sub_max);
        s[at] = uint32_t(s.size() - at - 1);
        break;
    }
    case NK_SPC: emit_sc_subtree(nd.depth, nd.size, nd.lb, nd.lb, s, sub_max); break;
    case NK_REP: s.push_back(plb::op_pack(plb::OP_REP, nd.depth, lg, nd.lb)); break;
    }
}

// Lane schedules: an F / G op whose next ops are F ops (the left descent
// below its child) takes up to jmax of them along: the op computes its own
// output chunk group and the F levels below it in registers and stores every
// level, so the chained F ops never read their input segment back
// (kOpChainShift bits of the op word = the number of chained F ops, which are
// dropped from the schedule).  Level j's segment must still hold whole
// 16-byte chunks: (m / 2) >> J >= ve values.  R1SC skip lengths are
// recomputed for the shortened expansions.
void fuse_lane_chains(const std::vector<uint32_t>& in, size_t lo, size_t hi,
                      std::vector<uint32_t>& out, int ve, int jmax, int jmax0, bool gr1, bool subf) {
    size_t i = lo;
    while (i < hi) {
        const uint32_t w = in[i];
        const int code = plb::op_code(w);
        if (gr1 && code == plb::OP_G && i + 2 < hi && plb::op_code(in[i + 1]) == plb::OP_R1SC &&
            plb::op_depth(in[i + 1]) == plb::op_depth(w) + 1 && (1 << plb::op_logm(w)) >= 64) {
            // G + rate-1 child: OP_GR1, count, then the plain G and the
            // expanded recursion of the child (taken when a g value is zero)
            out.push_back((w & ~15u) | plb::OP_GR1);
            const size_t at = out.size();
            out.push_back(0);
            out.push_back(w);
            const size_t len = in[i + 2];
            fuse_lane_chains(in, i + 3, i + 3 + len, out, ve, jmax, jmax0, gr1, subf);
            out[at] = uint32_t(out.size() - at - 1);
            i += 3 + len;
        } else if (code == plb::OP_SCSUB) {
            out.push_back(w);
            out.push_back(in[i + 1]);
            i += 2;
        } else if (code == plb::OP_R1SC) {
            out.push_back(w);
            const size_t at = out.size();
            out.push_back(0);
            const size_t len = in[i + 1];
            fuse_lane_chains(in, i + 2, i + 2 + len, out, ve, jmax, jmax0, gr1, subf);
            out[at] = uint32_t(out.size() - at - 1);
            i += 2 + len;
        } else if (subf && (code == plb::OP_F || code == plb::OP_G) && i + 2 < hi &&
                   plb::op_code(in[i + 1]) == plb::OP_SCSUB && plb::op_depth(in[i + 1]) == plb::op_depth(w) + 1) {
            // an in-register subtree takes its parent's F / G op along: its
            // LLRs come straight from the parent's values (lanes.cuh lane_sub)
            out.push_back(in[i + 1] | plb::kOpFused | (code == plb::OP_G ? plb::kOpFusedG : 0u));
            out.push_back(in[i + 2]);
            i += 3;
        } else if (code == plb::OP_F && i + 1 < hi && plb::op_code(in[i + 1]) == plb::OP_FROZEN &&
                   plb::op_depth(in[i + 1]) == plb::op_depth(w) + 1) {
            // the left child is a rate-0 node: SC decides it without its LLRs
            // (sc_decoder.hpp:80-83), so the F op that would form them is dropped
            ++i;
        } else if (code == plb::OP_F || code == plb::OP_G) {
            const int h = (1 << plb::op_logm(w)) >> 1;
            int j = 0;
            const int jm = plb::op_depth(w) == 0 ? jmax0 : jmax;
            while (j < jm && i + 1 + size_t(j) < hi && plb::op_code(in[i + 1 + size_t(j)]) == plb::OP_F &&
                   plb::op_depth(in[i + 1 + size_t(j)]) == plb::op_depth(w) + 1 + j &&
                   (h >> (j + 1)) >= ve)
                ++j;
            out.push_back(w | (uint32_t(j) << plb::kOpChainShift));
            i += 1 + size_t(j);
        } else {
            out.push_back(w);
            ++i;
        }
    }
}

bool uses_list(int k) { return k != PL_KIND_SC && k != PL_KIND_SSC; }
bool uses_crc(int k) { return k == PL_KIND_CA_SSCL || k == PL_KIND_PA_SSCL || k == PL_KIND_FA_SSCL; }
bool adaptive(int k) { return k == PL_KIND_PA_SSCL || k == PL_KIND_FA_SSCL; }
bool uses_pruning(int k) { return k != PL_KIND_SC && k != PL_KIND_SCL; }

// Host image of one code's device tables.
struct HostCode {
    int n = 0, k = 0, stages = 0, psize = 0, width = 0;
    std::vector<uint8_t> frozen;
    std::vector<uint32_t> sched_list, sched_listv[4], sched_sc, sched_lane; // (DevCode::sched_listv)
    std::vector<uint16_t> info_pos;
    std::vector<uint8_t> open_mask; // ceil(n/8): bit i of byte j = position 8j+i is open
    std::vector<uint64_t> crc_tab;
    uint64_t crc_c0 = 0;
};

HostCode make_host_code(const pl_code& c, const pl_decoder& dec) {
    if (c.n < 2 || (c.n & (c.n - 1)) != 0)
        throw ConfigError("N must be a power of two >= 2 (got " + std::to_string(c.n) + ")");
    // schedule words hold log2(m) and the depth in 4 bits each (polar_dev.h)
    if (c.n > 32768) throw ConfigError("N > 32768 is not supported by the GPU decoder");
    if (c.k < 1) throw ConfigError("K must be at least 1 (got " + std::to_string(c.k) + ")");
    if (!c.frozen) throw ConfigError("frozen mask is null");
    HostCode h;
    h.n = c.n;
    h.k = c.k;
    h.stages = ilog2i(c.n);
    h.frozen.assign(c.frozen, c.frozen + c.n);
    for (auto& b : h.frozen) b = b ? 1 : 0;
    h.width = c.crc.width;
    std::unique_ptr<Crc> crc;
    if (c.crc.width) crc = std::make_unique<Crc>(c.crc);
    int open = 0;
    for (int i = 0; i < c.n; ++i) open += h.frozen[size_t(i)] == 0;
    if (open != c.k + h.width)
        throw ConfigError("frozen mask leaves " + std::to_string(open) +
                          " information positions, need K + CRC bits = " +
                          std::to_string(c.k + h.width));
    h.psize = c.k + h.width;
    for (int i = 0; i < c.n; ++i)
        if (!h.frozen[size_t(i)]) h.info_pos.push_back(uint16_t(i));
    h.open_mask.assign(size_t((c.n + 7) / 8), 0);
    for (int i = 0; i < c.n; ++i)
        if (!h.frozen[size_t(i)]) h.open_mask[size_t(i >> 3)] |= uint8_t(1u << (i & 7));
    if (c.channel_use) { // make_code's puncture checks (code.cpp:112-125)
        int transmitted = 0;
        for (int i = 0; i < c.n; ++i) {
            if (c.channel_use[i] > PL_USE_SHORTENED)
                throw ConfigError("channel use " + std::to_string(int(c.channel_use[i])) +
                                  " at position " + std::to_string(i) + " (want T, P or S)");
            transmitted += c.channel_use[i] == PL_USE_TRANSMITTED;
        }
        if (transmitted < c.k + h.width)
            throw ConfigError("puncture pattern transmits only " + std::to_string(transmitted) +
                              " symbols, fewer than K + CRC bits = " + std::to_string(c.k + h.width));
    }

    static const pl_pruning none{0, 0, 0, 0, 0, 0};
    const pl_pruning& pc = uses_pruning(dec.kind) ? dec.pruning : none;
    std::vector<Node> tree;
    tree.reserve(size_t(2 * c.n));
    build_tree(tree, h.frozen.data(), 0, c.n, 0, pc);
    {
        // list-schedule variants (DevCode::sched_listv): big fused leaves
        // (PLB_FUSE_BIG=0: off) and, float, chained F ops (PLB_LIST_CHAIN=0:
        // one op per level)
        const char* fb = std::getenv("PLB_FUSE_BIG");
        const bool big_r1 = fb ? std::atoi(fb) != 0 : true;
        const char* lc = std::getenv("PLB_LIST_CHAIN");
        const bool chain = dec.precision == PL_F32 && !(lc && std::atoi(lc) == 0);
        const int fm = dec.precision == PL_I8 ? plb::kFuseMaxI8 : plb::kFuseMaxF32;
        emit_list(tree, 0, h.sched_listv[0], fm, big_r1);
        emit_list(tree, 0, h.sched_listv[1], fm, false);
        h.sched_list = h.sched_listv[0];
        for (int v = 0; v < 2; ++v) {
            h.sched_listv[2 + v] = h.sched_listv[v];
            if (chain) chain_list_ops(h.sched_listv[2 + v], 4);
        }
    }
    emit_sc(tree, 0, h.sched_sc, h.frozen.data());
    // frame-per-lane SC kernel: subtrees of <= PLB_LANE_SUB values (default and
    // maximum 16) are decoded in registers (OP_SCSUB), everything else op by op
    const char* ls = std::getenv("PLB_LANE_SUB");
    const int lane_sub = ls ? std::min(16, std::max(0, std::atoi(ls))) : 16;
    emit_sc(tree, 0, h.sched_lane, h.frozen.data(), lane_sub, true);
    {
        // chained F levels (PLB_LANE_CHAIN, at most 1; 0 = one op per level)
        const char* lc = std::getenv("PLB_LANE_CHAIN");
        const int jdef = dec.precision == PL_F32 ? 1 : 0; // float only (lanes.cuh lane_fg)
        const int jmax = dec.precision != PL_F32 ? 0 : lc ? std::min(1, std::max(0, std::atoi(lc))) : jdef;
        const char* lc0 = std::getenv("PLB_LANE_CHAIN0"); // ... of the ops on the channel
        const int jmax0 = dec.precision != PL_F32 ? 0 : lc0 ? std::min(1, std::max(0, std::atoi(lc0))) : 0;
        // G ops with a rate-1 child: decided in registers.  (Fixed point too:
        // zero channel LLRs are common there -- 0.2% at int8 x4 -- but the g
        // values of the rate-1 nodes are sums of magnitudes: measured on
        // FA@4.5 dB, every rate-1 node of >= 32 values took the shortcut.)
        const bool gr1 = !(std::getenv("PLB_LANE_GR1") && std::atoi(std::getenv("PLB_LANE_GR1")) == 0);
        // in-register subtrees fused with their parent's F / G op
        const bool subf = !(std::getenv("PLB_LANE_SUBF") && std::atoi(std::getenv("PLB_LANE_SUBF")) == 0);
        {
            std::vector<uint32_t> fused;
            fused.reserve(h.sched_lane.size());
            const int ve = dec.precision == PL_F32 ? 4 : dec.precision == PL_I8 ? 16 : 8;
            fuse_lane_chains(h.sched_lane, 0, h.sched_lane.size(), fused, ve, jmax, jmax0, gr1, subf);
            h.sched_lane.swap(fused);
        }
    }

    if (crc) {
        // affine map: crc(m) = c0 ^ XOR_i m_i col_i over the K message bits;
        // the tail bits enter the syndrome at their MSB-first weight
        std::vector<uint8_t> msg(size_t(c.k), 0);
        const uint64_t c0 = crc->compute(msg.data(), msg.size());
        std::vector<uint64_t> colpos(size_t(c.n), 0);
        for (int j = 0; j < c.k; ++j) {
            msg[size_t(j)] = 1;
            colpos[h.info_pos[size_t(j)]] = crc->compute(msg.data(), msg.size()) ^ c0;
            msg[size_t(j)] = 0;
        }
        for (int j = 0; j < h.width; ++j)
            colpos[h.info_pos[size_t(c.k + j)]] = 1ull << (h.width - 1 - j);
        const int nbytes = (c.n + 7) / 8;
        h.crc_tab.assign(size_t(nbytes) * 256, 0);
        for (int j = 0; j < nbytes; ++j)
            for (int v = 0; v < 256; ++v) {
                uint64_t acc = 0;
                for (int b = 0; b < 8; ++b)
                    if (((v >> b) & 1) && 8 * j + b < c.n) acc ^= colpos[size_t(8 * j + b)];
                h.crc_tab[size_t(j) * 256 + size_t(v)] = acc;
            }
        h.crc_c0 = c0;
    }
    return h;
}

struct RungCfg {
    int l = 1;
    int seg_max = 0;
    int smem_per_frame = 0;
    int64_t gscratch_per_frame = 0;
    int grid = 0;
    int wpb = plb::kMaxWarpsPerBlock;
    int fpw = 1; // frames per warp (sub-warp decoding, single-code batches)
    int team = 1; // >1: blocks of `team` warps, one frame each
    int seg_solo = 0; // solo-mode layout (warp 0 with the whole block's smem), 0 = none
    int64_t small_max = 0; // small-pass plan of an adaptive rung: used up to this many frames
    bool lanes = false; // frame-per-lane SC kernel (smem / gscratch figures per 32-frame warp)
    int64_t gscratch_total() const {
        return int64_t(grid) * (team > 1 ? 1 : wpb * fpw) * gscratch_per_frame;
    }
};

} // namespace

struct pl_handle {
    int device = 0;
    pl_decoder dec{};
    std::vector<HostCode> codes;
    int nmax = 0;
    int64_t pstride = 0, cstride = 0;
    int esz = 4;
    uint32_t* lat_ns = nullptr; // pl_frame_latency: per-frame decode time of pl_decode(_packed)
    uint32_t* path_alive = nullptr; // pl_list_paths: the final list of every frame
    float* path_metric = nullptr;
    int64_t host_chunk = 0;     // frames per chunk of pl_decode_host (0 = automatic)
    int list_alt = 0; // LaunchParams::list_alt
    int llr_layout = 0; // pl_set_llr_layout
    int sc_tr = 0; // LaunchParams::sc_tr
    int sc_keep = 0, sc_keep_hi = 0; // L2 hint split of the frame-per-lane SC pass (LaunchParams::sc_keep)
    int sc_discard = 0; // LaunchParams::sc_discard
    int list_discard = 0; // LaunchParams::list_discard
    int sms = 0;
    std::string err;
    // device residency
    std::vector<void*> allocs;
    plb::DevCode* d_codes = nullptr;
    int64_t gscratch_bytes = 0;
    RungCfg sc_cfg;
    std::vector<RungCfg> rungs; // list rungs in ladder order
    // adaptive rungs planned with several frames per warp also get a
    // 1-frame-per-warp plan for small passes (lower latency per frame); the
    // device picks one of the two launches from the pass's frame count
    std::vector<RungCfg> rungs_small;
    // FA ladder, speculative tail: when at most spec_max frames reach the
    // third-last rung, the last three rungs decode them side by side on
    // three streams into a staging area and a commit kernel keeps, per
    // frame, the first list size whose CRC passed (decoders.hpp:70-82 is a
    // sequence of independent decodes, so the results are the same): the
    // tail costs one frame latency instead of three.
    std::vector<RungCfg> spec; // plans of the last three rungs, grid <= spec_max blocks
    int spec_max = 0;          // 0 = off
    // Execution contexts: the scratch and control buffers one decode in
    // flight needs.  pl_decode uses ex[0]; pl_decode_host alternates ex[0]
    // and ex[1] on two compute streams, so one chunk's decode can fill the
    // SMs the previous chunk's tail leaves idle.
    struct Exec {
        void* d_gscratch = nullptr;           // global spill of the large depth pools
        unsigned long long* d_work = nullptr; // one work counter per launch
        int32_t* d_counts = nullptr;          // fail counts per launch
        int32_t* d_lists[2] = {nullptr, nullptr};
        int64_t list_cap = 0;
        int32_t* d_hist = nullptr;   // multi-code batches: frames bucketed by code
        int32_t* d_sorted = nullptr;
        int64_t sorted_cap = 0;
        // end of the last decode issued on this context, whatever its stream:
        // the next user waits on it, so pl_decode / pl_decode_host /
        // pl_sim_point on different streams never overlap on the scratch
        cudaEvent_t done = nullptr;
        bool issued = false;
        // speculative tail of the FA ladder (pl_handle::spec)
        cudaStream_t s_spec[2] = {nullptr, nullptr};
        cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
        void* spec_scratch[3] = {nullptr, nullptr, nullptr};
        uint8_t* st_payload = nullptr;
        uint8_t* st_codeword = nullptr;
        uint8_t* st_crc = nullptr;
        float* st_metric = nullptr;
    } ex[2];
    int64_t launches = 0;
    // live per-launch timing (pl_profile)
    bool profiling = false;
    std::vector<cudaEvent_t> prof_ev; // 2 per launch slot
    std::vector<int32_t> prof_kind, prof_l;
    // host staging for pl_decode_host
    cudaStream_t s_comp[2] = {nullptr, nullptr}, s_h2d = nullptr, s_d2h = nullptr;
    int64_t stage_frames = 0;
    // a ring of kStage chunk buffers: the H2D copy of chunk c waits only for
    // the decode of chunk c - kStage, so the copy engine keeps streaming while
    // two chunks decode (2 buffers: cfg3 e2e lost ~0.4 ms per chunk)
    static constexpr int kStage = 4;
    void* d_in[kStage] = {};
    int64_t in_cap = 0; // bytes of each d_in / h_stage_in buffer
    int32_t* d_cid[kStage] = {};
    int64_t* d_off[kStage] = {}; // packed input: chunk-relative frame offsets
    int64_t* h_stage_off[kStage] = {};
    uint8_t* d_out[kStage] = {};
    void* h_stage_in[kStage] = {};
    uint8_t* h_stage_out[kStage] = {};
    cudaEvent_t ev_h2d[kStage]{}, ev_dec[kStage]{}, ev_d2h[kStage]{};

    template <class T>
    T* dalloc(size_t bytes) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

namespace {

int target_warps_per_sm() {
    const char* e = std::getenv("PLB_TARGET_WARPS");
    return e ? std::max(1, std::atoi(e)) : 32;
}

// Pick where the depth segments live: the most shared-memory-resident
// layout that still keeps PLB_TARGET_WARPS warps resident per SM, else the
// layout with the most resident warps.  Small list sizes on single-code
// batches decode 2 or 4 frames per warp (one per sub-warp) when that still
// reaches the target; PLB_FPW forces frames per warp.  Ladder rungs (FA)
// use 2 frames per warp up to L = 8 (measured: FA@3.5 dB L=8 rung 19.9 ->
// 18.7 ms, @2.5 dB 178 -> 164 ms, @4.5 dB 0.72 -> 0.87 ms with its few
// frames); multi-code ladder rungs get unsorted failure lists: 1 per warp.
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// Team mode (opt-in, PLB_TEAM=<warps>): a team of warps per frame, few
// frames per SM, so the frames' depth pools (L x N values) stay in shared
// memory and L2 instead of overflowing the L2 into HBM.  Only the element
// ops (F/G, H) are split over the team; the path bookkeeping stays on warp
// 0, and with 2-4 frames per SM that serial part dominates: measured 2.4x
// slower than independent warps at L = 32 float, so it is
// off by default.  The largest shared-memory share that still keeps
// PLB_TEAM_BLOCKS frames resident per SM.
RungCfg plan_team(const pl_handle& h, int l, int team, const std::vector<int>& cands) {
    const int want = std::max(1, env_int("PLB_TEAM_BLOCKS", 2));
    RungCfg best;
    best.l = l;
    int best_nb = 0;
    for (int seg : cands) {
        RungCfg c;
        c.l = l;
        c.seg_max = seg;
        c.wpb = team;
        c.team = team;
        c.smem_per_frame = int(plb::smem_bytes_per_frame(h.nmax, l, h.esz, seg, 32));
        c.gscratch_per_frame = plb::gscratch_bytes_per_frame(h.nmax, l, h.esz, seg);
        const int nb = plb::occupancy_list(h.dec.precision, l, 1, c.smem_per_frame, team, true);
        if (nb <= 0) continue;
        c.grid = nb * h.sms;
        if (nb >= want) return c;
        if (nb > best_nb) {
            best = c;
            best_nb = nb;
        }
    }
    return best;
}

// The frame-per-lane SC pass: 32 frames per warp; the most shared-memory
// resident layout that keeps PLB_LANE_WARPS warps per SM (measured best:
// 12 for float, whose pass is DRAM-bound -- 16 until the pass stopped
// storing rate-1 inputs and chained its F ops: then fewer frames in flight
// (less depth-pool state than the L2 holds) won, 14.2 -> 13.6 ms per 2^20
// frames, 10 / 12 alike, 8: 14.6; int16, DRAM-bound too (46 KB per frame),
// likewise: 12 warps with segments <= 64 in shared memory 9.8 ms, 16 / 24
// warps 11.4 / 12.3; int8 is flat from 20 to 32 and keeps 24).
RungCfg plan_lanes(const pl_handle& h) {
    const int target = std::max(1, env_int("PLB_LANE_WARPS", h.dec.precision == PL_I8 ? 24 : 12));
    const int forced = env_int("PLB_SEGMAX", 0);
    std::vector<int> cands;
    if (forced) cands.push_back(forced);
    else
        for (int sg = h.nmax; sg >= 1; sg >>= 1) cands.push_back(sg);
    RungCfg best;
    int best_warps = 0;
    for (int wpb = plb::kMaxWarpsPerBlock; wpb >= 1; wpb >>= 1) {
        for (int seg : cands) {
            RungCfg c;
            c.l = 1;
            c.lanes = true;
            c.seg_max = seg;
            c.wpb = wpb;
            c.smem_per_frame = int(plb::lane_smem_bytes_per_warp(h.nmax, h.esz, seg, h.sc_tr != 0));
            c.gscratch_per_frame = plb::lane_gscratch_bytes_per_warp(h.nmax, h.esz, seg);
            const int nb = plb::occupancy_sc_lanes(h.dec.precision, c.smem_per_frame * wpb, wpb);
            if (nb <= 0) continue;
            c.grid = nb * h.sms;
            if (nb * wpb > best_warps) {
                best = c;
                best_warps = nb * wpb;
            }
            if (nb * wpb >= target) break;
        }
        if (best_warps >= target) break;
    }
    if (best.grid <= 0) throw ConfigError("no launch configuration fits the SC pass on the device");
    return best;
}

// Sub-warps of one warp read the same structures of their own frame areas in
// the same instruction (alive list, buffer indices, node statistics, psum
// words): with an area stride of a multiple of 128 bytes they hit the same
// banks.  Strides of 128/fpw (mod 128) spread the frames over the banks.
int skew_frame_area(int bytes, int fpw) {
    if (fpw <= 1 || !env_int("PLB_SKEW", 1)) return bytes;
    const int want = 128 / fpw;
    return bytes + (want - bytes % 128 + 128) % 128;
}

RungCfg plan_rung(const pl_handle& h, int l, bool list, bool ladder = false, int force_fpw = 0) {
    const char* forced = std::getenv("PLB_SEGMAX");
    const char* forced_fpw = force_fpw ? "1" : std::getenv("PLB_FPW");
    const int target = target_warps_per_sm();
    std::vector<int> cands;
    if (forced) cands.push_back(std::atoi(forced));
    else
        for (int s = h.nmax; s >= 8; s >>= 1) cands.push_back(s);
    if (cands.empty()) cands.push_back(h.nmax); // tiny codes: everything in shared memory
    if (list) {
        const int team = std::min(plb::kMaxTeam, env_int("PLB_TEAM", 1));
        // (team kernels exist for L = 16 and 32)
        const int team_l = std::max(16, env_int("PLB_TEAM_L", h.dec.precision == PL_F32 ? 16 : 32));
        if (team > 1 && l >= team_l) {
            RungCfg t = plan_team(h, l, team, cands);
            if (t.grid > 0) return t;
        }
    }
    // multi-code batches are bucketed by code before a non-ladder list pass;
    // ladder rungs get unsorted failure lists
    const bool multi = h.codes.size() > 1;
    const int fmax = (list && !(ladder && (l > 8 || multi))) ? plb::frames_per_warp_max(l) : 1;
    std::vector<int> fpws;
    // a list size has kernels for fmax and 1 frames per warp
    if (forced_fpw) {
        const int f = std::atoi(forced_fpw);
        fpws.push_back(fmax > 1 && plb::frames_per_warp_ok(l, f) ? f : 1);
    } else {
        fpws.push_back(fmax);
        if (fmax > 1) fpws.push_back(1);
    }
    RungCfg pick;
    pick.l = l;
    for (int fpw : fpws) {
        RungCfg best;
        best.l = l;
        int best_warps = 0;
        // 4-warp blocks first; 2 / 1 when a warp's area is too big (large N x L)
        for (int wpb = plb::kMaxWarpsPerBlock; wpb >= 1; wpb >>= 1) {
            for (int seg : cands) {
                RungCfg c;
                c.l = l;
                c.seg_max = seg;
                c.wpb = wpb;
                c.fpw = fpw;
                c.smem_per_frame = skew_frame_area(int(plb::smem_bytes_per_frame(h.nmax, l, h.esz, seg, 32 / fpw)), fpw);
                c.gscratch_per_frame = plb::gscratch_bytes_per_frame(h.nmax, l, h.esz, seg);
                const int smem = c.smem_per_frame * fpw * wpb;
                const int nb = list ? plb::occupancy_list(h.dec.precision, l, fpw, smem, wpb)
                                    : plb::occupancy_sc(h.dec.precision, smem, wpb);
                if (nb <= 0) continue;
                c.grid = nb * h.sms;
                if (nb * wpb > best_warps) {
                    best = c;
                    best_warps = nb * wpb;
                }
                if (nb * wpb >= target) break;
            }
            if (best_warps >= target) break;
        }
        // several frames per warp pay off down to half the warp target
        // (measured: cfg1 at 24 resident 2-frame warps beats 32 1-frame ones)
        if (best.grid > 0 && (best_warps * 2 >= target || fpw == fpws.back())) {
            pick = best;
            break;
        }
    }
    if (pick.grid <= 0) throw ConfigError("no launch configuration fits this code / list size on the device");
    // solo mode (passes with at most one frame per block): the most
    // shared-memory-resident layout in the area of all the block's warps
    if (pick.wpb > 1 && env_int("PLB_SOLO", 1)) {
        for (int seg = h.nmax; seg >= 1; seg >>= 1) {
            if (plb::smem_bytes_per_frame(h.nmax, l, h.esz, seg, 32 / pick.fpw) <= int64_t(pick.smem_per_frame) * pick.wpb) {
                pick.seg_solo = seg;
                break;
            }
        }
    }
    return pick;
}

void ensure_lists(pl_handle::Exec& x, int64_t nframes) {
    if (x.list_cap >= nframes && x.d_lists[0]) return;
    for (int i = 0; i < 2; ++i)
        if (x.d_lists[i]) cudaFree(x.d_lists[i]);
    x.list_cap = std::max<int64_t>(nframes, 1024);
    for (int i = 0; i < 2; ++i)
        ck(cudaMalloc(&x.d_lists[i], size_t(x.list_cap) * sizeof(int32_t)), "cudaMalloc lists");
}

void ensure_exec(pl_handle& h, int e) {
    pl_handle::Exec& x = h.ex[e];
    if (x.d_work) return;
    x.d_gscratch = h.dalloc<void>(size_t(h.gscratch_bytes));
    x.d_work = h.dalloc<unsigned long long>(16 * sizeof(unsigned long long));
    x.d_counts = h.dalloc<int32_t>(16 * sizeof(int32_t));
    ck(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming), "event");
    if (h.spec_max > 0) {
        // the speculative ladder tail: two side streams, the scratch of its
        // three concurrent passes and the staging area of their outputs
        for (int j = 0; j < 2; ++j) {
            ck(cudaStreamCreateWithFlags(&x.s_spec[j], cudaStreamNonBlocking), "stream");
            ck(cudaEventCreateWithFlags(&x.ev_join[j], cudaEventDisableTiming), "event");
        }
        ck(cudaEventCreateWithFlags(&x.ev_fork, cudaEventDisableTiming), "event");
        for (int j = 0; j < 3; ++j)
            x.spec_scratch[j] = h.dalloc<void>(size_t(h.spec[size_t(j)].gscratch_total()));
        const size_t cap = size_t(3) * size_t(h.spec_max);
        x.st_payload = h.dalloc<uint8_t>(cap * size_t(h.pstride));
        x.st_codeword = h.dalloc<uint8_t>(cap * size_t(h.cstride));
        x.st_crc = h.dalloc<uint8_t>(cap);
        x.st_metric = h.dalloc<float>(cap * sizeof(float));
    }
}

int fail(pl_handle* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    g_thread_err = msg;
    return code;
}

void run_decode(pl_handle& h, const void* llr, const int32_t* code_id, int64_t nframes,
                uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc,
                float* metric, cudaStream_t s0, int exec = 0, const int64_t* llr_offset = nullptr,
                uint32_t* lat_ns = nullptr, bool paths = false, bool il32 = false) {
    cudaStream_t s = s0;
    ck(cudaSetDevice(h.device), "cudaSetDevice");
    h.launches = 0;
    h.prof_kind.clear(); // timed decode launches of this call (pl_last_kernel_ms)
    h.prof_l.clear();
    if (nframes <= 0) return;
    const int kind = h.dec.kind;
    const bool need_lists = adaptive(kind);
    ensure_exec(h, exec);
    pl_handle::Exec& x = h.ex[exec];
    if (x.issued) ck(cudaStreamWaitEvent(s, x.done, 0), "wait");
    if (need_lists) ensure_lists(x, nframes);
    ck(cudaMemsetAsync(x.d_work, 0, 16 * sizeof(unsigned long long), s), "memset");
    ck(cudaMemsetAsync(x.d_counts, 0, 16 * sizeof(int32_t), s), "memset");

    plb::LaunchParams base{};
    base.codes = h.d_codes;
    base.llr = llr;
    base.llr_stride = h.nmax;
    base.llr_offset = llr_offset;
    base.code_id = code_id;
    base.nframes = nframes;
    base.payload = payload;
    base.payload_stride = h.pstride;
    base.codeword = codeword;
    base.codeword_stride = h.cstride;
    base.crc_ok = crc_ok;
    base.esc = esc;
    base.metric = metric;
    base.lat_ns = lat_ns;
    base.path_alive = paths ? h.path_alive : nullptr;
    base.path_metric = paths ? h.path_metric : nullptr;
    base.path_stride = h.dec.l;
    if (lat_ns) ck(cudaMemsetAsync(lat_ns, 0, size_t(nframes) * sizeof(uint32_t), s), "memset");
    base.gscratch = x.d_gscratch;
    base.nmax = h.nmax;
    int slot = 0;

    // (spec_j >= 0: speculative rung j of the ladder's tail, on its own
    // stream and scratch, outputs staged by list position)
    auto run = [&](const RungCfg& rc, bool list, int select, const int32_t* in_list,
                   const int32_t* in_count, int32_t* out_list, int32_t* out_count,
                   int64_t count_lo = -1, int64_t count_hi = INT64_MAX, int spec_j = -1) {
        plb::LaunchParams p = base;
        cudaStream_t s = s0;
        if (spec_j >= 0) {
            if (spec_j > 0) s = x.s_spec[spec_j - 1];
            const int64_t o = int64_t(spec_j) * h.spec_max;
            p.gscratch = x.spec_scratch[spec_j];
            p.payload = x.st_payload + o * h.pstride;
            p.codeword = codeword ? x.st_codeword + o * h.cstride : nullptr;
            p.crc_ok = x.st_crc + o;
            p.metric = x.st_metric + o;
            p.esc = nullptr;
            p.out_by_idx = 1;
        }
        p.count_lo = count_lo;
        p.count_hi = count_hi;
        p.work = x.d_work + slot;
        p.frame_list = in_list;
        p.frame_count = in_count;
        p.fail_list = out_list;
        p.fail_count = out_count;
        p.l = rc.l;
        p.select_by_crc = select;
        p.seg_smem_max = rc.seg_max;
        p.smem_per_frame = rc.smem_per_frame;
        p.smem_per_warp = rc.smem_per_frame * rc.fpw;
        p.gscratch_per_frame = rc.gscratch_per_frame;
        p.esc_level = rc.l;
        p.wpb = rc.wpb;
        p.fpw = rc.fpw;
        p.team = rc.team;
        p.seg_solo = rc.seg_solo;
        p.sc_keep = rc.lanes ? h.sc_keep : 0;
        p.sc_keep_hi = rc.lanes ? h.sc_keep_hi : 0;
        p.sc_discard = rc.lanes ? h.sc_discard : 0;
        p.list_discard = rc.lanes ? 0 : h.list_discard;
        p.list_alt = h.list_alt;
        p.llr_il32 = rc.lanes && il32 ? 1 : 0;
        p.sc_tr = rc.lanes ? h.sc_tr : 0;
        p.solo_max = rc.grid * rc.fpw;
        if (h.profiling) {
            while (h.prof_ev.size() < size_t(2 * (slot + 1))) {
                cudaEvent_t ev;
                ck(cudaEventCreate(&ev), "event");
                h.prof_ev.push_back(ev);
            }
            h.prof_kind.resize(size_t(slot + 1));
            h.prof_l.resize(size_t(slot + 1));
            h.prof_kind[size_t(slot)] = list ? 1 : 0;
            h.prof_l[size_t(slot)] = rc.l;
            ck(cudaEventRecord(h.prof_ev[size_t(2 * slot)], s), "record");
        }
        cudaError_t e = list       ? plb::launch_list(p, h.dec.precision, rc.grid, s)
                        : rc.lanes ? plb::launch_sc_lanes(p, h.dec.precision, rc.grid, s)
                                   : plb::launch_sc(p, h.dec.precision, rc.grid, s);
        ck(e, list ? "list kernel launch" : "sc kernel launch");
        if (h.profiling) ck(cudaEventRecord(h.prof_ev[size_t(2 * slot + 1)], s), "record");
        ++slot;
        ++h.launches;
    };

    // Kernels that decode several frames in lockstep (sub-warps, the
    // frame-per-lane SC kernel) need one code per warp: multi-code batches
    // are bucketed by code first (the frame list of that pass).
    const int32_t* blist = nullptr;
    const int32_t* bcount = nullptr;
    auto bucket = [&](const RungCfg& rc) {
        blist = nullptr;
        bcount = nullptr;
        if (!(code_id && h.codes.size() > 1 && (rc.fpw > 1 || rc.lanes))) return;
        if (x.sorted_cap < nframes) {
            if (x.d_sorted) cudaFree(x.d_sorted);
            x.sorted_cap = std::max<int64_t>(nframes, 1024);
            ck(cudaMalloc(&x.d_sorted, size_t(x.sorted_cap) * sizeof(int32_t)), "cudaMalloc");
        }
        if (!x.d_hist) ck(cudaMalloc(&x.d_hist, h.codes.size() * sizeof(int32_t)), "cudaMalloc");
        ck(plb::bucket_by_code(code_id, nframes, int(h.codes.size()), x.d_hist, x.d_sorted,
                               x.d_counts + 15, s),
           "bucket frames by code");
        h.launches += 3; // histogram, scan, scatter
        blist = x.d_sorted;
        bcount = x.d_counts + 15;
    };

    // an adaptive rung with a small-pass plan (pl_create): two launches
    // with complementary frame-count ranges, the device picks
    // (lo: the pass runs only with more than lo frames; fewer went to the
    // speculative tail)
    auto rung = [&](size_t i, const int32_t* in_list, const int32_t* in_count, int32_t* out_list,
                    int32_t* out_count, int64_t lo = -1) {
        const RungCfg& sm = h.rungs_small[i];
        if (sm.grid > 0) {
            const int64_t t = sm.small_max;
            if (t > lo) run(sm, true, 1, in_list, in_count, out_list, out_count, lo, t);
            run(h.rungs[i], true, 1, in_list, in_count, out_list, out_count, std::max(t, lo), INT64_MAX);
        } else {
            run(h.rungs[i], true, 1, in_list, in_count, out_list, out_count, lo, INT64_MAX);
        }
    };
    // the speculative tail: rungs [first, first + 3) side by side on the
    // frames of in_list when there are at most spec_max of them
    auto spec_tail = [&](size_t first, const int32_t* in_list, const int32_t* in_count) {
        ck(cudaEventRecord(x.ev_fork, s0), "record");
        for (int j = 0; j < 3; ++j) {
            if (j > 0) ck(cudaStreamWaitEvent(x.s_spec[j - 1], x.ev_fork, 0), "wait");
            run(h.spec[size_t(j)], true, 1, in_list, in_count, nullptr, nullptr, -1, h.spec_max, j);
            if (j > 0) {
                ck(cudaEventRecord(x.ev_join[j - 1], x.s_spec[j - 1]), "record");
                ck(cudaStreamWaitEvent(s0, x.ev_join[j - 1], 0), "wait");
            }
        }
        plb::CommitParams cp{};
        cp.codes = h.d_codes;
        cp.code_id = code_id;
        cp.list = in_list;
        cp.count = in_count;
        cp.count_hi = h.spec_max;
        cp.nst = 3;
        cp.cap = h.spec_max;
        for (int j = 0; j < 3; ++j) cp.levels[j] = h.spec[size_t(j)].l;
        cp.st_payload = x.st_payload;
        cp.st_codeword = codeword ? x.st_codeword : nullptr;
        cp.st_crc = x.st_crc;
        cp.st_metric = x.st_metric;
        cp.payload = payload;
        cp.codeword = codeword;
        cp.crc_ok = crc_ok;
        cp.esc = esc;
        cp.metric = metric;
        cp.payload_stride = h.pstride;
        cp.codeword_stride = h.cstride;
        ck(plb::launch_commit(cp, std::max(1, (h.spec_max + 3) / 4), s0), "commit launch");
        ++h.launches;
    };

    switch (kind) {
    case PL_KIND_SC:
    case PL_KIND_SSC:
        bucket(h.sc_cfg);
        run(h.sc_cfg, false, 0, blist, bcount, nullptr, nullptr);
        break;
    case PL_KIND_SCL:
    case PL_KIND_SSCL:
    case PL_KIND_CA_SSCL:
        bucket(h.rungs.back());
        run(h.rungs.back(), true, kind == PL_KIND_CA_SSCL ? 1 : 0, blist, bcount, nullptr, nullptr);
        break;
    case PL_KIND_PA_SSCL:
        bucket(h.sc_cfg);
        run(h.sc_cfg, false, 0, blist, bcount, x.d_lists[0], x.d_counts + 0);
        rung(h.rungs.size() - 1, x.d_lists[0], x.d_counts + 0, nullptr, nullptr);
        break;
    case PL_KIND_FA_SSCL: {
        bucket(h.sc_cfg);
        run(h.sc_cfg, false, 0, blist, bcount, x.d_lists[0], x.d_counts + 0);
        int cur = 0;
        // (per-frame latency and list introspection follow the plain ladder)
        const bool spec = h.spec_max > 0 && !lat_ns && !base.path_alive;
        for (size_t i = 0; i < h.rungs.size(); ++i) {
            const bool last = i + 1 == h.rungs.size();
            const bool tail = spec && i + 3 == h.rungs.size();
            if (tail) spec_tail(i, x.d_lists[cur], x.d_counts + i);
            rung(i, x.d_lists[cur], x.d_counts + i, last ? nullptr : x.d_lists[cur ^ 1],
                 last ? nullptr : x.d_counts + i + 1, tail ? int64_t(h.spec_max) : int64_t(-1));
            cur ^= 1;
        }
        break;
    }
    default: throw ConfigError("unhandled decoder variant");
    }
    ck(cudaEventRecord(x.done, s), "record");
    x.issued = true;
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

} // namespace

extern "C" {

int pl_crc_parse(const char* text, pl_crc* out) {
    if (!text || !out) return fail(nullptr, PL_ERR_ARG, "null argument");
    try {
        *out = parse_crc(text);
        return PL_OK;
    } catch (const std::exception& e) {
        return fail(nullptr, PL_ERR_PARSE, e.what());
    }
}

namespace {
// A text file read whole and split at whitespace, as operator>> reads it.
struct TextTokens {
    std::string text;
    size_t pos = 0;
    bool load(const char* path) {
        FILE* fp = std::fopen(path, "r");
        if (!fp) return false;
        char buf[4096];
        size_t got;
        while ((got = std::fread(buf, 1, sizeof buf, fp)) > 0) text.append(buf, got);
        std::fclose(fp);
        return true;
    }
    bool next(std::string& out) {
        while (pos < text.size() && std::isspace(static_cast<unsigned char>(text[pos]))) ++pos;
        const size_t b = pos;
        while (pos < text.size() && !std::isspace(static_cast<unsigned char>(text[pos]))) ++pos;
        out = text.substr(b, pos - b);
        return !out.empty();
    }
    bool next_int(int32_t& v) {
        std::string t;
        if (!next(t)) return false;
        char* end = nullptr;
        const long x = std::strtol(t.c_str(), &end, 10);
        if (*end || x < INT32_MIN || x > INT32_MAX) return false;
        v = int32_t(x);
        return true;
    }
};

// One line of n characters from `alphabet`; value = index in the alphabet.
// Messages as the reference's ParseError (code.cpp:164-221).
int read_pattern(TextTokens& tt, const std::string& what, const std::string& path, int32_t n,
                 const char* alphabet, const char* want, const char* count_word, std::string& out) {
    if (!tt.next(out))
        return fail(nullptr, PL_ERR_PARSE, what + " file '" + path + "': missing " + count_word + " line");
    if (out.size() != size_t(n))
        return fail(nullptr, PL_ERR_PARSE,
                    what + " file '" + path + "': " + count_word + " has " + std::to_string(out.size()) +
                        " characters, header says N = " + std::to_string(n));
    for (size_t i = 0; i < out.size(); ++i)
        if (!std::strchr(alphabet, out[i]))
            return fail(nullptr, PL_ERR_PARSE,
                        what + " file '" + path + "': " + count_word + " character '" +
                            std::string(1, out[i]) + "' at position " + std::to_string(i) + " (want " +
                            want + ")");
    return PL_OK;
}
} // namespace

// Frozen-set files in the reference format (code.cpp:164-194): "N K" then
// one line of N characters, '1' = frozen.  Messages as the reference's
// ParseError / IoError.
int pl_frozen_file_load(const char* path, int32_t* n, int32_t* k, uint8_t* frozen_out, int32_t cap) {
    if (!path || !n || !k) return fail(nullptr, PL_ERR_ARG, "null argument");
    const std::string p(path);
    TextTokens tt;
    if (!tt.load(path)) return fail(nullptr, PL_ERR_IO, "cannot open '" + p + "' for reading");
    int32_t vn = 0, vk = 0;
    if (!tt.next_int(vn) || !tt.next_int(vk))
        return fail(nullptr, PL_ERR_PARSE, "frozen file '" + p + "': header must be 'N K'");
    std::string mask;
    if (const int rc = read_pattern(tt, "frozen", p, vn, "01", "0 or 1", "mask", mask)) return rc;
    *n = vn;
    *k = vk;
    if (frozen_out) {
        if (cap < vn) return fail(nullptr, PL_ERR_ARG, "frozen buffer too small");
        for (int32_t i = 0; i < vn; ++i) frozen_out[i] = mask[size_t(i)] == '1';
    }
    return PL_OK;
}

// Puncture files (load_puncture_file, code.cpp:196-221): "N" then N
// characters T / P / S -> PL_USE_*.
int pl_puncture_file_load(const char* path, int32_t* n, uint8_t* use_out, int32_t cap) {
    if (!path || !n) return fail(nullptr, PL_ERR_ARG, "null argument");
    const std::string p(path);
    TextTokens tt;
    if (!tt.load(path)) return fail(nullptr, PL_ERR_IO, "cannot open '" + p + "' for reading");
    int32_t vn = 0;
    if (!tt.next_int(vn)) return fail(nullptr, PL_ERR_PARSE, "puncture file '" + p + "': header must be 'N'");
    std::string pat;
    if (const int rc = read_pattern(tt, "puncture", p, vn, "TPS", "T, P or S", "pattern", pat)) return rc;
    *n = vn;
    if (use_out) {
        if (cap < vn) return fail(nullptr, PL_ERR_ARG, "pattern buffer too small");
        for (int32_t i = 0; i < vn; ++i)
            use_out[i] = uint8_t(std::strchr("TPS", pat[size_t(i)]) - "TPS"); // PL_USE_* order
    }
    return PL_OK;
}

int pl_frozen_file_save(const char* path, int32_t n, int32_t k, const uint8_t* frozen) {
    if (!path || (!frozen && n > 0) || n < 0) return fail(nullptr, PL_ERR_ARG, "bad argument");
    const std::string p(path);
    FILE* fp = std::fopen(path, "w");
    if (!fp) return fail(nullptr, PL_ERR_IO, "cannot open '" + p + "' for writing");
    std::string out = std::to_string(n) + ' ' + std::to_string(k) + '\n';
    for (int32_t i = 0; i < n; ++i) out += frozen[i] ? '1' : '0';
    out += '\n';
    const bool ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    if (std::fclose(fp) != 0 || !ok) return fail(nullptr, PL_ERR_IO, "failed writing '" + p + "'");
    return PL_OK;
}

int pl_crc_compute(const pl_crc* spec, const uint8_t* bits, int64_t len, uint64_t* out) {
    if (!spec || (!bits && len) || !out || len < 0) return fail(nullptr, PL_ERR_ARG, "bad argument");
    try {
        Crc c(*spec);
        *out = c.compute(bits, size_t(len));
        return PL_OK;
    } catch (const ConfigError& e) {
        return fail(nullptr, PL_ERR_CONFIG, e.what());
    }
}

int32_t pl_tree_build(const uint8_t* frozen, int32_t n, const pl_pruning* cfg, int32_t* out,
                      int32_t max_nodes) {
    if (!frozen || !cfg || !out) return -1;
    try {
        if (n < 2 || (n & (n - 1)) != 0)
            throw ConfigError("decode tree needs a power-of-two block length, got " + std::to_string(n));
        check_pruning(*cfg);
        std::vector<Node> t;
        build_tree(t, frozen, 0, n, 0, *cfg);
        if (int(t.size()) > max_nodes) return -1;
        for (size_t i = 0; i < t.size(); ++i) {
            const Node& nd = t[i];
            int32_t* o = out + 6 * i;
            o[0] = nd.kind;
            o[1] = nd.depth;
            o[2] = nd.lb;
            o[3] = nd.size;
            o[4] = nd.left;
            o[5] = nd.right;
        }
        return int32_t(t.size());
    } catch (const std::exception& e) {
        g_thread_err = e.what();
        return -1;
    }
}

int pl_create(const pl_code* codes, int32_t ncodes, const pl_decoder* dec, int32_t device,
              pl_handle** out) {
    if (!codes || ncodes < 1 || !dec || !out) return fail(nullptr, PL_ERR_ARG, "bad argument");
    *out = nullptr;
    pl_handle* h = new pl_handle();
    try {
        h->device = device;
        h->dec = *dec;
        const int kind = dec->kind;
        if (kind < PL_KIND_SC || kind > PL_KIND_FA_SSCL) throw ConfigError("unknown decoder kind");
        if (dec->precision != PL_F32 && dec->precision != PL_I8 && dec->precision != PL_I16)
            throw ConfigError("precision must be PL_F32, PL_I8 or PL_I16");
        h->esz = dec->precision == PL_F32 ? 4 : dec->precision == PL_I16 ? 2 : 1;
        // FrameDecoder validation (decoders.hpp:40-55)
        const int l = uses_list(kind) ? dec->l : 1;
        h->dec.l = l;
        if (adaptive(kind) && l < 2)
            throw ConfigError("adaptive decoding needs a list limit of at least 2, got " + std::to_string(l));
        if (uses_list(kind) && (l < 1 || (l & (l - 1)) != 0))
            throw ConfigError("list size must be a power of two, got " + std::to_string(l));
        if (l > 32) throw ConfigError("list sizes above 32 are not supported by the GPU decoder");
        if (uses_pruning(kind)) check_pruning(dec->pruning);
        for (int i = 0; i < ncodes; ++i) {
            if (uses_crc(kind) && codes[i].crc.width == 0)
                throw ConfigError("CRC-aided decoding needs a code with a CRC");
            h->codes.push_back(make_host_code(codes[i], h->dec));
        }
        for (const auto& c : h->codes) {
            h->nmax = std::max(h->nmax, c.n);
            h->pstride = std::max<int64_t>(h->pstride, (c.psize + 7) / 8);
            h->cstride = std::max<int64_t>(h->cstride, (c.n + 7) / 8);
        }
        // ---- device residency
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw CudaError("no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device), "attr");
        std::vector<plb::DevCode> dc(h->codes.size());
        // the universal byte-compaction table of the payload gather
        const uint8_t* comp_tab = nullptr;
        {
            std::vector<uint8_t> t(size_t(256) * 256);
            for (int m = 0; m < 256; ++m)
                for (int v = 0; v < 256; ++v) {
                    uint32_t o = 0;
                    for (int i = 0; i < 8; ++i)
                        if ((m >> i) & 1) o = (o << 1) | ((v >> i) & 1);
                    t[size_t(m) * 256 + size_t(v)] = uint8_t(o);
                }
            uint8_t* p = h->dalloc<uint8_t>(t.size());
            ck(cudaMemcpy(p, t.data(), t.size(), cudaMemcpyHostToDevice), "upload");
            comp_tab = p;
        }
        for (size_t i = 0; i < h->codes.size(); ++i) {
            const HostCode& c = h->codes[i];
            plb::DevCode& d = dc[i];
            d.n = c.n;
            d.stages = c.stages;
            d.k = c.k;
            d.psize = c.psize;
            d.crc_width = c.width;
            auto up = [&](const void* src, size_t bytes) {
                void* p = h->dalloc<void>(bytes);
                if (bytes) ck(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "upload");
                return p;
            };
            // schedules carry one padding word (kernels may fetch one op ahead)
            auto up_sched = [&](const std::vector<uint32_t>& v) {
                std::vector<uint32_t> padded(v);
                padded.push_back(0u);
                return static_cast<const uint32_t*>(up(padded.data(), padded.size() * 4));
            };
            d.sched_list = up_sched(c.sched_list);
            d.sched_sc = up_sched(c.sched_sc);
            d.sched_lane = up_sched(c.sched_lane);
            d.nops_lane = int(c.sched_lane.size());
            d.nops_list = int(c.sched_list.size());
            d.sched_listv[0] = d.sched_list;
            d.nops_listv[0] = d.nops_list;
            for (int v = 1; v < 4; ++v) {
                // (equal variants share one upload)
                int same = -1;
                for (int u = 0; u < v && same < 0; ++u)
                    if (c.sched_listv[u] == c.sched_listv[v]) same = u;
                d.sched_listv[v] = same >= 0 ? d.sched_listv[same] : up_sched(c.sched_listv[v]);
                d.nops_listv[v] = int(c.sched_listv[v].size());
            }
            for (int v = 0; v < 4; ++v) {
                int same = -1;
                for (int u = 0; u < v && same < 0; ++u)
                    if (d.sched_listv[u] == d.sched_listv[v]) same = u;
                if (same >= 0) {
                    d.sched_listx[v] = d.sched_listx[same];
                    continue;
                }
                const std::vector<uint32_t>& sv = v == 0 ? c.sched_list : c.sched_listv[v];
                std::vector<uint4> x(sv.size() + 1, make_uint4(0, 0, 0, 0));
                for (size_t i = 0; i < sv.size(); ++i)
                    x[i] = make_uint4(sv[i], uint32_t(plb::op_depth(sv[i])), 1u << plb::op_logm(sv[i]),
                                      uint32_t(plb::op_lb(sv[i])));
                d.sched_listx[v] = static_cast<const uint4*>(up(x.data(), x.size() * sizeof(uint4)));
            }
            d.nops_sc = int(c.sched_sc.size());
            d.info_pos = static_cast<const uint16_t*>(up(c.info_pos.data(), c.info_pos.size() * 2));
            d.crc_tab = c.crc_tab.empty() ? nullptr
                                          : static_cast<const uint64_t*>(up(c.crc_tab.data(), c.crc_tab.size() * 8));
            d.crc_c0 = c.crc_c0;
            d.open_mask = static_cast<const uint8_t*>(up(c.open_mask.data(), c.open_mask.size()));
            d.comp_tab = comp_tab;
        }
        h->d_codes = h->dalloc<plb::DevCode>(dc.size() * sizeof(plb::DevCode));
        ck(cudaMemcpy(h->d_codes, dc.data(), dc.size() * sizeof(plb::DevCode), cudaMemcpyHostToDevice),
           "upload codes");
        // ---- launch plans for every pass this kind can run
        // frame-per-lane SC pass: the ops on a frame-major channel read it in
        // coalesced tiles transposed through shared memory (lanes.cuh
        // lane_fg0_tr; the tile lives in the shared-memory pools' area, dead
        // during those ops).  Float only: the fixed-point kernels spill with it
        h->sc_tr = h->dec.precision == PL_F32 ? env_int("PLB_SC_TR", 1) : 0;
        if (!uses_list(kind) || adaptive(kind))
            h->sc_cfg = env_int("PLB_SC_LANES", 1) ? plan_lanes(*h) : plan_rung(*h, 1, false);
            // L2 hints of the frame-per-lane pass: segments <= 256 values kept
            // (evict_last), larger ones and the channel streamed (evict_first).
            // FA@4.5 dB float SC pass 23.1 -> 21.7 ms per 2^20 frames; int8 is
            // slower with hints (9.4 -> 9.9 ms), so only float takes them
            // Three classes (round 2, with the GR1 / chained ops): <= 64 values
            // evict_last, <= 256 evict_normal: 15.65 -> 15.4 ms
            h->sc_keep = env_int("PLB_SC_KEEP", h->dec.precision == PL_F32 ? 64 : 0);
            h->sc_keep_hi = env_int("PLB_SC_KEEP_HI", h->dec.precision == PL_F32 ? 256 : 0);
            // ... and dead global segments dropped from the L2 after their
            // last read (float: SC pass 21.9 -> 20.7 ms)
            h->sc_discard = env_int("PLB_SC_DISCARD", h->dec.precision == PL_F32 ? 1 : 0);
            h->list_discard = env_int("PLB_LIST_DISCARD", h->dec.precision == PL_F32 ? 1 : 0);
            // float sub-warp list kernels: chained F ops pay where depth pools
            // spill to the L2 (N >= 2048), big fused leaves where everything is
            // shared-memory resident (kernels.cu kChainKernel)
            h->list_alt = env_int("PLB_LIST_ALT", h->dec.precision == PL_F32 && h->nmax <= 1024 ? 1 : 0);
            h->host_chunk = env_int("PLB_HOST_CHUNK", 0);
        if (kind == PL_KIND_FA_SSCL)
            for (int ll = 2; ll <= l; ll *= 2) h->rungs.push_back(plan_rung(*h, ll, true, true));
        else if (uses_list(kind))
            h->rungs.push_back(plan_rung(*h, l, true, adaptive(kind)));
        for (const auto& r : h->rungs) {
            RungCfg sm;
            if (adaptive(kind) && r.team <= 1 && env_int("PLB_SMALL_RUNGS", 1)) {
                if (r.fpw > 1) {
                    // 32 lanes per frame.  Measured crossovers (FA@4.5 dB, N=2048):
                    // float gains up to one frame per resident warp (L=2 rung,
                    // 4.5k frames: 0.84 -> 0.63 ms); int8 / int16 only with at
                    // most ~8 frames per SM (at 4.5k frames the 8-lane
                    // sub-warps stay faster: 0.42 vs 0.65 ms)
                    sm = plan_rung(*h, r.l, true, true, 1);
                    sm.small_max = h->dec.precision == PL_F32 ? int64_t(sm.grid) * sm.wpb : int64_t(h->sms) * 8;
                } else if (r.l >= 16) {
                    // a team of 8 warps per frame (one frame per block, one
                    // wave): L=32 with 48 frames 1.52 -> 0.79 ms float, 0.76
                    // -> 0.63 int8; L=16 0.74 -> 0.53 float
                    std::vector<int> cands;
                    for (int sg = h->nmax; sg >= 8; sg >>= 1) cands.push_back(sg);
                    if (cands.empty()) cands.push_back(h->nmax);
                    sm = plan_team(*h, r.l, plb::kMaxTeam, cands);
                    sm.small_max = sm.grid;
                }
            }
            h->rungs_small.push_back(sm);
        }
        // speculative tail of the FA ladder (PLB_SPEC=0: off): the plans of
        // the last three rungs for at most spec_max frames, one block per
        // frame (team plans at L >= 16, warp 0 of a block in solo mode below),
        // so that the blocks of all three are resident together
        if (kind == PL_KIND_FA_SSCL && h->rungs.size() >= 3 && env_int("PLB_SPEC", 1)) {
            h->spec_max = std::max(1, env_int("PLB_SPEC_MAX", h->sms / 2));
            for (size_t i = h->rungs.size() - 3; i < h->rungs.size(); ++i) {
                RungCfg c = h->rungs_small[i].grid > 0 ? h->rungs_small[i] : h->rungs[i];
                if (c.fpw > 1) c = plan_rung(*h, c.l, true, true, 1);
                c.grid = std::min(c.grid, h->spec_max);
                h->spec.push_back(c);
            }
        }
        int64_t gs = 0;
        auto acc = [&](const RungCfg& r) {
            gs = std::max<int64_t>(gs, r.gscratch_total());
        };
        if (h->sc_cfg.grid) acc(h->sc_cfg);
        for (const auto& r : h->rungs) acc(r);
        for (const auto& r : h->rungs_small)
            if (r.grid) acc(r);
        h->gscratch_bytes = gs;
        ensure_exec(*h, 0);
        *out = h;
        return PL_OK;
    } catch (const ConfigError& e) {
        int rc = fail(nullptr, PL_ERR_CONFIG, e.what());
        pl_destroy(h);
        return rc;
    } catch (const std::exception& e) {
        int rc = fail(nullptr, PL_ERR_CUDA, e.what());
        pl_destroy(h);
        return rc;
    }
}

const char* pl_last_error(const pl_handle* h) {
    return h ? h->err.c_str() : g_thread_err.c_str();
}

void pl_destroy(pl_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    for (void* p : h->allocs) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        for (int j = 0; j < 2; ++j)
            if (h->ex[i].d_lists[j]) cudaFree(h->ex[i].d_lists[j]);
        if (h->ex[i].d_hist) cudaFree(h->ex[i].d_hist);
        if (h->ex[i].d_sorted) cudaFree(h->ex[i].d_sorted);
        if (h->ex[i].done) cudaEventDestroy(h->ex[i].done);
        if (h->ex[i].ev_fork) cudaEventDestroy(h->ex[i].ev_fork);
        for (int j = 0; j < 2; ++j) {
            if (h->ex[i].ev_join[j]) cudaEventDestroy(h->ex[i].ev_join[j]);
            if (h->ex[i].s_spec[j]) cudaStreamDestroy(h->ex[i].s_spec[j]);
        }
        if (h->s_comp[i]) cudaStreamDestroy(h->s_comp[i]);
    }
    for (int i = 0; i < pl_handle::kStage; ++i) {
        if (h->d_in[i]) cudaFree(h->d_in[i]);
        if (h->d_cid[i]) cudaFree(h->d_cid[i]);
        if (h->d_off[i]) cudaFree(h->d_off[i]);
        if (h->h_stage_off[i]) cudaFreeHost(h->h_stage_off[i]);
        if (h->d_out[i]) cudaFree(h->d_out[i]);
        if (h->h_stage_in[i]) cudaFreeHost(h->h_stage_in[i]);
        if (h->h_stage_out[i]) cudaFreeHost(h->h_stage_out[i]);
        if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
        if (h->ev_dec[i]) cudaEventDestroy(h->ev_dec[i]);
        if (h->ev_d2h[i]) cudaEventDestroy(h->ev_d2h[i]);
    }
    for (cudaEvent_t ev : h->prof_ev) cudaEventDestroy(ev);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h;
}

int64_t pl_llr_stride(const pl_handle* h) { return h ? h->nmax : 0; }
int64_t pl_payload_stride(const pl_handle* h) { return h ? h->pstride : 0; }
int64_t pl_codeword_stride(const pl_handle* h) { return h ? h->cstride : 0; }
int32_t pl_precision(const pl_handle* h) { return h ? h->dec.precision : -1; }
int64_t pl_last_launches(const pl_handle* h) { return h ? h->launches : 0; }

#ifdef PLB_OPTIME
// profiling build only: cycles and counts per list-op kind of frame 0
int pl_debug_optime(unsigned long long* out, int reset) {
    return plb::read_optime(out, reset != 0) == cudaSuccess ? PL_OK : PL_ERR_CUDA;
}
#endif

int pl_list_paths(pl_handle* h, uint32_t* alive, float* metric) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if ((alive == nullptr) != (metric == nullptr))
        return fail(h, PL_ERR_ARG, "alive and metric buffers are set together");
    h->path_alive = alive;
    h->path_metric = metric;
    return PL_OK;
}

int pl_set_host_chunk(pl_handle* h, int64_t frames) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if (frames < 0) return fail(h, PL_ERR_ARG, "chunk size must be >= 0");
    h->host_chunk = frames;
    return PL_OK;
}

int pl_set_llr_layout(pl_handle* h, int32_t layout) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if (layout != PL_LLR_FRAME_MAJOR && layout != PL_LLR_INTERLEAVED32)
        return fail(h, PL_ERR_ARG, "unknown LLR layout");
    if (layout == PL_LLR_INTERLEAVED32 &&
        (uses_list(h->dec.kind) || h->codes.size() != 1 || !h->sc_cfg.lanes))
        return fail(h, PL_ERR_CONFIG,
                    "the interleaved LLR layout is for SC / SSC handles with one code (frame-per-lane pass)");
    h->llr_layout = layout;
    return PL_OK;
}

int pl_frame_latency(pl_handle* h, uint32_t* lat_ns) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    h->lat_ns = lat_ns;
    return PL_OK;
}

int pl_kernel_selftest(int32_t device, uint64_t* mismatches) {
    if (!mismatches) return fail(nullptr, PL_ERR_ARG, "null argument");
    if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, PL_ERR_CUDA, "no such CUDA device");
    unsigned long long m = 0;
    const cudaError_t e = plb::kernel_selftest(&m);
    if (e != cudaSuccess) return fail(nullptr, PL_ERR_CUDA, cudaGetErrorString(e));
    *mismatches = m;
    return PL_OK;
}

int pl_profile(pl_handle* h, int32_t enable) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    h->profiling = enable != 0;
    return PL_OK;
}

int32_t pl_last_kernel_ms(pl_handle* h, float* ms, int32_t* kind, int32_t* l, int32_t max) {
    if (!h || !h->profiling) return 0;
    // decode kernels only (the bucketing kernels are counted in launches
    // but not timed)
    const int32_t n = int32_t(std::min<int64_t>(int64_t(h->prof_kind.size()), max));
    for (int32_t i = 0; i < n; ++i) {
        float t = 0.f;
        if (cudaEventSynchronize(h->prof_ev[size_t(2 * i + 1)]) != cudaSuccess ||
            cudaEventElapsedTime(&t, h->prof_ev[size_t(2 * i)], h->prof_ev[size_t(2 * i + 1)]) != cudaSuccess)
            return -1;
        if (ms) ms[i] = t;
        if (kind) kind[i] = h->prof_kind[size_t(i)];
        if (l) l[i] = h->prof_l[size_t(i)];
    }
    return n;
}

int pl_decode(pl_handle* h, const void* llr, const int32_t* code_id, int64_t nframes,
              uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc, float* metric,
              void* stream) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if (nframes < 0 || (nframes > 0 && (!llr || !payload)))
        return fail(h, PL_ERR_ARG, "llr and payload buffers are required");
    if (nframes > INT32_MAX) return fail(h, PL_ERR_ARG, "too many frames in one call");
    try {
        if (h->llr_layout == PL_LLR_INTERLEAVED32 && code_id)
            return fail(h, PL_ERR_CONFIG, "the interleaved LLR layout takes no per-frame code ids");
        run_decode(*h, llr, code_id, nframes, payload, codeword, crc_ok, esc, metric,
                   static_cast<cudaStream_t>(stream), 0, nullptr, h->lat_ns, true,
                   h->llr_layout == PL_LLR_INTERLEAVED32);
        h->err.clear();
        return PL_OK;
    } catch (const std::exception& e) {
        return fail(h, PL_ERR_CUDA, e.what());
    }
}

int pl_decode_packed(pl_handle* h, const void* llr, const int64_t* llr_offset, const int32_t* code_id,
                     int64_t nframes, uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc,
                     float* metric, void* stream) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if (nframes < 0 || (nframes > 0 && (!llr || !llr_offset || !payload)))
        return fail(h, PL_ERR_ARG, "llr, llr_offset and payload buffers are required");
    if (nframes > INT32_MAX) return fail(h, PL_ERR_ARG, "too many frames in one call");
    if (h->llr_layout != PL_LLR_FRAME_MAJOR)
        return fail(h, PL_ERR_CONFIG, "the interleaved LLR layout is accepted by pl_decode only");
    try {
        run_decode(*h, llr, code_id, nframes, payload, codeword, crc_ok, esc, metric,
                   static_cast<cudaStream_t>(stream), 0, llr_offset, h->lat_ns, true);
        h->err.clear();
        return PL_OK;
    } catch (const std::exception& e) {
        return fail(h, PL_ERR_CUDA, e.what());
    }
}

namespace {
int decode_host_impl(pl_handle* h, const void* llr, const int64_t* offsets, const int32_t* code_id,
                     int64_t nframes, uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok,
                     uint8_t* esc, float* metric);
}

int pl_decode_host(pl_handle* h, const void* llr, const int32_t* code_id, int64_t nframes,
                   uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc,
                   float* metric) {
    return decode_host_impl(h, llr, nullptr, code_id, nframes, payload, codeword, crc_ok, esc, metric);
}

int pl_decode_host_packed(pl_handle* h, const void* llr, const int64_t* llr_offset,
                          const int32_t* code_id, int64_t nframes, uint8_t* payload,
                          uint8_t* codeword, uint8_t* crc_ok, uint8_t* esc, float* metric) {
    if (h && nframes > 0 && !llr_offset) return fail(h, PL_ERR_ARG, "llr_offset is required");
    return decode_host_impl(h, llr, llr_offset, code_id, nframes, payload, codeword, crc_ok, esc, metric);
}

} // extern "C"

namespace {
int decode_host_impl(pl_handle* h, const void* llr, const int64_t* offsets, const int32_t* code_id,
                     int64_t nframes, uint8_t* payload, uint8_t* codeword, uint8_t* crc_ok,
                     uint8_t* esc, float* metric) {
    if (!h) return fail(nullptr, PL_ERR_ARG, "null handle");
    if (nframes < 0 || (nframes > 0 && (!llr || !payload)))
        return fail(h, PL_ERR_ARG, "llr and payload buffers are required");
    if (h->llr_layout != PL_LLR_FRAME_MAJOR)
        return fail(h, PL_ERR_CONFIG, "the interleaved LLR layout is accepted by pl_decode only");
    // packed frames: ascending, 16-byte aligned offsets (the kernels read
    // the channel with 16-byte vectors), code ids in range
    auto frame_n = [&](int64_t f) {
        const int32_t c = code_id ? code_id[f] : 0;
        return (c >= 0 && c < int32_t(h->codes.size())) ? h->codes[size_t(c)].n : -1;
    };
    if (offsets) {
        for (int64_t f = 0; f < nframes; ++f) {
            const int n = frame_n(f);
            if (n < 0) return fail(h, PL_ERR_ARG, "code id out of range");
            if (offsets[f] < 0 || (offsets[f] * h->esz) % 16 != 0)
                return fail(h, PL_ERR_ARG, "packed frame offsets must be non-negative and 16-byte aligned");
            if (f > 0 && offsets[f] < offsets[f - 1] + frame_n(f - 1))
                return fail(h, PL_ERR_ARG, "packed frames must be ascending and must not overlap");
        }
    }
    try {
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        if (!h->s_comp[0]) {
            ck(cudaStreamCreateWithFlags(&h->s_comp[0], cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&h->s_comp[1], cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking), "stream");
            for (int i = 0; i < pl_handle::kStage; ++i) {
                ck(cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&h->ev_dec[i], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&h->ev_d2h[i], cudaEventDisableTiming), "event");
            }
        }
        // ~20 chunks so the copies of one chunk overlap the decode of another
        // and the pipeline fill / drain stays short (measured: cfg1 e2e 16.2 ->
        // 16.7 Gb/s going from 8 to 16 chunks, 18.50 -> 18.61 at ~21; float
        // cfg0 best at 8192 frames).  Multi-code batches keep 16: every chunk
        // also buckets its frames by code (cfg3 e2e 5.6 at 16, 5.2 at 20).
        // Adaptive kinds on int8 LLRs: ~8 chunks, since every chunk pays the
        // latency of the upper ladder rungs (a few frames each) and the int8
        // copies are short (measured FA@4.5 dB int8 e2e 33.1 -> 39.2-40.7
        // Gb/s; the PCIe-bound float / int16 ladders keep 16: 11.25 vs 11.09,
        // 21.8 vs 20.9)
        const int64_t chunk = h->host_chunk > 0 ? h->host_chunk
                              : adaptive(h->dec.kind) && h->esz == 1
                                  ? std::clamp<int64_t>((nframes + 7) / 8, 8192, 131072)
                              : h->codes.size() > 1 ? std::clamp<int64_t>((nframes + 15) / 16, 8192, 65536)
                                                  : std::clamp<int64_t>((nframes + 19) / 20, 8192, 65536);
        const int64_t in_bytes = h->nmax * int64_t(h->esz);
        const int64_t nchunks = (nframes + chunk - 1) / chunk;
        // input element range of a chunk (packed: first offset .. end of its
        // last frame; padded: nf strides)
        auto in_range = [&](int64_t f0, int64_t nf, int64_t& e0, int64_t& e1) {
            if (offsets) {
                e0 = offsets[f0];
                e1 = offsets[f0 + nf - 1] + frame_n(f0 + nf - 1);
            } else {
                e0 = f0 * h->nmax;
                e1 = (f0 + nf) * h->nmax;
            }
        };
        int64_t need = chunk * in_bytes;
        if (offsets) {
            need = 16;
            for (int64_t c = 0; c < nchunks; ++c) {
                int64_t e0, e1;
                in_range(c * chunk, std::min(chunk, nframes - c * chunk), e0, e1);
                need = std::max(need, (e1 - e0) * int64_t(h->esz));
            }
        }
        // per frame output record: payload | codeword | crc | esc | metric
        const int64_t ob_pay = h->pstride, ob_cw = codeword ? h->cstride : 0;
        if (h->stage_frames < chunk || h->in_cap < need || (offsets && !h->d_off[0])) {
            const int64_t cap = std::max(need, chunk * in_bytes);
            for (int i = 0; i < pl_handle::kStage; ++i) {
                if (h->d_in[i]) cudaFree(h->d_in[i]);
                if (h->d_cid[i]) cudaFree(h->d_cid[i]);
                if (h->d_off[i]) cudaFree(h->d_off[i]);
                if (h->h_stage_off[i]) cudaFreeHost(h->h_stage_off[i]);
                if (h->d_out[i]) cudaFree(h->d_out[i]);
                if (h->h_stage_in[i]) cudaFreeHost(h->h_stage_in[i]);
                if (h->h_stage_out[i]) cudaFreeHost(h->h_stage_out[i]);
                ck(cudaMalloc(&h->d_in[i], size_t(cap)), "cudaMalloc");
                ck(cudaMalloc(&h->d_cid[i], size_t(chunk) * 4), "cudaMalloc");
                ck(cudaMalloc(&h->d_off[i], size_t(chunk) * 8), "cudaMalloc");
                ck(cudaMallocHost(&h->h_stage_off[i], size_t(chunk) * 8), "cudaMallocHost");
                ck(cudaMalloc(&h->d_out[i], size_t(chunk * (h->pstride + h->cstride + 6) + 64)), "cudaMalloc");
                ck(cudaMallocHost(&h->h_stage_in[i], size_t(cap)), "cudaMallocHost");
                ck(cudaMallocHost(&h->h_stage_out[i], size_t(chunk * (h->pstride + h->cstride + 6))),
                   "cudaMallocHost");
            }
            h->stage_frames = chunk;
            h->in_cap = cap;
        }
        const bool pin_in = is_pinned_host(llr);
        const bool pin_out = is_pinned_host(payload) && (!codeword || is_pinned_host(codeword)) &&
                             (!crc_ok || is_pinned_host(crc_ok)) && (!esc || is_pinned_host(esc)) &&
                             (!metric || is_pinned_host(metric));
        int64_t launches = 0;
        std::vector<int64_t> pending(pl_handle::kStage, -1);
        auto finish_chunk = [&](int64_t c) {
            // unpack a chunk that went through the host staging buffer
            const int b = int(c % pl_handle::kStage);
            ck(cudaEventSynchronize(h->ev_d2h[b]), "sync");
            if (pin_out) return;
            const int64_t f0 = c * chunk, nf = std::min(chunk, nframes - f0);
            const uint8_t* o = h->h_stage_out[b];
            std::memcpy(payload + f0 * h->pstride, o, size_t(nf * ob_pay));
            o += nf * ob_pay;
            if (codeword) std::memcpy(codeword + f0 * h->cstride, o, size_t(nf * ob_cw));
            o += nf * ob_cw;
            if (crc_ok) std::memcpy(crc_ok + f0, o, size_t(nf));
            o += nf;
            if (esc) std::memcpy(esc + f0, o, size_t(nf));
            o += nf;
            if (metric) std::memcpy(metric + f0, o, size_t(nf) * 4);
        };
        for (int64_t c = 0; c < nchunks; ++c) {
            const int b = int(c % pl_handle::kStage); // staging buffer
            const int e = int(c & 1);                 // execution context + compute stream
            const int64_t f0 = c * chunk, nf = std::min(chunk, nframes - f0);
            if (pending[size_t(b)] >= 0) {
                finish_chunk(pending[size_t(b)]);
                pending[size_t(b)] = -1;
            }
            int64_t e0, e1;
            in_range(f0, nf, e0, e1);
            const int64_t nbytes = (e1 - e0) * int64_t(h->esz);
            const char* src = static_cast<const char*>(llr) + e0 * int64_t(h->esz);
            if (!pin_in) {
                std::memcpy(h->h_stage_in[b], src, size_t(nbytes));
                src = static_cast<const char*>(h->h_stage_in[b]);
            }
            ck(cudaStreamWaitEvent(h->s_h2d, h->ev_dec[b], 0), "wait");
            ck(cudaMemcpyAsync(h->d_in[b], src, size_t(nbytes), cudaMemcpyHostToDevice, h->s_h2d), "h2d");
            if (offsets) {
                // chunk-relative offsets (the chunk's input starts at its first frame)
                for (int64_t i = 0; i < nf; ++i) h->h_stage_off[b][i] = offsets[f0 + i] - e0;
                ck(cudaMemcpyAsync(h->d_off[b], h->h_stage_off[b], size_t(nf) * 8, cudaMemcpyHostToDevice,
                                   h->s_h2d),
                   "h2d");
            }
            if (code_id)
                ck(cudaMemcpyAsync(h->d_cid[b], code_id + f0, size_t(nf) * 4, cudaMemcpyHostToDevice,
                                   h->s_h2d),
                   "h2d");
            ck(cudaEventRecord(h->ev_h2d[b], h->s_h2d), "record");
            ck(cudaStreamWaitEvent(h->s_comp[e], h->ev_h2d[b], 0), "wait");
            ck(cudaStreamWaitEvent(h->s_comp[e], h->ev_d2h[b], 0), "wait");
            uint8_t* o = h->d_out[b];
            uint8_t* d_pay = o;
            uint8_t* d_cw = codeword ? o + nf * ob_pay : nullptr;
            uint8_t* d_ok = o + nf * (ob_pay + ob_cw);
            uint8_t* d_esc = d_ok + nf;
            float* d_met = reinterpret_cast<float*>(d_esc + nf);
            // metric must be 4-byte aligned
            const uintptr_t mis = reinterpret_cast<uintptr_t>(d_met) & 3u;
            if (mis) d_met = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(d_met) + (4 - mis));
            run_decode(*h, h->d_in[b], code_id ? h->d_cid[b] : nullptr, nf, d_pay, d_cw, d_ok, d_esc,
                       d_met, h->s_comp[e], e, offsets ? h->d_off[b] : nullptr);
            launches += h->launches;
            ck(cudaEventRecord(h->ev_dec[b], h->s_comp[e]), "record");
            ck(cudaStreamWaitEvent(h->s_d2h, h->ev_dec[b], 0), "wait");
            auto d2h = [&](void* dst_pinned, uint8_t* dst_stage, const void* srcp, size_t bytes) {
                void* dst = pin_out ? dst_pinned : static_cast<void*>(dst_stage);
                ck(cudaMemcpyAsync(dst, srcp, bytes, cudaMemcpyDeviceToHost, h->s_d2h), "d2h");
            };
            uint8_t* st = h->h_stage_out[b];
            d2h(payload + f0 * h->pstride, st, d_pay, size_t(nf * ob_pay));
            st += nf * ob_pay;
            if (codeword) d2h(codeword + f0 * h->cstride, st, d_cw, size_t(nf * ob_cw));
            st += nf * ob_cw;
            if (crc_ok) d2h(crc_ok + f0, st, d_ok, size_t(nf));
            st += nf;
            if (esc) d2h(esc + f0, st, d_esc, size_t(nf));
            st += nf;
            if (metric) d2h(metric + f0, st, d_met, size_t(nf) * 4);
            ck(cudaEventRecord(h->ev_d2h[b], h->s_d2h), "record");
            pending[size_t(b)] = c;
        }
        for (int b = 0; b < pl_handle::kStage; ++b)
            if (pending[size_t(b)] >= 0) finish_chunk(pending[size_t(b)]);
        // finish in chunk order is not required: chunks write disjoint ranges
        h->launches = launches;
        h->err.clear();
        return PL_OK;
    } catch (const std::exception& e) {
        return fail(h, PL_ERR_CUDA, e.what());
    }
}

} // namespace
