// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the *unmodified* reference decoder headers and
// sources under /root/reference/proj (compiled in place by oracle/Makefile,
// output only into oracle/_ref/).  It exposes exactly the calls the parity
// tests and bench.py's cpu_baseline / --impl reference leg need:
//
//   polref_create/decode/destroy  -> FrameDecoder<R>(code, tree, kind, L)
//                                    + decode()  (proj/include/polar/decoders.hpp:37-85)
//                                    with the tree chosen as run_montecarlo
//                                    does (proj/src/sim.cpp:161-164)
//   polref_list_decode            -> ListDecoder<R>::decode + alive/metric
//                                    introspection (list_decoder.hpp:77-93)
//   polref_tree                   -> PruneTree (prune_tree.hpp:49-73)
//   polref_crc / polref_crc_check -> CrcEngine::compute/check (crc.cpp:121-154)
//   polref_construct_frozen       -> construct_frozen (code.cpp:63-77)
//   polref_channel                -> run_frame's input side: FrameRng,
//                                    random_payload, encode_systematic,
//                                    transmit (sim.cpp:45-51, channel.hpp)
//   polref_montecarlo             -> run_montecarlo (sim.cpp:148-174),
//                                    timing off: the error counts of a sweep
//   polref_format_csv_row         -> format_csv_row (report.cpp:40-50)
//   polref_frozen_load / _save    -> load_frozen_file / save_frozen_file
//                                    (code.cpp:164-194)
//
// Payload and codeword outputs are packed MSB-first, the BitVector byte
// convention (bit_vector.hpp:11-14, 57-59).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "polar/channel.hpp"
#include "polar/code.hpp"
#include "polar/crc.hpp"
#include "polar/decoders.hpp"
#include "polar/errors.hpp"
#include "polar/prune_tree.hpp"
#include "polar/report.hpp"
#include "polar/sim.hpp"

using namespace polar;

namespace {

void set_err(char* err, int errlen, const std::string& msg) {
    if (err && errlen > 0) {
        std::snprintf(err, std::size_t(errlen), "%s", msg.c_str());
    }
}

BitVector mask_from_bytes(const std::uint8_t* b, int n) {
    BitVector v(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) v.set(std::size_t(i), b[i] != 0);
    return v;
}

void pack_bits(const BitVector& v, std::uint8_t* out) {
    const std::size_t nb = (v.size() + 7) / 8;
    for (std::size_t k = 0; k < nb; ++k) out[k] = v.byte(k);
}

std::optional<CrcSpec> crc_opt(const char* spec) {
    if (!spec || !*spec) return std::nullopt;
    return CrcSpec::parse(spec);
}

struct Handle {
    PolarCode code;
    std::unique_ptr<PruneTree> tree;
    DecoderKind kind;
    int l;
    int precision; // 0 f32, 1 int8, 2 int16
};

template <class R>
void decode_range(const Handle& h, const R* llr, std::int64_t f0, std::int64_t f1,
                  std::uint8_t* payload, std::uint8_t* codeword,
                  std::uint8_t* crc_ok, std::uint8_t* esc, double* metric) {
    FrameDecoder<R> dec(h.code, *h.tree, h.kind, h.l);
    const std::size_t pbytes = std::size_t(h.code.payload_size() + 7) / 8;
    const std::size_t cbytes = std::size_t(h.code.n + 7) / 8;
    for (std::int64_t f = f0; f < f1; ++f) {
        const DecodeResult r = dec.decode(llr + std::size_t(f) * std::size_t(h.code.n));
        if (payload) pack_bits(r.payload, payload + std::size_t(f) * pbytes);
        if (codeword) pack_bits(r.codeword, codeword + std::size_t(f) * cbytes);
        if (crc_ok) crc_ok[f] = r.crc_ok ? 1 : 0;
        if (esc) esc[f] = std::uint8_t(r.escalation_level);
        if (metric) metric[f] = r.metric;
    }
}

template <class F>
void parallel_frames(std::int64_t nframes, int nthreads, F&& fn) {
    if (nthreads <= 1 || nframes < 2) {
        fn(std::int64_t(0), nframes);
        return;
    }
    const int nt = int(std::min<std::int64_t>(nthreads, nframes));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
        const std::int64_t a = nframes * t / nt, b = nframes * (t + 1) / nt;
        pool.emplace_back([&fn, a, b] { fn(a, b); });
    }
    for (auto& th : pool) th.join();
}

} // namespace

extern "C" {

void* polref_create(int n, int k, const std::uint8_t* frozen, const char* crc_spec,
                    int kind, int l, int precision, int r0, int r1, int rep,
                    int spc, int rep_max, int spc_max, char* err, int errlen) {
    try {
        auto h = std::make_unique<Handle>();
        h->code = make_code(n, k, mask_from_bytes(frozen, n), crc_opt(crc_spec));
        h->kind = DecoderKind(kind);
        PruningConfig pc{r0 != 0, r1 != 0, rep != 0, spc != 0, rep_max, spc_max};
        // sim.cpp:161-164: the pruned tree only for SSC-family decoders
        h->tree = std::make_unique<PruneTree>(
            h->code.frozen, decoder_uses_pruning(h->kind) ? pc : PruningConfig::none());
        h->l = l;
        h->precision = precision;
        // construct once to surface ConfigError at create time
        switch (precision) {
        case 0: FrameDecoder<float>(h->code, *h->tree, h->kind, l); break;
        case 1: FrameDecoder<std::int8_t>(h->code, *h->tree, h->kind, l); break;
        case 2: FrameDecoder<std::int16_t>(h->code, *h->tree, h->kind, l); break;
        default: throw ConfigError("bad precision");
        }
        return h.release();
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}

void polref_destroy(void* h) { delete static_cast<Handle*>(h); }

int polref_payload_bits(void* hv) {
    return static_cast<Handle*>(hv)->code.payload_size();
}

int polref_decode(void* hv, const void* llr, std::int64_t nframes, int nthreads,
                  std::uint8_t* payload, std::uint8_t* codeword, std::uint8_t* crc_ok,
                  std::uint8_t* esc, double* metric) {
    const Handle& h = *static_cast<Handle*>(hv);
    try {
        parallel_frames(nframes, nthreads, [&](std::int64_t a, std::int64_t b) {
            switch (h.precision) {
            case 0:
                decode_range<float>(h, static_cast<const float*>(llr), a, b, payload,
                                    codeword, crc_ok, esc, metric);
                break;
            case 1:
                decode_range<std::int8_t>(h, static_cast<const std::int8_t*>(llr), a,
                                          b, payload, codeword, crc_ok, esc, metric);
                break;
            default:
                decode_range<std::int16_t>(h, static_cast<const std::int16_t*>(llr),
                                           a, b, payload, codeword, crc_ok, esc,
                                           metric);
                break;
            }
        });
    } catch (const std::exception&) {
        return 1;
    }
    return 0;
}

// One frame through ListDecoder<R> directly, with post-decode introspection.
int polref_list_decode(void* hv, const void* llr, int l, int select_by_crc,
                       std::uint8_t* payload, std::uint8_t* codeword,
                       std::uint8_t* crc_ok, double* metric, std::uint8_t* alive,
                       double* slot_metric, char* err, int errlen) {
    const Handle& h = *static_cast<Handle*>(hv);
    try {
        auto run = [&](auto tag) {
            using R = decltype(tag);
            ListDecoder<R> dec(h.code, *h.tree, h.l, PsumLayout::copy);
            const DecodeResult r =
                dec.decode(static_cast<const R*>(llr), l, select_by_crc != 0);
            pack_bits(r.payload, payload);
            pack_bits(r.codeword, codeword);
            *crc_ok = r.crc_ok;
            *metric = r.metric;
            for (int p = 0; p < h.l; ++p) {
                alive[p] = dec.is_alive(p) ? 1 : 0;
                slot_metric[p] = dec.is_alive(p) ? dec.metric_of(p) : 0.0;
            }
        };
        if (h.precision == 0) run(float{});
        else if (h.precision == 1) run(std::int8_t{});
        else run(std::int16_t{});
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
    return 0;
}

// Node list: 6 ints per node (kind, depth, leaf_begin, size, left, right).
int polref_tree(const std::uint8_t* frozen, int n, int r0, int r1, int rep, int spc,
                int rep_max, int spc_max, std::int32_t* out, int max_nodes, char* err,
                int errlen) {
    try {
        PruneTree t(mask_from_bytes(frozen, n),
                    PruningConfig{r0 != 0, r1 != 0, rep != 0, spc != 0, rep_max, spc_max});
        const int cnt = int(t.node_count());
        if (cnt > max_nodes) throw ConfigError("node buffer too small");
        for (int i = 0; i < cnt; ++i) {
            const TreeNode& nd = t.node(i);
            out[6 * i + 0] = int(nd.kind);
            out[6 * i + 1] = nd.depth;
            out[6 * i + 2] = nd.leaf_begin;
            out[6 * i + 3] = nd.size;
            out[6 * i + 4] = nd.left;
            out[6 * i + 5] = nd.right;
        }
        return cnt;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return -1;
    }
}

// CRC of `len` bits given as 0/1 bytes.
int polref_crc(const char* spec, const std::uint8_t* bits, std::int64_t len,
               std::uint64_t* out, char* err, int errlen) {
    try {
        CrcEngine eng(CrcSpec::parse(spec));
        BitVector v(static_cast<std::size_t>(len));
        for (std::int64_t i = 0; i < len; ++i) v.set(std::size_t(i), bits[i] != 0);
        *out = eng.compute(v);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int polref_crc_check(const char* spec, const std::uint8_t* bits, std::int64_t len) {
    try {
        CrcEngine eng(CrcSpec::parse(spec));
        BitVector v(static_cast<std::size_t>(len));
        for (std::int64_t i = 0; i < len; ++i) v.set(std::size_t(i), bits[i] != 0);
        return eng.check(v) ? 1 : 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int polref_construct_frozen(int n, int reliable, double design, std::uint8_t* out,
                            char* err, int errlen) {
    try {
        const BitVector m = construct_frozen(n, reliable, design);
        for (int i = 0; i < n; ++i) out[i] = m.get(std::size_t(i)) ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// run_frame's input side (sim.cpp:48-51) for frames [frame0, frame0+nframes):
// info bits as 0/1 bytes (k per frame) and channel LLRs in the requested
// representation (precision 0 f32, 1 int8, 2 int16; scale <= 0 = default).
// punct: "" or n characters T / P / S (the PuncturePattern of make_code)
int polref_channel_ids(int n, int k, const std::uint8_t* frozen, const char* crc_spec,
                       double ebn0_db, std::uint64_t seed, std::uint64_t frame0,
                       const std::uint64_t* ids, std::int64_t nframes, int precision,
                       float scale, std::uint8_t* info_out, void* llr_out, int nthreads,
                       const char* punct, char* err, int errlen);

int polref_channel(int n, int k, const std::uint8_t* frozen, const char* crc_spec,
                   double ebn0_db, std::uint64_t seed, std::uint64_t frame0,
                   std::int64_t nframes, int precision, float scale,
                   std::uint8_t* info_out, void* llr_out, int nthreads, const char* punct,
                   char* err, int errlen) {
    return polref_channel_ids(n, k, frozen, crc_spec, ebn0_db, seed, frame0, nullptr, nframes,
                              precision, scale, info_out, llr_out, nthreads, punct, err, errlen);
}

// frame f of the batch is global frame ids[f] (ids == nullptr: frame0 + f)
int polref_channel_ids(int n, int k, const std::uint8_t* frozen, const char* crc_spec,
                       double ebn0_db, std::uint64_t seed, std::uint64_t frame0,
                       const std::uint64_t* ids, std::int64_t nframes, int precision,
                       float scale, std::uint8_t* info_out, void* llr_out, int nthreads,
                       const char* punct, char* err, int errlen) {
    try {
        std::optional<PuncturePattern> pp;
        if (punct && *punct) {
            PuncturePattern p;
            for (const char* c = punct; *c; ++c) {
                p.use.push_back(*c == 'T' ? ChannelUse::transmitted
                                : *c == 'P' ? ChannelUse::punctured : ChannelUse::shortened);
                p.transmitted += *c == 'T';
            }
            pp = std::move(p);
        }
        const PolarCode code = make_code(n, k, mask_from_bytes(frozen, n), crc_opt(crc_spec), pp);
        const double sigma2 = awgn_sigma2(code, ebn0_db);
        parallel_frames(nframes, nthreads, [&](std::int64_t a, std::int64_t b) {
            for (std::int64_t f = a; f < b; ++f) {
                FrameRng rng(seed, ids ? ids[f] : frame0 + std::uint64_t(f));
                const BitVector info = random_payload(rng, std::size_t(k));
                const BitVector x = encode_systematic(code, info);
                if (info_out)
                    for (int i = 0; i < k; ++i)
                        info_out[std::size_t(f) * std::size_t(k) + std::size_t(i)] =
                            info.get(std::size_t(i));
                const std::size_t off = std::size_t(f) * std::size_t(n);
                if (precision == 0)
                    transmit<float>(code, x, sigma2, rng,
                                    scale > 0 ? scale : default_quant_scale<float>(),
                                    static_cast<float*>(llr_out) + off);
                else if (precision == 1)
                    transmit<std::int8_t>(code, x, sigma2, rng,
                                          scale > 0 ? scale : default_quant_scale<std::int8_t>(),
                                          static_cast<std::int8_t*>(llr_out) + off);
                else
                    transmit<std::int16_t>(code, x, sigma2, rng,
                                           scale > 0 ? scale : default_quant_scale<std::int16_t>(),
                                           static_cast<std::int16_t*>(llr_out) + off);
            }
        });
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// out: 7 doubles per point (ebn0, frames, bit_errors, frame_errors, ber,
// fer, esc_mean); returns the number of points or -1
int polref_montecarlo(int n, int k, const std::uint8_t* frozen, const char* crc_spec, int kind,
                      int l, int precision, float quant_scale, int r0, int r1, int rep, int spc,
                      int rep_max, int spc_max, double ebn0_min, double ebn0_max, double ebn0_step,
                      std::uint64_t max_frames, std::uint64_t max_fe, std::uint64_t seed,
                      int workers, int max_points, double* out, char* err, int errlen) {
    try {
        SimConfig cfg;
        cfg.code = make_code(n, k, mask_from_bytes(frozen, n), crc_opt(crc_spec));
        cfg.decoder = DecoderKind(kind);
        cfg.list_size = l;
        cfg.precision = precision == 0 ? Precision::f32 : precision == 1 ? Precision::q8 : Precision::q16;
        cfg.quant_scale = quant_scale;
        cfg.pruning = PruningConfig{r0 != 0, r1 != 0, rep != 0, spc != 0, rep_max, spc_max};
        cfg.ebn0_min = ebn0_min;
        cfg.ebn0_max = ebn0_max;
        cfg.ebn0_step = ebn0_step;
        cfg.max_frames = max_frames;
        cfg.max_fe = max_fe;
        cfg.seed = seed;
        cfg.workers = workers;
        cfg.timing = false;
        const SimStats st = run_montecarlo(cfg);
        int i = 0;
        for (const auto& p : st.points) {
            if (i >= max_points) break;
            double* o = out + 7 * i++;
            o[0] = p.ebn0_db;
            o[1] = double(p.frames);
            o[2] = double(p.bit_errors);
            o[3] = double(p.frame_errors);
            o[4] = p.ber;
            o[5] = p.fer;
            o[6] = p.esc_mean;
        }
        return i;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return -1;
    }
}

// v: ebn0, frames, bit_errors, frame_errors, ber, fer, ti_mbps, lat_avg_us,
// lat_worst_us, esc_mean
int polref_format_csv_row(const double* v, char* buf, int len) {
    PointStats p;
    p.ebn0_db = v[0];
    p.frames = std::uint64_t(v[1]);
    p.bit_errors = std::uint64_t(v[2]);
    p.frame_errors = std::uint64_t(v[3]);
    p.ber = v[4];
    p.fer = v[5];
    p.ti_mbps = v[6];
    p.lat_avg_us = v[7];
    p.lat_worst_us = v[8];
    p.esc_mean = v[9];
    const std::string row = format_csv_row(p);
    std::snprintf(buf, std::size_t(len), "%s", row.c_str());
    return int(row.size());
}

// returns 0, 1 (ParseError), 2 (IoError) with the message in err
int polref_frozen_load(const char* path, int* n, int* k, std::uint8_t* out, int cap, char* err,
                       int errlen) {
    try {
        const FrozenFile f = load_frozen_file(path);
        *n = f.n;
        *k = f.k;
        for (int i = 0; i < f.n && i < cap; ++i) out[i] = f.mask.get(std::size_t(i)) ? 1 : 0;
        return 0;
    } catch (const ParseError& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const IoError& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

int polref_frozen_save(const char* path, int n, int k, const std::uint8_t* frozen, char* err,
                       int errlen) {
    try {
        save_frozen_file(path, n, k, mask_from_bytes(frozen, n));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

// load_puncture_file: uses 0 T / 1 P / 2 S; 0, 1 (ParseError), 2 (IoError)
int polref_puncture_load(const char* path, int* n, std::uint8_t* out, int cap, char* err, int errlen) {
    try {
        const PuncturePattern p = load_puncture_file(path);
        *n = int(p.use.size());
        for (int i = 0; i < *n && i < cap; ++i) out[i] = std::uint8_t(p.use[std::size_t(i)]);
        return 0;
    } catch (const ParseError& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const IoError& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

} // extern "C"
