// GpuFrameDecoder<R>: the adapter a maintainer of the reference adds to use
// the B200 decoder behind the reference's own types.
//
// Same constructor arguments and decode() contract as FrameDecoder<R>
// (reference proj/include/polar/decoders.hpp:37-85), plus decode_batch()
// for throughput.  R = float, std::int8_t or std::int16_t.  Compiled against
// the reference's headers (proj/include) and this repo's include/polar_b200.h;
// integration/check_adapter.cpp decodes through it next to FrameDecoder<R>
// and compares every DecodeResult field.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "polar/code.hpp"          // reference: PolarCode, CrcSpec
#include "polar/decode_result.hpp" // reference: DecodeResult
#include "polar/decoders.hpp"      // reference: DecoderKind
#include "polar/errors.hpp"        // reference: ConfigError
#include "polar/prune_tree.hpp"    // reference: PruningConfig
#include "polar_b200.h"            // this repo: the C ABI

namespace polar {

template <class R>
class GpuFrameDecoder {
public:
    // (layout: FrameDecoder's PsumLayout; copy and shared are decision-
    // identical in the reference, the GPU decoder has one layout)
    GpuFrameDecoder(const PolarCode& code, const PruningConfig& pruning, DecoderKind kind, int l,
                    PsumLayout layout = PsumLayout::copy, int device = 0)
        : code_(&code) {
        (void)layout;
        mask_.resize(std::size_t(code.n));
        for (int i = 0; i < code.n; ++i) mask_[std::size_t(i)] = code.frozen.get(std::size_t(i));
        pl_code c{code.n, code.k, mask_.data(), {0, 0, 0, 0, 0}, nullptr};
        if (code.crc) {
            const CrcSpec& s = code.crc->spec();
            c.crc = {s.width, s.reflect ? 1 : 0, s.poly, s.init, s.xorout};
        }
        // (the decoder ignores puncturing: punctured / shortened LLRs arrive
        // already demapped, as from transmit())
        pl_decoder d{int(kind), l, sizeof(R) == 1 ? PL_I8 : sizeof(R) == 2 ? PL_I16 : PL_F32,
                     {pruning.rate_zero, pruning.rate_one, pruning.repetition,
                      pruning.single_parity, pruning.rep_max, pruning.spc_max}};
        if (int rc = pl_create(&c, 1, &d, device, &h_); rc != PL_OK) {
            if (rc == PL_ERR_CONFIG) throw ConfigError(pl_last_error(nullptr));
            throw std::runtime_error(pl_last_error(nullptr));
        }
    }
    GpuFrameDecoder(const GpuFrameDecoder&) = delete;
    GpuFrameDecoder& operator=(const GpuFrameDecoder&) = delete;
    ~GpuFrameDecoder() { pl_destroy(h_); }

    // Host LLRs in (frame-major, code.n values each), DecodeResults out;
    // host<->device copies overlap decoding inside pl_decode_host.
    std::vector<DecodeResult> decode_batch(const R* llr, std::int64_t nframes) {
        const std::int64_t ps = pl_payload_stride(h_), cs = pl_codeword_stride(h_);
        const std::size_t nf = std::size_t(nframes);
        std::vector<std::uint8_t> pay(nf * std::size_t(ps)), cw(nf * std::size_t(cs));
        std::vector<std::uint8_t> ok(nf), esc(nf);
        std::vector<float> met(nf);
        if (pl_decode_host(h_, llr, nullptr, nframes, pay.data(), cw.data(), ok.data(), esc.data(),
                           met.data()) != PL_OK)
            throw std::runtime_error(pl_last_error(h_));
        std::vector<DecodeResult> out(nf);
        for (std::int64_t f = 0; f < nframes; ++f) {
            DecodeResult& r = out[std::size_t(f)];
            r.payload = truncate(BitVector::from_bytes(&pay[std::size_t(f * ps)], std::size_t(ps)),
                                 std::size_t(code_->payload_size()));
            r.codeword = truncate(BitVector::from_bytes(&cw[std::size_t(f * cs)], std::size_t(cs)),
                                  std::size_t(code_->n));
            r.crc_ok = ok[std::size_t(f)] != 0;
            r.escalation_level = esc[std::size_t(f)];
            r.metric = met[std::size_t(f)];
        }
        return out;
    }
    DecodeResult decode(const R* channel) { return decode_batch(channel, 1)[0]; }

private:
    static BitVector truncate(const BitVector& v, std::size_t n) {
        BitVector o(n);
        for (std::size_t i = 0; i < n; ++i) o.set(i, v.get(i));
        return o;
    }
    const PolarCode* code_;
    std::vector<std::uint8_t> mask_;
    pl_handle* h_ = nullptr;
};

} // namespace polar
