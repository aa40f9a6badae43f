// The drop-in boundary exercised from the reference's side: in one binary,
// the reference's own FrameDecoder<R> (proj/include/polar/decoders.hpp:37-85)
// and this repo's GpuFrameDecoder<R> (integration/gpu_frame_decoder.hpp, over
// libpolar_b200.so) decode the same frames -- made by the reference's own
// FrameRng / random_payload / encode_systematic / transmit
// (channel.hpp:17-89) -- and every DecodeResult field is compared.  Codes use
// the committed GA frozen files through the reference's load_frozen_file.
//
//   check_adapter <repo root>      (exit 0 = every field of every frame equal)
//
// Built by oracle/Makefile (target `adapter`, into oracle/_ref/); run by
// tests/test_integration.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gpu_frame_decoder.hpp"
#include "polar/channel.hpp"
#include "polar/errors.hpp"

using namespace polar;

namespace {

struct Case {
    const char* name;
    const char* frozen;
    int n, k;
    const char* crc;
    DecoderKind kind;
    int l;
    PruningConfig pruning;
    double ebn0;
    int frames;
};

template <class R>
int run_case(const std::string& root, const Case& c, float scale) {
    const FrozenFile ff = load_frozen_file(root + "/oracle/frozen/" + c.frozen);
    const PolarCode code = make_code(c.n, c.k, ff.mask, CrcSpec::parse(c.crc));
    const PruneTree tree(code.frozen, decoder_uses_pruning(c.kind) ? c.pruning : PruningConfig::none());
    FrameDecoder<R> cpu(code, tree, c.kind, c.l);
    GpuFrameDecoder<R> gpu(code, c.pruning, c.kind, c.l);
    const double sigma2 = awgn_sigma2(code, c.ebn0);
    std::vector<R> llr(std::size_t(c.frames) * std::size_t(c.n));
    for (int f = 0; f < c.frames; ++f) {
        FrameRng rng(42, std::uint64_t(f));
        const BitVector info = random_payload(rng, std::size_t(code.k));
        transmit<R>(code, encode_systematic(code, info), sigma2, rng,
                    scale > 0 ? scale : default_quant_scale<R>(), llr.data() + std::size_t(f) * c.n);
    }
    const std::vector<DecodeResult> got = gpu.decode_batch(llr.data(), c.frames);
    int bad[5] = {0, 0, 0, 0, 0}, esc_hist[64] = {0};
    for (int f = 0; f < c.frames; ++f) {
        const DecodeResult want = cpu.decode(llr.data() + std::size_t(f) * c.n);
        const DecodeResult& g = got[std::size_t(f)];
        bad[0] += !(g.payload == want.payload);
        bad[1] += !(g.codeword == want.codeword);
        bad[2] += g.crc_ok != want.crc_ok;
        bad[3] += g.escalation_level != want.escalation_level;
        bad[4] += g.metric != want.metric;
        if (want.escalation_level < 64) ++esc_hist[want.escalation_level];
    }
    // the one-frame decode() of the adapter, as run_frame calls it (sim.cpp:56)
    const DecodeResult one = gpu.decode(llr.data());
    const DecodeResult want0 = cpu.decode(llr.data());
    const bool one_ok = one.payload == want0.payload && one.metric == want0.metric &&
                        one.escalation_level == want0.escalation_level;
    const int nbad = bad[0] + bad[1] + bad[2] + bad[3] + bad[4] + !one_ok;
    std::printf("%-24s frames %5d  mismatches: payload %d codeword %d crc_ok %d esc %d metric %d "
                "decode() %s  esc levels:",
                c.name, c.frames, bad[0], bad[1], bad[2], bad[3], bad[4], one_ok ? "ok" : "BAD");
    for (int l = 1; l < 64; l *= 2)
        if (esc_hist[l]) std::printf(" L%d:%d", l, esc_hist[l]);
    std::printf("\n");
    return nbad;
}

// ConfigError surfaces from the adapter exactly where FrameDecoder<R> throws it
int check_errors(const std::string& root) {
    const FrozenFile ff = load_frozen_file(root + "/oracle/frozen/ga_n2048_k1723_c32_d4.5.frozen");
    const PolarCode code = make_code(2048, 1723, ff.mask, CrcSpec::parse("32-GZIP"));
    const PolarCode nocrc = make_code(2048, 1755, ff.mask);
    const PruneTree tree(code.frozen, PruningConfig{});
    int bad = 0;
    auto expect = [&](const char* what, auto&& make_cpu, auto&& make_gpu) {
        std::string a, b;
        try { make_cpu(); } catch (const ConfigError& e) { a = e.what(); }
        try { make_gpu(); } catch (const ConfigError& e) { b = e.what(); }
        const bool ok = !a.empty() && a == b;
        std::printf("config error %-22s reference '%s' / adapter '%s' %s\n", what, a.c_str(), b.c_str(),
                    ok ? "ok" : "BAD");
        bad += !ok;
    };
    expect("L=3", [&] { FrameDecoder<float>(code, tree, DecoderKind::ca_sscl, 3); },
           [&] { GpuFrameDecoder<float>(code, PruningConfig{}, DecoderKind::ca_sscl, 3); });
    expect("FA with L=1", [&] { FrameDecoder<float>(code, tree, DecoderKind::fa_sscl, 1); },
           [&] { GpuFrameDecoder<float>(code, PruningConfig{}, DecoderKind::fa_sscl, 1); });
    expect("CA without CRC", [&] { FrameDecoder<float>(nocrc, tree, DecoderKind::ca_sscl, 8); },
           [&] { GpuFrameDecoder<float>(nocrc, PruningConfig{}, DecoderKind::ca_sscl, 8); });
    return bad;
}

} // namespace

int main(int argc, char** argv) {
    const std::string root = argc > 1 ? argv[1] : ".";
    const PruningConfig dflt{};
    PruningConfig rep8{};
    rep8.rep_max = 8;
    const char* g45 = "ga_n2048_k1723_c32_d4.5.frozen";
    int bad = 0;
    try {
        // configs[1]-like: CA-SCL L=8, int8 x4, REP_8-, 3.5 dB
        bad += run_case<std::int8_t>(root, {"cfg1 ca_sscl L8 i8", g45, 2048, 1723, "32-GZIP",
                                            DecoderKind::ca_sscl, 8, rep8, 3.5, 2048}, 4.0f);
        // configs[0]-like: CA-SCL L=4, float, 4.5 dB
        bad += run_case<float>(root, {"cfg0 ca_sscl L4 f32", g45, 2048, 1723, "32-GZIP",
                                      DecoderKind::ca_sscl, 4, dflt, 4.5, 2048}, 0.0f);
        // configs[2]-like: FA-SCL Lmax=32, float, 3.5 dB (every rung runs)
        bad += run_case<float>(root, {"cfg2 fa_sscl L32 f32", g45, 2048, 1723, "32-GZIP",
                                      DecoderKind::fa_sscl, 32, dflt, 3.5, 1024}, 0.0f);
        // the paper's int16 point and the PA / plain SSC variants
        bad += run_case<std::int16_t>(root, {"fa_sscl L32 i16", g45, 2048, 1723, "32-GZIP",
                                             DecoderKind::fa_sscl, 32, dflt, 3.0, 512}, 0.0f);
        bad += run_case<float>(root, {"pa_sscl L8 f32", g45, 2048, 1723, "32-GZIP",
                                      DecoderKind::pa_sscl, 8, dflt, 3.5, 512}, 0.0f);
        bad += run_case<float>(root, {"ssc f32", g45, 2048, 1723, "32-GZIP", DecoderKind::ssc, 1,
                                      dflt, 4.5, 512}, 0.0f);
        bad += check_errors(root);
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 2;
    }
    std::printf(bad ? "adapter MISMATCH\n" : "adapter ok: every DecodeResult field equal\n");
    return bad ? 1 : 0;
}
