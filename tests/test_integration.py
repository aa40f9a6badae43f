"""The C ABI is consumable from plain C and C++ exactly as INTEGRATION.md
shows: compile a translation unit against include/ and link the library;
and the reference-side adapter (integration/gpu_frame_decoder.hpp, compiled
against the reference's own headers) decodes like FrameDecoder<R>."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

C_SRC = r"""
#include <stdio.h>
#include <string.h>
#include "polar_b200.h"
#include "polar_b200_sim.h"
int main(void) {
    pl_crc c;
    if (pl_crc_parse("32-GZIP", &c) != PL_OK) return 1;
    unsigned char bits[72];
    const char* s = "123456789";
    for (int i = 0; i < 72; ++i) bits[i] = (unsigned char)((s[i / 8] >> (7 - i % 8)) & 1);
    unsigned long long v = 0;
    if (pl_crc_compute(&c, bits, 72, (uint64_t*)&v) != PL_OK) return 2;
    if (v != 0xCBF43926ull) return 3;
    unsigned char frozen[16];
    if (pl_construct_frozen_bhat(16, 12, 0.5, frozen) != PL_OK) return 4;
    pl_code code = {16, 4, frozen, c};
    code.crc.width = 8; code.crc.poly = 7; code.crc.reflect = 0; code.crc.init = 0; code.crc.xorout = 0;
    pl_decoder d = {PL_KIND_FA_SSCL, 1, PL_F32, {1, 1, 1, 1, 0, 4}};
    pl_handle* h = NULL;
    if (pl_create(&code, 1, &d, 0, &h) != PL_ERR_CONFIG) return 5;   /* adaptive needs L >= 2 */
    if (strstr(pl_last_error(NULL), "at least 2") == NULL) return 6;
    puts("ok");
    return 0;
}
"""


def test_c_consumer_compiles_links_and_runs(native, tmp_path):
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "consumer.c"
    src.write_text(C_SRC)
    exe = tmp_path / "consumer"
    lib = os.path.join(ROOT, "paper_1710_08314_b200")
    subprocess.check_call([cc, "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                           "-L", lib, "-lpolar_b200", f"-Wl,-rpath,{lib}", "-lstdc++"],
                          env={**os.environ, "LIBRARY_PATH": lib})
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stderr)
    assert out.stdout.strip() == "ok"


@pytest.mark.gpu
def test_reference_side_adapter_matches_frame_decoder(native, gpu):
    """oracle/_ref/check_adapter: GpuFrameDecoder<R> and
    the reference's FrameDecoder<R> (decoders.hpp:60-85) in one binary, on
    frames from the reference's own channel: payload, codeword, crc_ok,
    escalation level and metric of every frame equal, decode() too, and the
    same ConfigError messages (cfg1-, cfg0- and cfg2-like codes, int16 FA,
    PA, SSC)."""
    from oracle import oracle

    exe = oracle.build_adapter()
    if exe is None:
        pytest.fail("oracle/_ref/check_adapter was not built (build() builds it with /root/reference)")
    r = subprocess.run([exe, ROOT], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter ok" in r.stdout
