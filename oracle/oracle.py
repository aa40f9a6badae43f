"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the two CPU checkers.

* ``Oracle``     — the plain-C restatement (oracle/polar_oracle.c).
* ``Reference``  — the unmodified reference decoder compiled from
                   /root/reference/proj (oracle/_ref/libpolar_ref.so, see
                   oracle/Makefile and oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  Nothing in the product
package (paper_1710_08314_b200/) imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libpolar_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpolar_ref.so")
REF_SRC = "/root/reference/proj"

KINDS = {"sc": 0, "ssc": 1, "scl": 2, "sscl": 3, "ca_sscl": 4, "pa_sscl": 5, "fa_sscl": 6}
PRECISIONS = {"f32": 0, "i8": 1, "i16": 2}

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


_BUILT = False


def build_oracle(force: bool = False) -> str:
    """make keeps it incremental: a no-op when the .so is up to date."""
    global _BUILT
    if force or not _BUILT or not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
        _BUILT = True
    return ORACLE_SO


def build_ref(force: bool = False) -> str | None:
    """Compile oracle/_ref when the reference sources are present (make keeps
    it current); elsewhere (the GPU box) use the prebuilt library."""
    if not os.path.isdir(REF_SRC):
        return REF_SO if os.path.exists(REF_SO) else None
    if force and os.path.exists(REF_SO):
        os.remove(REF_SO)
    subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    return REF_SO


ADAPTER_BIN = os.path.join(HERE, "_ref", "check_adapter")


def build_adapter() -> str | None:
    """oracle/_ref/check_adapter (integration/check_adapter.cpp: the
    reference's FrameDecoder<R> and the GpuFrameDecoder<R> adapter in one
    binary) when the reference sources are present; else the prebuilt one."""
    if not os.path.isdir(REF_SRC):
        return ADAPTER_BIN if os.path.exists(ADAPTER_BIN) else None
    subprocess.check_call(["make", "-s", "-C", HERE, "adapter"])
    return ADAPTER_BIN


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _pruning_tuple(pruning):
    if pruning is None:
        return (1, 1, 1, 1, 0, 4)
    return tuple(int(x) for x in pruning)


class _Outputs:
    def __init__(self, nframes, n, psize):
        self.payload = np.zeros((nframes, (psize + 7) // 8), np.uint8)
        self.codeword = np.zeros((nframes, (n + 7) // 8), np.uint8)
        self.crc_ok = np.zeros(nframes, np.uint8)
        self.esc = np.zeros(nframes, np.uint8)
        self.metric = np.zeros(nframes, np.float64)


class Oracle:
    """FrameDecoder-shaped wrapper over the C restatement."""

    def __init__(self, n, k, frozen, crc=None, kind="ca_sscl", l=8, precision="f32",
                 pruning=None):
        lib = C.CDLL(build_oracle())
        lib.orc_create.restype = C.c_void_p
        lib.orc_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_uint64,
                                   C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                   C.c_int, C.c_void_p, C.c_char_p, C.c_int]
        lib.orc_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int] + [C.c_void_p] * 5
        lib.orc_list_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 6
        lib.orc_destroy.argtypes = [C.c_void_p]
        self.lib = lib
        self.n, self.k = n, k
        self.frozen = np.ascontiguousarray(frozen, np.uint8)
        w, poly, refl, init, xo = crc if crc else (0, 0, 0, 0, 0)
        self.crc_width = w
        self.psize = k + w
        self.precision = precision
        pr = np.array(_pruning_tuple(pruning), np.int32)
        err = C.create_string_buffer(256)
        self.h = lib.orc_create(n, k, _ptr(self.frozen), w, poly, refl, init, xo,
                                KINDS[kind], l, PRECISIONS[precision], _ptr(pr), err, 256)
        if not self.h:
            raise ValueError(err.value.decode())
        self.l = l

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_destroy(self.h)
            self.h = None

    def decode(self, llr, nthreads=1):
        llr = np.ascontiguousarray(llr)
        nframes = llr.size // self.n
        o = _Outputs(nframes, self.n, self.psize)
        rc = self.lib.orc_decode(self.h, _ptr(llr), nframes, nthreads, _ptr(o.payload),
                                 _ptr(o.codeword), _ptr(o.crc_ok), _ptr(o.esc), _ptr(o.metric))
        if rc:
            raise RuntimeError("oracle decode failed")
        return o

    def list_decode(self, llr, l, select_by_crc):
        llr = np.ascontiguousarray(llr)
        o = _Outputs(1, self.n, self.psize)
        ok = np.zeros(1, np.uint8)
        met = np.zeros(1, np.float64)
        alive = np.zeros(self.l, np.uint8)
        sm = np.zeros(self.l, np.float64)
        rc = self.lib.orc_list_decode(self.h, _ptr(llr), l, int(select_by_crc), _ptr(o.payload),
                                      _ptr(o.codeword), _ptr(ok), _ptr(met), _ptr(alive), _ptr(sm))
        if rc:
            raise ValueError("bad list decode request")
        return o.payload[0], o.codeword[0], bool(ok[0]), float(met[0]), alive, sm


def oracle_tree(frozen, pruning=None):
    lib = C.CDLL(build_oracle())
    lib.orc_tree.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    fz = np.ascontiguousarray(frozen, np.uint8)
    n = fz.size
    out = np.zeros((2 * n, 6), np.int32)
    pr = np.array(_pruning_tuple(pruning), np.int32)
    cnt = lib.orc_tree(_ptr(fz), n, _ptr(pr), _ptr(out), 2 * n)
    if cnt < 0:
        raise ValueError("bad tree request")
    return out[:cnt].copy()


def oracle_crc(spec, bits):
    lib = C.CDLL(build_oracle())
    lib.orc_crc.restype = C.c_uint64
    lib.orc_crc.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p,
                            C.c_int64]
    b = np.ascontiguousarray(bits, np.uint8)
    w, poly, refl, init, xo = spec
    return int(lib.orc_crc(w, poly, refl, init, xo, _ptr(b), b.size))


class Reference:
    """The unmodified reference FrameDecoder<R> via oracle/_ref."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            so = build_ref()
            if so is None or not os.path.exists(so):
                raise FileNotFoundError("oracle/_ref/libpolar_ref.so not built")
            lib = C.CDLL(so)
            lib.polref_create.restype = C.c_void_p
            lib.polref_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int,
                                          C.c_int, C.c_int] + [C.c_int] * 6 + [C.c_char_p, C.c_int]
            lib.polref_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int] + [C.c_void_p] * 5
            lib.polref_list_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int] + \
                [C.c_void_p] * 6 + [C.c_char_p, C.c_int]
            lib.polref_destroy.argtypes = [C.c_void_p]
            lib.polref_tree.argtypes = [C.c_void_p, C.c_int] + [C.c_int] * 6 + \
                [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
            lib.polref_crc.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_char_p,
                                       C.c_int]
            lib.polref_crc_check.argtypes = [C.c_char_p, C.c_void_p, C.c_int64]
            lib.polref_construct_frozen.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p,
                                                    C.c_char_p, C.c_int]
            lib.polref_channel.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_double,
                                           C.c_uint64, C.c_uint64, C.c_int64, C.c_int, C.c_float,
                                           C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_char_p,
                                           C.c_int]
            lib.polref_channel_ids.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_char_p,
                                               C.c_double, C.c_uint64, C.c_uint64, C.c_void_p,
                                               C.c_int64, C.c_int, C.c_float, C.c_void_p,
                                               C.c_void_p, C.c_int, C.c_char_p, C.c_char_p,
                                               C.c_int]
            cls._lib = lib
        return cls._lib

    def __init__(self, n, k, frozen, crc_spec="", kind="ca_sscl", l=8, precision="f32",
                 pruning=None):
        lib = self.lib()
        self.n, self.k = n, k
        self.frozen = np.ascontiguousarray(frozen, np.uint8)
        pr = _pruning_tuple(pruning)
        err = C.create_string_buffer(512)
        self.h = lib.polref_create(n, k, _ptr(self.frozen), (crc_spec or "").encode(),
                                   KINDS[kind], l, PRECISIONS[precision], *pr, err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.psize = lib.polref_payload_bits(C.c_void_p(self.h))
        self.l = l

    def __del__(self):
        if getattr(self, "h", None):
            self.lib().polref_destroy(self.h)
            self.h = None

    def decode(self, llr, nthreads=1):
        llr = np.ascontiguousarray(llr)
        nframes = llr.size // self.n
        o = _Outputs(nframes, self.n, self.psize)
        rc = self.lib().polref_decode(self.h, _ptr(llr), nframes, nthreads, _ptr(o.payload),
                                      _ptr(o.codeword), _ptr(o.crc_ok), _ptr(o.esc),
                                      _ptr(o.metric))
        if rc:
            raise RuntimeError("reference decode failed")
        return o

    def list_decode(self, llr, l, select_by_crc):
        llr = np.ascontiguousarray(llr)
        o = _Outputs(1, self.n, self.psize)
        ok = np.zeros(1, np.uint8)
        met = np.zeros(1, np.float64)
        alive = np.zeros(self.l, np.uint8)
        sm = np.zeros(self.l, np.float64)
        err = C.create_string_buffer(256)
        rc = self.lib().polref_list_decode(self.h, _ptr(llr), l, int(select_by_crc),
                                           _ptr(o.payload), _ptr(o.codeword), _ptr(ok),
                                           _ptr(met), _ptr(alive), _ptr(sm), err, 256)
        if rc:
            raise ValueError(err.value.decode())
        return o.payload[0], o.codeword[0], bool(ok[0]), float(met[0]), alive, sm


def ref_tree(frozen, pruning=None):
    lib = Reference.lib()
    fz = np.ascontiguousarray(frozen, np.uint8)
    n = fz.size
    out = np.zeros((2 * n, 6), np.int32)
    err = C.create_string_buffer(256)
    cnt = lib.polref_tree(_ptr(fz), n, *_pruning_tuple(pruning), _ptr(out), 2 * n, err, 256)
    if cnt < 0:
        raise ValueError(err.value.decode())
    return out[:cnt].copy()


def ref_crc(spec_text, bits):
    lib = Reference.lib()
    b = np.ascontiguousarray(bits, np.uint8)
    out = np.zeros(1, np.uint64)
    err = C.create_string_buffer(256)
    if lib.polref_crc(spec_text.encode(), _ptr(b), b.size, _ptr(out), err, 256):
        raise ValueError(err.value.decode())
    return int(out[0])


def ref_construct_frozen(n, reliable, design):
    lib = Reference.lib()
    out = np.zeros(n, np.uint8)
    err = C.create_string_buffer(256)
    if lib.polref_construct_frozen(n, reliable, design, _ptr(out), err, 256):
        raise ValueError(err.value.decode())
    return out


def ref_channel(n, k, frozen, crc_spec, ebn0_db, seed, frame0, nframes, precision="f32",
                scale=0.0, nthreads=8, punct=""):
    """run_frame's inputs (sim.cpp:48-51): info bits and channel LLRs."""
    lib = Reference.lib()
    fz = np.ascontiguousarray(frozen, np.uint8)
    info = np.zeros((nframes, k), np.uint8)
    dt = {"f32": np.float32, "i8": np.int8, "i16": np.int16}[precision]
    llr = np.zeros((nframes, n), dt)
    err = C.create_string_buffer(256)
    rc = lib.polref_channel(n, k, _ptr(fz), (crc_spec or "").encode(), ebn0_db, seed, frame0,
                            nframes, PRECISIONS[precision], scale, _ptr(info), _ptr(llr),
                            nthreads, punct.encode(), err, 256)
    if rc:
        raise ValueError(err.value.decode())
    return info, llr


def ref_channel_ids(n, k, frozen, crc_spec, ebn0_db, seed, ids, precision="f32", scale=0.0,
                    nthreads=8):
    """ref_channel over explicit global frame indices (mixed-code batches)."""
    lib = Reference.lib()
    fz = np.ascontiguousarray(frozen, np.uint8)
    ids = np.ascontiguousarray(ids, np.uint64)
    info = np.zeros((ids.size, k), np.uint8)
    dt = {"f32": np.float32, "i8": np.int8, "i16": np.int16}[precision]
    llr = np.zeros((ids.size, n), dt)
    err = C.create_string_buffer(256)
    rc = lib.polref_channel_ids(n, k, _ptr(fz), (crc_spec or "").encode(), ebn0_db, seed, 0,
                                _ptr(ids), ids.size, PRECISIONS[precision], scale, _ptr(info),
                                _ptr(llr), nthreads, b"", err, 256)
    if rc:
        raise ValueError(err.value.decode())
    return info, llr


def ref_montecarlo(n, k, frozen, crc_spec, kind, l, precision, pruning, ebn0_min, ebn0_max,
                   ebn0_step, max_frames, max_fe, seed=42, quant_scale=0.0, workers=8):
    """The reference's run_montecarlo (sim.cpp:148-174), timing off: per
    point (ebn0, frames, bit_errors, frame_errors, ber, fer, esc_mean)."""
    lib = Reference.lib()
    lib.polref_montecarlo.argtypes = (
        [C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_float]
        + [C.c_int] * 6 + [C.c_double] * 3 + [C.c_uint64] * 3
        + [C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int])
    fz = np.ascontiguousarray(frozen, np.uint8)
    out = np.zeros((64, 7), np.float64)
    err = C.create_string_buffer(512)
    npts = lib.polref_montecarlo(n, k, _ptr(fz), (crc_spec or "").encode(), KINDS[kind], l,
                                 PRECISIONS[precision], quant_scale, *_pruning_tuple(pruning),
                                 ebn0_min, ebn0_max, ebn0_step, max_frames, max_fe, seed, workers,
                                 64, _ptr(out), err, 512)
    if npts < 0:
        raise ValueError(err.value.decode())
    return out[:npts]


def ref_format_csv_row(vals):
    """The reference's format_csv_row (report.cpp:40-50) for (ebn0, frames,
    bit_errors, frame_errors, ber, fer, ti_mbps, lat_avg_us, lat_worst_us,
    esc_mean)."""
    lib = Reference.lib()
    lib.polref_format_csv_row.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
    v = np.ascontiguousarray(vals, np.float64)
    buf = C.create_string_buffer(512)
    lib.polref_format_csv_row(_ptr(v), buf, 512)
    return buf.value.decode()


def ref_frozen_load(path, nmax=1 << 16):
    """load_frozen_file; returns (n, k, mask) or raises (kind, message)."""
    lib = Reference.lib()
    lib.polref_frozen_load.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                       C.c_char_p, C.c_int]
    n, k = C.c_int(), C.c_int()
    out = np.zeros(nmax, np.uint8)
    err = C.create_string_buffer(512)
    rc = lib.polref_frozen_load(str(path).encode(), C.byref(n), C.byref(k), _ptr(out), nmax, err, 512)
    if rc:
        raise RuntimeError(("parse" if rc == 1 else "io"), err.value.decode())
    return n.value, k.value, out[:n.value]


def ref_frozen_save(path, n, k, frozen):
    lib = Reference.lib()
    lib.polref_frozen_save.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int]
    fz = np.ascontiguousarray(frozen, np.uint8)
    err = C.create_string_buffer(512)
    if lib.polref_frozen_save(str(path).encode(), n, k, _ptr(fz), err, 512):
        raise RuntimeError("io", err.value.decode())


def ref_puncture_load(path, nmax=1 << 16):
    """load_puncture_file -> channel uses (0 T / 1 P / 2 S) or raises (kind, message)."""
    lib = Reference.lib()
    lib.polref_puncture_load.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int, C.c_char_p,
                                         C.c_int]
    n = C.c_int()
    out = np.zeros(nmax, np.uint8)
    err = C.create_string_buffer(512)
    rc = lib.polref_puncture_load(str(path).encode(), C.byref(n), _ptr(out), nmax, err, 512)
    if rc:
        raise RuntimeError(("parse" if rc == 1 else "io"), err.value.decode())
    return out[:n.value]
