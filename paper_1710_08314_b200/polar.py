"""Host-side mirror of the reference decoder API over the C ABI.

Names, argument meaning and error behaviour follow the reference's C++
interface (/root/reference/proj/include/polar/):

  reference (C++)                         here (Python, over libpolar_b200.so)
  --------------------------------------- ------------------------------------
  CrcSpec{width,poly,reflect,init,xorout} CrcSpec (dataclass), CrcSpec.parse
    + CrcSpec::parse   crc.hpp:16-26
  CrcEngine::compute   crc.cpp:121-144    crc_compute
  PruningConfig        prune_tree.hpp:25-34 PruningConfig, PruningConfig.none()
  PruneTree            prune_tree.hpp:49-73 prune_tree() -> node array
  make_code            code.hpp:43-45     make_code -> PolarCode
  construct_frozen     code.hpp:55        construct_frozen (Bhattacharyya)
  DecoderKind          decoders.hpp:10-18 DecoderKind
  FrameDecoder<R>      decoders.hpp:37-103 FrameDecoder (batched: decode_batch;
    ::decode(const R*) -> DecodeResult      decode() for one frame)
  ConfigError / ParseError errors.hpp:9-21 ConfigError / ParseError

The decode path has no CPU fallback: if the native library or a GPU is
missing, constructing a FrameDecoder raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class IoError(OSError):
    """errors.hpp:19-21"""


class ConfigError(ValueError):
    """Invalid code, decoder or tree parameters (errors.hpp:9-11)."""


class ParseError(ValueError):
    """Malformed option string (errors.hpp:14-16)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the native library."""


def _raise(rc: int, msg: str):
    if rc == L.PL_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == L.PL_ERR_PARSE:
        raise ParseError(msg)
    if rc == L.PL_ERR_ARG:
        raise ValueError(msg)
    if rc == L.PL_ERR_IO:
        raise IoError(msg)
    raise DeviceError(msg)


def interleave32(llr):
    """PL_LLR_INTERLEAVED32 of a (frames, n) array: groups of 32 frames
    (zero-padded), 16-byte chunks interleaved -- chunk c of frame f at chunk
    index ((f // 32) * chunks + c) * 32 + f % 32 (include/polar_b200.h)."""
    llr = np.ascontiguousarray(llr)
    nf, n = llr.shape
    v = min(16 // llr.dtype.itemsize, n)
    g = (nf + 31) // 32
    buf = np.zeros((g * 32, n), llr.dtype)
    buf[:nf] = llr
    return np.ascontiguousarray(buf.reshape(g, 32, n // v, v).transpose(0, 2, 1, 3)).reshape(g * 32, n)


def pack_frames(frames, dtype):
    """Packed layout of variable-length frames (pl_decode_packed): frame i
    at element offset off[i], ascending, each 16-byte aligned."""
    dt = np.dtype(dtype)
    align = 16 // dt.itemsize
    off = np.zeros(len(frames), np.int64)
    pos = 0
    for i, f in enumerate(frames):
        off[i] = pos
        pos += -(-len(f) // align) * align
    buf = np.zeros(max(pos, align), dt)
    for i, f in enumerate(frames):
        buf[off[i]: off[i] + len(f)] = f
    return buf, off


def pack_batch(llr: np.ndarray, ns: np.ndarray):
    """pack_frames of a padded batch (frame f: llr[f, :ns[f]]), vectorised
    per frame length."""
    align = 16 // llr.dtype.itemsize
    ns = np.asarray(ns, np.int64)
    sz = -(-ns // align) * align
    off = np.zeros(ns.size, np.int64)
    if ns.size > 1:
        np.cumsum(sz[:-1], out=off[1:])
    buf = np.zeros(max(int(sz.sum()), align), llr.dtype)
    for n in np.unique(ns):
        rows = np.flatnonzero(ns == n)
        buf[(off[rows][:, None] + np.arange(n)).ravel()] = llr[rows, :n].ravel()
    return buf, off


def load_frozen_file(path: str):
    """load_frozen_file (code.cpp:164-185) -> (n, k, frozen mask as uint8)."""
    n, k = C.c_int32(), C.c_int32()
    rc = L.lib().pl_frozen_file_load(str(path).encode(), C.byref(n), C.byref(k), None, 0)
    if rc:
        _raise(rc, L.last_error(None))
    out = np.zeros(n.value, np.uint8)
    rc = L.lib().pl_frozen_file_load(str(path).encode(), C.byref(n), C.byref(k),
                                     out.ctypes.data_as(C.c_void_p), out.size)
    if rc:
        _raise(rc, L.last_error(None))
    return n.value, k.value, out


def save_frozen_file(path: str, n: int, k: int, frozen):
    """save_frozen_file (code.cpp:187-194)."""
    fz = (np.ascontiguousarray(frozen).astype(np.uint8) != 0).astype(np.uint8)
    assert fz.size == n
    rc = L.lib().pl_frozen_file_save(str(path).encode(), n, k, fz.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc, L.last_error(None))


class DecoderKind(enum.IntEnum):
    """decoders.hpp:10-18 (same order)."""
    sc = 0
    ssc = 1
    scl = 2
    sscl = 3
    ca_sscl = 4
    pa_sscl = 5
    fa_sscl = 6

    @property
    def uses_list(self):
        return self not in (DecoderKind.sc, DecoderKind.ssc)

    @property
    def uses_crc(self):
        return self in (DecoderKind.ca_sscl, DecoderKind.pa_sscl, DecoderKind.fa_sscl)

    @property
    def adaptive(self):
        return self in (DecoderKind.pa_sscl, DecoderKind.fa_sscl)

    @property
    def uses_pruning(self):
        return self not in (DecoderKind.sc, DecoderKind.scl)


class Precision(enum.IntEnum):
    f32 = 0
    i8 = 1
    i16 = 2


_NP_DTYPE = {"f32": np.float32, "i8": np.int8, "i16": np.int16}


@dataclass(frozen=True)
class CrcSpec:
    width: int = 32
    poly: int = 0x04C11DB7
    reflect: bool = True
    init: int = 0xFFFFFFFF
    xorout: int = 0xFFFFFFFF

    @staticmethod
    def parse(text: str) -> "CrcSpec":
        """CrcSpec::parse (crc.cpp:42-84): preset or width:poly:reflect:init:xorout."""
        out = L.pl_crc()
        rc = L.lib().pl_crc_parse(text.encode(), C.byref(out))
        if rc:
            _raise(rc, L.last_error(None))
        return CrcSpec(out.width, out.poly, bool(out.reflect), out.init, out.xorout)

    def to_c(self) -> "L.pl_crc":
        return L.pl_crc(self.width, int(self.reflect), self.poly, self.init, self.xorout)

    def raw(self) -> str:
        return f"{self.width}:{self.poly:x}:{int(self.reflect)}:{self.init:x}:{self.xorout:x}"


def crc_compute(spec: CrcSpec, bits) -> int:
    b = np.ascontiguousarray(bits, np.uint8)
    out = C.c_uint64(0)
    c = spec.to_c()
    rc = L.lib().pl_crc_compute(C.byref(c), b.ctypes.data_as(C.c_void_p), b.size, C.byref(out))
    if rc:
        _raise(rc, L.last_error(None))
    return int(out.value)


@dataclass(frozen=True)
class PruningConfig:
    """prune_tree.hpp:25-34: 0 caps mean unlimited."""
    rate_zero: bool = True
    rate_one: bool = True
    repetition: bool = True
    single_parity: bool = True
    rep_max: int = 0
    spc_max: int = 4

    @staticmethod
    def none() -> "PruningConfig":
        return PruningConfig(False, False, False, False, 0, 0)

    def to_c(self) -> "L.pl_pruning":
        return L.pl_pruning(int(self.rate_zero), int(self.rate_one), int(self.repetition),
                            int(self.single_parity), self.rep_max, self.spc_max)

    def as_tuple(self):
        return (int(self.rate_zero), int(self.rate_one), int(self.repetition),
                int(self.single_parity), self.rep_max, self.spc_max)


NODE_KINDS = ("branch", "frozen", "info", "R0", "R1", "REP", "SPC")


def prune_tree(frozen, cfg: PruningConfig = PruningConfig()) -> np.ndarray:
    """PruneTree node array, rows (kind, depth, leaf_begin, size, left, right)."""
    fz = np.ascontiguousarray(frozen, np.uint8)
    n = fz.size
    out = np.zeros((2 * n, 6), np.int32)
    c = cfg.to_c()
    cnt = L.lib().pl_tree_build(fz.ctypes.data_as(C.c_void_p), n, C.byref(c),
                                out.ctypes.data_as(C.c_void_p), 2 * n)
    if cnt < 0:
        raise ConfigError(L.last_error(None) or "bad decode tree request")
    return out[:cnt].copy()


@dataclass
class PolarCode:
    """code.hpp:29-41 (puncturing lives in the channel, never in the decoder)."""
    n: int
    k: int
    frozen: np.ndarray
    crc: CrcSpec | None = None
    info_pos: np.ndarray = field(default=None)
    # PuncturePattern.use (code.hpp:13-24): 0 T / 1 P / 2 S per position, or None
    channel_use: np.ndarray | None = None

    @property
    def crc_width(self) -> int:
        return self.crc.width if self.crc else 0

    @property
    def payload_size(self) -> int:
        return self.k + self.crc_width

    def rate(self) -> float:
        """code.hpp:40: information bits over transmitted channel uses"""
        t = self.n if self.channel_use is None else int((self.channel_use == 0).sum())
        return self.k / t

    def to_c(self) -> "L.pl_code":
        c = L.pl_code()
        c.n = self.n
        c.k = self.k
        c.frozen = self.frozen.ctypes.data_as(C.POINTER(C.c_uint8))
        c.crc = self.crc.to_c() if self.crc else L.pl_crc(0, 0, 0, 0, 0)
        c.channel_use = (self.channel_use.ctypes.data_as(C.POINTER(C.c_uint8))
                         if self.channel_use is not None else None)
        return c


def make_code(n: int, k: int, frozen, crc: CrcSpec | str | None = None, punct=None) -> PolarCode:
    """make_code (code.cpp:79-126): validates N, K, the open-position count and
    the puncture pattern (``punct``: n channel uses 0 T / 1 P / 2 S, or a
    "TPS..." string)."""
    if isinstance(crc, str):
        crc = CrcSpec.parse(crc)
    fz = (np.ascontiguousarray(frozen).astype(np.uint8) != 0).astype(np.uint8)
    if n < 2 or n & (n - 1):
        raise ConfigError(f"N must be a power of two >= 2 (got {n})")
    if k < 1:
        raise ConfigError(f"K must be at least 1 (got {k})")
    if fz.size != n:
        raise ConfigError(f"frozen mask has {fz.size} bits, code has N = {n}")
    w = crc.width if crc else 0
    open_ = int(n - fz.sum())
    if open_ != k + w:
        raise ConfigError(f"frozen mask leaves {open_} information positions, need K + CRC bits = {k + w}")
    use = None
    if punct is not None:
        if isinstance(punct, str):
            punct = ["TPS".index(ch) for ch in punct]
        use = np.ascontiguousarray(punct, np.uint8)
        if use.size != n:
            raise ConfigError(f"puncture pattern has {use.size} entries, code has N = {n}")
        if use.max(initial=0) > 2:
            raise ConfigError("channel uses must be 0 (T), 1 (P) or 2 (S)")
        t = int((use == 0).sum())
        if t < k + w:
            raise ConfigError(f"puncture pattern transmits only {t} symbols, fewer than K + CRC bits = {k + w}")
    return PolarCode(n, k, fz, crc, np.flatnonzero(fz == 0).astype(np.int32), use)


def load_puncture_file(path: str) -> np.ndarray:
    """load_puncture_file (code.cpp:196-221) -> channel uses (0 T / 1 P / 2 S)."""
    n = C.c_int32()
    rc = L.lib().pl_puncture_file_load(str(path).encode(), C.byref(n), None, 0)
    if rc:
        _raise(rc, L.last_error(None))
    out = np.zeros(n.value, np.uint8)
    rc = L.lib().pl_puncture_file_load(str(path).encode(), C.byref(n), out.ctypes.data_as(C.c_void_p),
                                       out.size)
    if rc:
        _raise(rc, L.last_error(None))
    return out


def construct_frozen(n: int, reliable: int, design_erasure: float) -> np.ndarray:
    """construct_frozen (code.cpp:63-77), Bhattacharyya ordering."""
    out = np.zeros(n, np.uint8)
    rc = L.lib().pl_construct_frozen_bhat(n, reliable, design_erasure,
                                          out.ctypes.data_as(C.c_void_p))
    if rc:
        raise ConfigError("bad construction request")
    return out


def construct_frozen_ga(n: int, reliable: int, design_ebn0_db: float, rate: float) -> np.ndarray:
    """Gaussian-approximation construction (absent from the reference)."""
    out = np.zeros(n, np.uint8)
    rc = L.lib().pl_construct_frozen_ga(n, reliable, design_ebn0_db, rate,
                                        out.ctypes.data_as(C.c_void_p))
    if rc:
        raise ConfigError("bad construction request")
    return out


def channel_device(code: PolarCode, ebn0_db: float, seed: int, frame0: int, nframes: int,
                   precision: str = "f32", scale: float = 0.0, device: int = 0, with_info=True):
    """Device-side channel (Philox, statistically equivalent to ``channel``)."""
    import torch

    dev = f"cuda:{device}"
    dt = {"f32": torch.float32, "i8": torch.int8, "i16": torch.int16}[precision]
    llr = torch.empty((nframes, code.n), dtype=dt, device=dev)
    info = torch.empty((nframes, code.k), dtype=torch.uint8, device=dev) if with_info else None
    c = code.to_c()
    s = torch.cuda.current_stream(device)
    rc = L.lib().pl_channel_generate_device(
        C.byref(c), ebn0_db, seed, frame0, nframes, int(Precision[precision]), scale,
        C.c_void_p(info.data_ptr()) if info is not None else None, C.c_void_p(llr.data_ptr()),
        C.c_void_p(s.cuda_stream))
    if rc:
        _raise(rc, "device channel generation failed")
    return info, llr


def channel(code: PolarCode, ebn0_db: float, seed: int, frame0: int, nframes: int,
            precision: str = "f32", scale: float = 0.0, nthreads: int = 0):
    """run_frame's inputs (sim.cpp:48-51), frame-keyed like FrameRng."""
    info = np.zeros((nframes, code.k), np.uint8)
    dt = _NP_DTYPE[precision]
    llr = np.zeros((nframes, code.n), dt)
    c = code.to_c()
    rc = L.lib().pl_channel_generate(C.byref(c), ebn0_db, seed, frame0, nframes,
                                     int(Precision[precision]), scale,
                                     info.ctypes.data_as(C.c_void_p),
                                     llr.ctypes.data_as(C.c_void_p), nthreads)
    if rc:
        _raise(rc, "channel generation failed")
    return info, llr


def channel_frames(code: PolarCode, ebn0_db: float, seed: int, frame_ids, llr_out, info_out=None,
                   precision: str = "f32", scale: float = 0.0, nthreads: int = 0):
    """Frames keyed by explicit global indices, written into rows of wider
    batch buffers (mixed-code batches): llr_out[i, :n], info_out[i, :k]."""
    ids = np.ascontiguousarray(frame_ids, np.uint64)
    assert llr_out.flags.c_contiguous and llr_out.shape[0] == ids.size
    c = code.to_c()
    rc = L.lib().pl_channel_generate_frames(
        C.byref(c), ebn0_db, seed, ids.ctypes.data_as(C.c_void_p), ids.size,
        int(Precision[precision]), scale,
        info_out.ctypes.data_as(C.c_void_p) if info_out is not None else None,
        info_out.shape[1] if info_out is not None else 0,
        llr_out.ctypes.data_as(C.c_void_p), llr_out.shape[1], nthreads)
    if rc:
        _raise(rc, "channel generation failed")


@dataclass
class DecodeResult:
    """decode_result.hpp:7-14 (payload/codeword as 0/1 numpy arrays)."""
    codeword: np.ndarray | None
    payload: np.ndarray
    crc_ok: bool
    escalation_level: int
    metric: float


def unpack_msb(packed: np.ndarray, nbits: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(packed, np.uint8), axis=-1)[..., :nbits]


class FrameDecoder:
    """FrameDecoder<R> (decoders.hpp:37-103) on the GPU, over a batch.

    ``codes`` is one PolarCode or a list of them (mixed-code batches pick a
    code per frame with ``code_id``).  ``precision`` is "f32", "i8" or "i16".
    """

    def __init__(self, codes, kind, l: int = 8, precision: str = "f32",
                 pruning: PruningConfig = PruningConfig(), device: int = 0,
                 psum_layout: str = "copy"):
        import torch  # device memory and streams only

        # PsumLayout (list_decoder.hpp:22): "copy" and "shared" are
        # decision-identical in the reference (test_list.cpp:253-289); the GPU
        # decoder has one layout (lazy pointer rows), so both are accepted
        if psum_layout not in ("copy", "shared"):
            raise ConfigError(f"unknown partial-sum layout {psum_layout!r}")

        self._torch = torch
        if isinstance(codes, PolarCode):
            codes = [codes]
        self.codes = list(codes)
        self.kind = DecoderKind(kind) if not isinstance(kind, str) else DecoderKind[kind]
        self.l = l if self.kind.uses_list else 1
        self.precision = Precision[precision] if isinstance(precision, str) else Precision(precision)
        self.pruning = pruning
        self.device = device
        arr = (L.pl_code * len(self.codes))(*[c.to_c() for c in self.codes])
        dec = L.pl_decoder(int(self.kind), l, int(self.precision), pruning.to_c())
        h = C.c_void_p()
        rc = L.lib().pl_create(arr, len(self.codes), C.byref(dec), device, C.byref(h))
        if rc:
            _raise(rc, L.last_error(None))
        self._h = h
        lib = L.lib()
        self.llr_stride = int(lib.pl_llr_stride(h))
        self.payload_stride = int(lib.pl_payload_stride(h))
        self.codeword_stride = int(lib.pl_codeword_stride(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                L.lib().pl_destroy(h)
            except TypeError:  # interpreter shutdown: the module globals are already gone
                pass

    @property
    def llr_dtype(self):
        t = self._torch
        return {Precision.f32: t.float32, Precision.i8: t.int8, Precision.i16: t.int16}[self.precision]

    def alloc_outputs(self, nframes: int, codeword: bool = False):
        t = self._torch
        dev = f"cuda:{self.device}"
        return {
            "payload": t.empty((nframes, self.payload_stride), dtype=t.uint8, device=dev),
            "codeword": t.empty((nframes, self.codeword_stride), dtype=t.uint8, device=dev) if codeword else None,
            "crc_ok": t.empty(nframes, dtype=t.uint8, device=dev),
            "esc": t.empty(nframes, dtype=t.uint8, device=dev),
            "metric": t.empty(nframes, dtype=t.float32, device=dev),
        }

    def decode_batch(self, llr, code_id=None, out=None, codeword: bool = False, stream=None, nframes=None):
        """Decode a device-resident batch (torch CUDA tensor, frames x stride;
        ``nframes``: fewer than the buffer holds, e.g. a padded interleaved one)."""
        t = self._torch
        assert llr.is_cuda and llr.dtype == self.llr_dtype and llr.is_contiguous()
        if nframes is None:
            nframes = llr.numel() // self.llr_stride
        assert nframes * self.llr_stride <= llr.numel()
        if out is None:
            out = self.alloc_outputs(nframes, codeword)
        ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None
        if code_id is not None:
            assert code_id.is_cuda and code_id.dtype == t.int32
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        rc = L.lib().pl_decode(self._h, ptr(llr), ptr(code_id), nframes, ptr(out["payload"]),
                               ptr(out.get("codeword")), ptr(out["crc_ok"]), ptr(out["esc"]),
                               ptr(out["metric"]), C.c_void_p(s.cuda_stream))
        if rc:
            _raise(rc, L.last_error(self._h))
        return out

    def pack_frames(self, frames, code_id=None):
        """Variable-length frames (a list of 1-D arrays, frame i of its code's
        n) -> (packed host buffer, element offsets): each frame starts 16-byte
        aligned, in order (the layout pl_decode_packed / pl_decode_host_packed
        take)."""
        return pack_frames(frames, self._torch.empty(0, dtype=self.llr_dtype).numpy().dtype)

    def pack_batch(self, llr: np.ndarray, code_id: np.ndarray):
        """A padded mixed batch (frames x pl_llr_stride, frame f valid up to
        its code's n) -> (packed buffer, offsets), vectorised per code length."""
        return pack_batch(llr, np.array([c.n for c in self.codes], np.int64)[np.asarray(code_id)])

    def decode_packed(self, llr, offsets, code_id=None, out=None, codeword: bool = False, stream=None):
        """Device-resident packed frames: llr (1-D CUDA tensor), offsets
        (int64 CUDA tensor, element offset of each frame)."""
        t = self._torch
        assert llr.is_cuda and llr.dtype == self.llr_dtype and llr.is_contiguous()
        assert offsets.is_cuda and offsets.dtype == t.int64
        nframes = offsets.numel()
        if out is None:
            out = self.alloc_outputs(nframes, codeword)
        ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None
        if code_id is not None:
            assert code_id.is_cuda and code_id.dtype == t.int32
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        rc = L.lib().pl_decode_packed(self._h, ptr(llr), ptr(offsets), ptr(code_id), nframes,
                                      ptr(out["payload"]), ptr(out.get("codeword")), ptr(out["crc_ok"]),
                                      ptr(out["esc"]), ptr(out["metric"]), C.c_void_p(s.cuda_stream))
        if rc:
            _raise(rc, L.last_error(self._h))
        return out

    def _check_host_buffers(self, llr, o, nframes, code_id=None):
        """The C side reads nframes * stride LLRs and writes nframes rows of
        each output: reject buffers of the wrong type, layout or size."""
        t = self._torch
        want_np = _NP_DTYPE[self.precision.name]
        if hasattr(llr, "data_ptr"):
            if llr.dtype != self.llr_dtype or not llr.is_contiguous() or llr.is_cuda:
                raise ValueError(f"llr must be a contiguous CPU {self.llr_dtype} tensor")
        elif not (isinstance(llr, np.ndarray) and llr.dtype == want_np and llr.flags.c_contiguous):
            raise ValueError(f"llr must be a C-contiguous {np.dtype(want_np).name} array")
        need = {"payload": nframes * self.payload_stride, "crc_ok": nframes, "esc": nframes,
                "metric": nframes}
        if o.get("codeword") is not None:
            need["codeword"] = nframes * self.codeword_stride
        for key, n in need.items():
            x = o.get(key)
            if x is None:
                continue
            nbytes = x.numel() * x.element_size() if hasattr(x, "numel") else x.nbytes
            esz = 4 if key == "metric" else 1
            contig = x.is_contiguous() if hasattr(x, "is_contiguous") else x.flags.c_contiguous
            if nbytes < n * esz or not contig:
                raise ValueError(f"output '{key}' must be contiguous with room for {nframes} frames")
        if code_id is not None:
            ok = (code_id.dtype == t.int32 and code_id.numel() >= nframes and code_id.is_contiguous()
                  if hasattr(code_id, "data_ptr") else code_id.size >= nframes)
            if not ok:
                raise ValueError("code_id must hold one int32 per frame")

    def decode_host_packed_into(self, llr, offsets, o, code_id=None):
        """Host packed frames (pl_decode_host_packed): only each frame's own
        n LLRs cross the host link."""
        def ptr(x):
            if x is None:
                return None
            if hasattr(x, "data_ptr"):
                return C.c_void_p(x.data_ptr())
            return x.ctypes.data_as(C.c_void_p)
        if not hasattr(offsets, "data_ptr"):
            offsets = np.ascontiguousarray(offsets, np.int64)
        nframes = offsets.numel() if hasattr(offsets, "numel") else offsets.size
        if code_id is not None and not hasattr(code_id, "data_ptr"):
            code_id = np.ascontiguousarray(code_id, np.int32)
        self._check_host_buffers(llr, o, nframes, code_id)
        rc = L.lib().pl_decode_host_packed(self._h, ptr(llr), ptr(offsets), ptr(code_id), nframes,
                                           ptr(o["payload"]), ptr(o.get("codeword")), ptr(o["crc_ok"]),
                                           ptr(o["esc"]), ptr(o["metric"]))
        if rc:
            _raise(rc, L.last_error(self._h))
        return o

    def decode_host(self, llr: np.ndarray, code_id: np.ndarray | None = None, codeword: bool = False):
        """Host buffers in, host buffers out (copies overlap decoding)."""
        llr = np.ascontiguousarray(llr, _NP_DTYPE[self.precision.name])
        if llr.size % self.llr_stride:
            raise ValueError(f"llr holds {llr.size} values, not a multiple of the frame stride "
                             f"{self.llr_stride}")
        nframes = llr.size // self.llr_stride
        o = {
            "payload": np.zeros((nframes, self.payload_stride), np.uint8),
            "codeword": np.zeros((nframes, self.codeword_stride), np.uint8) if codeword else None,
            "crc_ok": np.zeros(nframes, np.uint8),
            "esc": np.zeros(nframes, np.uint8),
            "metric": np.zeros(nframes, np.float32),
        }
        return self.decode_host_into(llr, o, code_id)

    def decode_host_into(self, llr, o, code_id=None):
        """Same with caller-provided (ideally pinned) host buffers; accepts
        numpy arrays or CPU torch tensors."""
        def ptr(x):
            if x is None:
                return None
            if hasattr(x, "data_ptr"):
                return C.c_void_p(x.data_ptr())
            return x.ctypes.data_as(C.c_void_p)
        size = llr.numel() if hasattr(llr, "numel") else llr.size
        if size % self.llr_stride:
            raise ValueError(f"llr holds {size} values, not a multiple of the frame stride "
                             f"{self.llr_stride}")
        nframes = size // self.llr_stride
        if code_id is not None and not hasattr(code_id, "data_ptr"):
            code_id = np.ascontiguousarray(code_id, np.int32)
        self._check_host_buffers(llr, o, nframes, code_id)
        rc = L.lib().pl_decode_host(self._h, ptr(llr), ptr(code_id), nframes, ptr(o["payload"]),
                                    ptr(o.get("codeword")), ptr(o["crc_ok"]), ptr(o["esc"]),
                                    ptr(o["metric"]))
        if rc:
            _raise(rc, L.last_error(self._h))
        return o

    def list_paths(self, alive=None, metric=None):
        """pl_list_paths: later decode_batch / decode_packed calls write each
        frame's final list — ``alive`` (CUDA int32, one mask per frame, bit s
        = slot s) and ``metric`` (CUDA float32, frames x L) — as the
        reference's ListDecoder alive/metric_of expose it; None switches it off."""
        t = self._torch
        if alive is not None:
            assert alive.is_cuda and alive.dtype == t.int32 and alive.is_contiguous()
            assert metric.is_cuda and metric.dtype == t.float32 and metric.is_contiguous()
        self._paths = (alive, metric)  # keep the buffers alive while the library holds them
        ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None  # noqa: E731
        rc = L.lib().pl_list_paths(self._h, ptr(alive), ptr(metric))
        if rc:
            _raise(rc, L.last_error(self._h))

    def set_host_chunk(self, frames: int = 0):
        """pl_set_host_chunk: frames per chunk of the host-buffer decodes
        (0 = automatic)."""
        rc = L.lib().pl_set_host_chunk(self._h, int(frames))
        if rc:
            _raise(rc, L.last_error(self._h))

    def set_llr_layout(self, interleaved32: bool):
        """pl_set_llr_layout: decode_batch then takes LLRs interleaved in
        groups of 32 frames (``interleave32``); SC / SSC with one code."""
        rc = L.lib().pl_set_llr_layout(self._h, 1 if interleaved32 else 0)
        if rc:
            _raise(rc, L.last_error(self._h))
        self._il32 = bool(interleaved32)

    def frame_latency(self, lat_ns=None):
        """pl_frame_latency: later decode_batch / decode_packed calls write
        each frame's device decode time in ns into ``lat_ns`` (a CUDA int32
        tensor, one entry per frame); None switches it off."""
        if lat_ns is not None:
            assert lat_ns.is_cuda and lat_ns.dtype == self._torch.int32 and lat_ns.is_contiguous()
        self._lat = lat_ns  # keep the buffer alive while the library holds it
        rc = L.lib().pl_frame_latency(self._h, C.c_void_p(lat_ns.data_ptr()) if lat_ns is not None else None)
        if rc:
            _raise(rc, L.last_error(self._h))

    def last_launches(self) -> int:
        return int(L.lib().pl_last_launches(self._h))

    def profile(self, enable: bool = True):
        """Bracket every kernel launch with CUDA events (pl_profile)."""
        L.lib().pl_profile(self._h, int(enable))

    def last_kernel_ms(self):
        """[(kind 'sc'|'list', l, ms)] for each launch of the last decode."""
        ms = (C.c_float * 64)()
        kd = (C.c_int32 * 64)()
        ll = (C.c_int32 * 64)()
        n = L.lib().pl_last_kernel_ms(self._h, ms, kd, ll, 64)
        if n < 0:
            raise DeviceError("kernel timing failed")
        return [("list" if kd[i] else "sc", int(ll[i]), float(ms[i])) for i in range(n)]

    def decode(self, llr) -> DecodeResult:
        """One frame (reference-shaped convenience; batch for throughput)."""
        t = self._torch
        arr = np.ascontiguousarray(llr).reshape(1, -1)
        x = t.zeros((1, self.llr_stride), dtype=self.llr_dtype)
        x[:, :arr.shape[1]] = t.from_numpy(arr)
        o = self.decode_batch(x.cuda(self.device), codeword=True)
        t.cuda.synchronize(self.device)
        code = self.codes[0]
        return DecodeResult(
            codeword=unpack_msb(o["codeword"].cpu().numpy()[0], code.n),
            payload=unpack_msb(o["payload"].cpu().numpy()[0], code.payload_size),
            crc_ok=bool(o["crc_ok"].item()),
            escalation_level=int(o["esc"].item()),
            metric=float(o["metric"].item()),
        )
