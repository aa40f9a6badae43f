"""B200-native batched polar decoder (SC / SSC / SCL / CA-SCL / PA / FA-SCL).

A drop-in for the reference's decoder path (FrameDecoder<R>::decode,
/root/reference/proj/include/polar/decoders.hpp:60-85) built as hand-written
sm_100a kernels behind a C ABI (include/polar_b200.h).  ``polar`` mirrors
the reference's C++ interface in Python over that ABI.
"""
from .polar import (  # noqa: F401
    ConfigError,
    CrcSpec,
    DecodeResult,
    DecoderKind,
    DeviceError,
    FrameDecoder,
    IoError,
    ParseError,
    PolarCode,
    Precision,
    PruningConfig,
    channel,
    channel_device,
    channel_frames,
    construct_frozen,
    construct_frozen_ga,
    crc_compute,
    interleave32,
    load_frozen_file,
    load_puncture_file,
    make_code,
    prune_tree,
    save_frozen_file,
    unpack_msb,
)
