"""Device-level kernel checks (the test_kernels.cpp analogue on the GPU)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def test_packed_int8_f_g_exhaustive(native, gpu):
    """Packed int8 f/g == scalar f/g (llr.hpp:55-69) for every operand pair,
    byte position and partial-sum pattern, including saturation at +-127."""
    out = C.c_uint64(99)
    rc = native.pl_kernel_selftest(0, C.byref(out))
    assert rc == 0
    assert out.value == 0
