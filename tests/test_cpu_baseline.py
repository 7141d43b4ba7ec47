"""The timed CPU baseline (oracle/hp_cpu_baseline.c, fp32 accumulate) computes
the same layer forward as the exact fp64 oracle (hp_oracle.c), and the CPU
arm of bench.py (oracle/cpu_baseline.py) never imports the product package."""
import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from tests.util import to_bf16_bits

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("bits,scheme", [(3, 1), (4, 0), (8, 1), (16, 1)])
@pytest.mark.parametrize("m", [1, 8, 33])
def test_fp32_baseline_matches_fp64_oracle(bits, scheme, m):
    import oracle
    from oracle import cpu_baseline as cb
    cb._bind()
    rng = np.random.default_rng(bits * 10 + m)
    n, k = 72, 650  # ragged groups and row blocks
    wb = to_bf16_bits(rng.normal(0, 0.02, (n, k)))
    xb = to_bf16_bits(rng.normal(0.05, 1.0, (m, k)))
    port = oracle.port()
    if bits == 16:
        codes, st, z = wb, None, None
        ref = port.qlinear(xb, wb, None, None, 16, scheme)
    else:
        codes, st, z = port.quantize_matrix(wb, bits, scheme)
        ref = port.qlinear(xb, codes, st, z, bits, scheme)
    y = np.empty((m, n), dtype=np.float32)
    st32 = np.ascontiguousarray(st, dtype=np.float32) if st is not None else None
    z32 = np.ascontiguousarray(z, dtype=np.float32) if (z is not None and scheme == 0) else None
    rc = port.lib.hpo_cpu_qlinear_f32(xb.ctypes.data, m, k, np.ascontiguousarray(codes).ctypes.data,
                                      st32.ctypes.data if st32 is not None else None,
                                      z32.ctypes.data if z32 is not None else None, n, bits,
                                      scheme, y.ctypes.data, 0)
    assert rc == 0
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


def test_cpu_arm_does_not_import_the_product():
    code = ("import sys; sys.path.insert(0, %r); from oracle import cpu_baseline as cb; "
            "p, m = cb.load_plan('opt125m_b8_1gpu'); cb._bind(); "
            "assert not any(k.startswith('paper_2403_01136_b200') for k in sys.modules), "
            "[k for k in sys.modules if 'paper' in k]" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
