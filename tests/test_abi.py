"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/gls.h declares, and its host-built 4-value LUT (the table the kernel
stages in shared memory) agrees with the oracle's gate functions."""
import itertools
import os
import re

import pytest

from oracle import oracle
from paper_2304_13398_b200 import gls
from paper_2304_13398_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "gls.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gls_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = gls.load_library()
    names = header_functions()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(gls.EXPORTS)


def test_version():
    assert "sm_100a" in gls.gls_version()


@pytest.mark.parametrize("t", range(9))
def test_lut_matches_oracle_gate_functions(t):
    ks = [1] if t in (W.BUF, W.NOT) else ([3] if t == W.MUX2 else [2, 3, 4])
    for k in ks:
        for v in itertools.product(range(4), repeat=k):
            assert gls.gls_lut_lookup(t, k, list(v)) == oracle.eval_gate(t, list(v)), (t, v)


def test_lut_rejects_bad_arity():
    assert gls.gls_lut_lookup(W.AND, 1, [0]) == gls.GLS_EINVAL
    assert gls.gls_lut_lookup(W.MUX2, 2, [0, 1]) == gls.GLS_EINVAL
    assert gls.gls_lut_lookup(99, 2, [0, 1]) == gls.GLS_EINVAL


def test_no_cpu_fallback_without_gpu():
    """Without a GPU the library must fail loudly, never compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gls.GlsError):
        gls.Context(0)
