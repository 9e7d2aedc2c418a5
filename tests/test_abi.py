"""The C-ABI library (include/skb.h) builds for sm_100a, loads without a GPU,
and exports every declared entry point; the product fails loudly (no CPU
fallback) when no CUDA device is visible."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "skb.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_entry_points():
    names = declared_functions()
    for must in ("skb_rnn_forward", "skb_rnn_pack", "skb_rnn_plan", "skb_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1810_08061_b200 import build, runtime
    build.build()
    lib = runtime.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in runtime.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.skb_version().decode().startswith("skb ")


def test_library_contains_tcgen05_code():
    """SASS of libskb.so holds UTCHMMA (tcgen05.mma), LDTM (tcgen05.ld) and
    UBLKCP (bulk async copies): the kernels are sm_100a-native."""
    import shutil
    import subprocess
    from paper_1810_08061_b200 import build
    lib = build.build()
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "UBLKCP", "STTM"):
        assert mnemonic in sass, mnemonic


def test_execute_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from oracle import fixtures
    from paper_1810_08061_b200 import BackendUnavailable, execute, ir
    doc = fixtures.load_golden("lstm_4x8x8")
    g = ir.from_json(doc["graph"])
    with pytest.raises(BackendUnavailable):
        execute(g, fixtures.make_feeds(doc["case"]))
