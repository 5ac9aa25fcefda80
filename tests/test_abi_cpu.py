"""CPU-side checks of the boundary: libnndtw.so builds for sm_100a, loads, and exports every
symbol include/nndtw.h declares; the binding rejects bad arguments before any compute.
No compute calls are made here (no GPU in this container)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nndtw.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"NNDTW_API\s+[\w\s\*]*?\b(nndtw_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1808_09617_b200 import build, nndtw
    build.build()
    return nndtw.load()


def test_header_declares_the_five_calls():
    syms = header_symbols()
    for s in ("nndtw_envelopes", "nndtw_lb_enhanced", "nndtw_dtw_batch", "nndtw_classify",
              "nndtw_loocv_window"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_1808_09617_b200 import nndtw
    out = subprocess.check_output(["nm", "-D", "--defined-only", nndtw.LIB_PATH], text=True)
    exported = set(re.findall(r" T (nndtw_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    # the binding declares a signature for every symbol of the header and nothing else
    assert sorted(nndtw.EXPORTED) == header_symbols()
    for s in header_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a(lib):
    from paper_1808_09617_b200 import nndtw
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                                   nndtw.LIB_PATH], text=True)
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_host_only_calls(lib):
    assert lib.nndtw_version() == 1
    assert lib.nndtw_launch_count() >= 0
    ws = lib.nndtw_classify_workspace_bytes(100, 1000, 128, 13)
    # LB matrix + worst-case item list dominate: 100*1000*(4+8) bytes
    assert ws >= 100 * 1000 * 12
    assert lib.nndtw_loocv_workspace_bytes(300, 64, 0, 300) > 300 * 64 * 8


def test_binding_rejects_bad_tensors():
    import torch
    from paper_1808_09617_b200 import nndtw
    with pytest.raises(nndtw.NNDTWError):
        nndtw._series(torch.zeros(4, 8), "x")  # CPU tensor: no fallback path exists


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1808_09617_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "nndtw_oracle" not in txt, f
