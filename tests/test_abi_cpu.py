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
    assert lib.nndtw_version() == 2
    assert lib.nndtw_launch_count() >= 0
    ws = lib.nndtw_classify_workspace_bytes(100, 1000, 128, 13)
    # LB matrix + worst-case item list dominate: 100*1000*(4+8) bytes
    assert ws >= 100 * 1000 * 12
    assert lib.nndtw_loocv_workspace_bytes(300, 64, 0, 300) > 300 * 64 * 8


def test_capped_workspace_sizes(lib):
    """nndtw_classify_workspace_bytes_capped: 20 bytes per reserved pair on top of the bound
    matrix and the fixed part, never more than the full layout, at least the seed rounds."""
    import ctypes as C
    f = lib.nndtw_classify_workspace_bytes_capped
    f.restype = C.c_size_t
    f.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64]
    full = lib.nndtw_classify_workspace_bytes(10000, 100000, 512, 103)
    a = f(10000, 100000, 512, 103, 10 ** 8)
    b = f(10000, 100000, 512, 103, 2 * 10 ** 8)
    assert a < b < full
    assert abs((b - a) - 20 * 10 ** 8) <= 4 * 256
    assert f(10000, 100000, 512, 103, 10 ** 12) == full      # capacity >= every pair: full
    assert f(10000, 100000, 512, 103, -1) == full
    assert f(10000, 100000, 512, 103, 0) == f(10000, 100000, 512, 103, 2 * 10000 + 2)
    # config 2 at the default 1/8: about a quarter of the full layout's 24 bytes per pair
    c = f(10000, 100000, 512, 103, 10 ** 9 // 8 + 1)
    assert c < 0.3 * full


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


def test_stats_struct_matches_header(tmp_path):
    """The ctypes Stats mirror of nndtw_stats has the header's field order, offsets and size
    (compiled against include/nndtw.h with gcc)."""
    import ctypes as C
    from paper_1808_09617_b200 import nndtw
    names = [f for f, _ in nndtw.Stats._fields_]
    for f in ("pruned_kim", "pruned_bands", "pruned_keogh", "ms_envelopes"):
        assert f in names
    src = tmp_path / "s.c"
    body = "".join(f'printf("{f} %zu\\n", offsetof(nndtw_stats, {f}));' for f in names)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "nndtw.h"\n'
                   'int main(void){' + body +
                   'printf("size %zu\\n", sizeof(nndtw_stats)); return 0;}\n')
    exe = tmp_path / "s"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).split("\n")
               if line)
    for f in names:
        assert int(out[f]) == getattr(nndtw.Stats, f).offset, f
    assert int(out["size"]) == C.sizeof(nndtw.Stats)


def test_dtw_kernel_name_rule(lib):
    """nndtw_dtw_kernel_name (host-only) names the S4 kernel dispatch_dtw picks: w = 0 is the
    squared-ED kernel, narrow bands the wavefront kernel, config 4's full window the strips."""
    name = lambda L, w: lib.nndtw_dtw_kernel_name(L, w).decode()  # noqa: E731
    assert name(300, 0) == "k_dtw_w0"
    assert name(512, 103) == "k_dtw_band"
    assert name(256, 26) == "k_dtw_band"
    assert name(2048, 2047) == "k_dtw_strip"
    assert name(2048, 5000) == "k_dtw_strip"      # clamped to L-1
    assert name(1024, 511) == "k_dtw_band"        # R = 32 is the only band layout (2w+2 = 1024)
    assert name(1, 0) == "" and name(16, -1) == ""


def test_band_limited_window_rule(lib, monkeypatch):
    """nndtw_band_limited_window (host-only): the band of the S4 band-limited pass -- the
    R = 26 full-warp layout's wb = 13 G - 1 <= w / 2 for band-kernel windows w >= 64, <= w / 8
    in front of the row-strip kernel where that is >= 103, else -1."""
    wb = lib.nndtw_band_limited_window
    monkeypatch.delenv("NNDTW_ADAPT", raising=False)
    monkeypatch.delenv("NNDTW_ADAPT_FULL", raising=False)
    assert wb(512, 103) == 51          # config 2
    assert wb(256, 128) == 51          # config 1, p = 50
    assert wb(300, 210) == 103
    assert wb(256, 52) == -1           # w < 64
    # full windows (the row-strip kernel): a band of <= w / 8 offsets, where that is >= 103
    assert wb(256, 255) == -1          # config 1, p = 100: 25 would be too narrow
    assert wb(2048, 2047) == 207       # config 4
    assert wb(1024, 1023) == 103
    monkeypatch.setenv("NNDTW_ADAPT_FULL", "0")
    assert wb(2048, 2047) == -1 and wb(512, 103) == 51
    monkeypatch.setenv("NNDTW_ADAPT_FULL", "1")
    assert wb(256, 255) == 25
    monkeypatch.delenv("NNDTW_ADAPT_FULL")
    assert wb(510, 103) == -1          # L % 4 != 0 (the layout's 16-byte rows)
    assert wb(512, 0) == -1 and wb(1, 5) == -1 and wb(16, -1) == -1
    for w in range(64, 400, 7):
        b = wb(1024, w)
        assert b in (-1, 12, 25, 51, 103, 207) and (b == -1 or 2 * b <= w), (w, b)
    monkeypatch.setenv("NNDTW_ADAPT", "0")
    assert wb(512, 103) == -1
    monkeypatch.setenv("NNDTW_ADAPT", "25")
    assert wb(512, 103) == 25
