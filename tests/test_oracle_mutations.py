"""Mutation harness for the oracle's pins (CPU).

Each mutation is a plausible slip in oracle/nndtw_oracle.c -- a wrong band index, a window
off by one, a dropped DP predecessor, a wrong n_bands rounding, a different Kim rule, a
bridge overlapping the bands, a lost tie rule, ...  The mutant is compiled with the oracle's
own flags and the pin suite (tests/test_oracle_pins.py) is run against it in a scratch copy of
the tests and the oracle package; every mutant must fail at least one pin.  This is what makes the
pins evidence about the oracle rather than about themselves."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "nndtw_oracle.c")
PY = os.path.join(ROOT, "oracle", "__init__.py")

# (name, original text, mutated text) -- each original must occur exactly once
MUTATIONS = [
    ("alg1_line8_band_index", "minL = min2(minL, delta(Ax(j), Bx(i)));",
     "minL = min2(minL, delta(Ax(j), Bx(j)));"),
    ("alg1_line9_right_band_mirror", "delta(Ax(L - i + 1), Bx(L - j + 1)));",
     "delta(Ax(L - i + 1), Bx(L - j)));"),
    ("alg1_band_window_start", "int j0 = i - W > 1 ? i - W : 1;",
     "int j0 = i - W + 1 > 1 ? i - W + 1 : 1;"),
    ("n_bands_rounding", "/* line 2 */\n    int n_bands = L / 2 < V ? L / 2 : V;",
     "/* line 2 */\n    int n_bands = (L + 1) / 2 < V ? (L + 1) / 2 : V;"),
    ("bridge_overlaps_bands", "for (int i = n_bands + 1; i <= L - n_bands; ++i) {\n        if (Ax(i)",
     "for (int i = n_bands; i <= L - n_bands + 1; ++i) {\n        if (Ax(i)"),
    ("envelope_window_short", "        int hi = i + w > L ? L : i + w;\n        float u",
     "        int hi = i + w - 1 > L ? L : i + w - 1;\n        float u"),
    ("dtw_dropped_predecessor", "double m = min2(min2(prev[j - 1], cur[j - 1]), prev[j]);",
     "double m = min2(prev[j - 1], prev[j]);"),
    ("dtw_window_off_by_one", "int jhi = i + w > L ? L : i + w;",
     "int jhi = i + w - 1 > L ? L : i + w - 1;"),
    ("delta_not_squared", "    double d = a - b;\n    return d * d;",
     "    double d = a - b;\n    return d < 0 ? -d : d;"),
    ("kim_rule_and", "if (usedA[u] == ia[f] || usedB[u] == ib[f]) clash = 1;",
     "if (usedA[u] == ia[f] && usedB[u] == ib[f]) clash = 1;"),
    ("nn_tie_rule_lost", "if (d < D || (d == D && n < nn) || nn < 0) { D = d; nn = n; }",
     "if (d <= D || nn < 0) { D = d; nn = n; }"),
    ("keogh_upper_side_dropped", "if (a > (double)U[i - 1]) res = res + delta(a, (double)U[i - 1]);",
     "if (a > (double)U[i - 1]) res = res + 0.0;"),
    ("lb_improved_no_projection", "        else Ap[i] = A[i];\n    }\n    oracle_envelope(Ap, L, W, Ua, La);\n    double res",
     "        else Ap[i] = A[i];\n        Ap[i] = A[i];\n    }\n    oracle_envelope(Ap, L, W, Ua, La);\n    double res"),
    ("lb_new_window_short", "        int hi = i + W > L ? L : i + W;\n        double m",
     "        int hi = i + W - 1 > L ? L : i + W - 1;\n        double m"),
    ("enh_improved_columns_into_bands",
     "res = res + oracle_lb_keogh_range(B, Ua, La, n_bands + 1, L - n_bands);",
     "res = res + oracle_lb_keogh_range(B, Ua, La, n_bands, L - n_bands + 1);"),
    ("enh_improved_no_projection", "        else Ap[i] = A[i];\n    }\n    oracle_envelope(Ap, L, W, Ua, La);\n    res = res + oracle_lb_keogh_range",
     "        else Ap[i] = A[i];\n        Ap[i] = A[i];\n    }\n    oracle_envelope(Ap, L, W, Ua, La);\n    res = res + oracle_lb_keogh_range"),
]
# mutations of the Python side of the oracle (oracle/__init__.py)
PY_MUTATIONS = [
    ("tightness_no_sqrt", "np.mean(np.sqrt(lb[m]) / np.sqrt(d[m]))", "np.mean(lb[m] / d[m])"),
    ("tightness_counts_zero_dtw", "    m = d > 0\n", "    m = d >= 0\n"),
]


def test_mutations_apply_once():
    src, py = open(SRC).read(), open(PY).read()
    for name, old, new in MUTATIONS:
        assert src.count(old) == 1, name
    for name, old, new in PY_MUTATIONS:
        assert py.count(old) == 1, name


def _run_pins_on_mutant(tmp_path, c_src, py_src):
    """The pin suite against a scratch copy: tests/ (pins, conftest, golden), datagen.py and
    an oracle/ package holding the mutated sources (built there by oracle.build())."""
    (tmp_path / "tests").mkdir()
    for f in ("conftest.py", "test_oracle_pins.py"):
        shutil.copy(os.path.join(ROOT, "tests", f), tmp_path / "tests" / f)
    shutil.copytree(os.path.join(ROOT, "tests", "golden"), tmp_path / "tests" / "golden",
                    ignore=shutil.ignore_patterns(".partial", "cfg*.npz"))
    shutil.copy(os.path.join(ROOT, "datagen.py"), tmp_path / "datagen.py")
    (tmp_path / "oracle").mkdir()
    (tmp_path / "oracle" / "nndtw_oracle.c").write_text(c_src)
    (tmp_path / "oracle" / "__init__.py").write_text(py_src)
    return subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x",
                           "-q", "-p", "no:cacheprovider"], cwd=tmp_path, capture_output=True,
                          text=True, timeout=600)


def test_unmutated_copy_passes(tmp_path):
    """Control: the harness's scratch copy of the real oracle passes every pin."""
    r = _run_pins_on_mutant(tmp_path, open(SRC).read(), open(PY).read())
    assert r.returncode == 0, r.stdout[-2000:]


@pytest.mark.parametrize("name,old,new", MUTATIONS + PY_MUTATIONS,
                         ids=[m[0] for m in MUTATIONS + PY_MUTATIONS])
def test_mutant_fails_a_pin(tmp_path, name, old, new):
    c_src, py_src = open(SRC).read(), open(PY).read()
    if (name, old, new) in MUTATIONS:
        c_src = c_src.replace(old, new)
    else:
        py_src = py_src.replace(old, new)
    r = _run_pins_on_mutant(tmp_path, c_src, py_src)
    assert r.returncode != 0, f"mutant {name} passed every pin:\n{r.stdout[-2000:]}"
    assert " failed" in r.stdout, r.stdout[-2000:]
