"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol include/rrq.h
declares; the oracle library exports its entry points; no CPU fallback exists."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rrq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rrq_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    import paper_2411_08342_b200 as pkg
    lib = pkg.load_library()
    names = _declared()
    assert "rrq_build_correction" in names and len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_no_cpu_fallback_without_device():
    import torch
    import paper_2411_08342_b200 as pkg
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(pkg.RRQError):
        pkg.RRQ(4)


def test_product_does_not_touch_oracle():
    """The product path never imports, links or executes anything under oracle/."""
    pkgdir = os.path.join(ROOT, "paper_2411_08342_b200")
    pat = re.compile(r"(import\s+oracle|from\s+oracle|liboracle|rrq_oracle|orc_)")
    for dp, _, fs in os.walk(pkgdir):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                assert not pat.search(open(os.path.join(dp, f)).read()), f


def test_flop_model_matches_survey():
    from paper_2411_08342_b200.flops import pair_flops, translation_terms
    assert translation_terms(8, 2) == 489 and translation_terms(8, 1) == 574
    assert pair_flops(8)["total"] == 302368


@pytest.mark.parametrize("p", [4, 6, 8, 10, 12, 14])
def test_translate_schedule_selftest(p):
    """Host logic: the packed k_translate schedule (lane pieces, window ring, prime codes, field widths -- 8-bit S'
    positions from p = 12 on) decodes to exactly the terms of the direct translation for every output (l, m)."""
    import ctypes
    import paper_2411_08342_b200 as pkg
    lib = pkg.load_library()
    lib.rrq_selftest_translate_schedule.argtypes = [ctypes.c_int]
    lib.rrq_selftest_translate_schedule.restype = ctypes.c_int
    assert lib.rrq_selftest_translate_schedule(p) == 0
    assert lib.rrq_selftest_translate_schedule(5) == -1
