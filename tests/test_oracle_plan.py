"""Pins for the oracle's planner: Eq. alpha, BPS, #GEMM,
no-overflow budget.  Values come from the paper's text (tests/golden/
paper_constants.txt) and SPEC worked examples, plus closed-form checks."""
import math

import oracle as O
from conftest import golden


def _const(key):
    for k, v, *_ in golden("paper_constants.txt"):
        if k == key:
            return v
    raise KeyError(key)


def test_alpha_paper_example_fp32():
    # FP32 accumulation (l_acc = 24), k = 4096 -> alpha = 6.
    assert O.alpha(24, 4096) == int(_const("alpha_fp32_k4096"))


def test_alpha_fp16_limits():
    # FP16 arithmetic (u = 2^-11): alpha > 0 requires k <= 2^9;
    # FP32-internal Tensor Cores (u = 2^-24): up to k = 2^22.
    kmax16 = int(_const("fp16_kmax_plain"))
    assert O.alpha(11, kmax16) >= 1 and O.alpha(11, 2 * kmax16) <= 0
    kmax32 = int(_const("fp16tc_kmax"))
    assert O.alpha(24, kmax32) >= 1 and O.alpha(24, 2 * kmax32) <= 0


def test_bps_int8_table2():
    l_in, l_acc = int(_const("int8_l_in")), int(_const("int8_l_acc"))
    assert (l_in, l_acc) == (7, 31)
    # (l_acc = 31, k = 2^12) -> alpha = 9, BPS = 7.
    assert O.alpha(31, 4096) == 9 and O.bps(7, 31, 4096) == 7
    # BPS = l_in for (power-of-two) k < 2^18, i.e. up to 2^17; then alpha binds.
    kb = int(_const("int8_bps_equals_lin_k"))
    for e in range(0, 18):
        assert O.slice_width(2 ** e) == 7
    assert O.slice_width(kb) == 7
    assert O.slice_width(2 * kb) == 6
    assert O.slice_width(2 ** 19) == 6
    assert O.slice_width(2 ** 20) == 5 and O.slice_width(2 ** 21) == 5


def test_alpha_integer_form_equivalence():
    # floor((l - log2 k)/2) == floor((l - ceil(log2 k))/2) for all k.
    for k in list(range(1, 5000)) + [2 ** e + d for e in range(12, 22) for d in (-1, 0, 1)]:
        c = math.ceil(math.log2(k)) if k > 1 else 0
        # exact integer ceil(log2 k):
        c = (k - 1).bit_length()
        assert O.alpha(31, k) == (31 - c) // 2, k


def test_gemm_count():
    assert O.gemm_count(9) == int(_const("gemm_count_s9"))
    for s in range(1, 20):
        assert O.gemm_count(s) == sum(1 for i in range(1, s + 1) for j in range(1, s + 1)
                                      if i + j <= s + 1)
    assert O.gemm_count(13) == 91 and O.gemm_count(1) == 1


def test_budget_holds_for_formula_w():
    # The formula's w always satisfies k (2^w - 1)^2 <= 2^31 - 1.
    for e in range(0, 22):
        for k in (2 ** e, 2 ** e + 1, max(1, 2 ** e - 1)):
            w = O.slice_width(k)
            assert w >= 1
            assert k * (2 ** w - 1) ** 2 <= 2 ** 31 - 1
            assert O.budget_ok(w, k)
    # SPEC S:342-343 (with the corrected product).
    assert 2 ** 17 * 127 ** 2 == 2114060288 and O.budget_ok(7, 2 ** 17)
    assert not O.budget_ok(7, 2 ** 18)
    # The exact INT32 limit for w = 7 is k = 133144.
    assert O.budget_ok(7, 133144) and not O.budget_ok(7, 133145)
