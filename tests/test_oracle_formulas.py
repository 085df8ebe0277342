"""Pins for the oracle's per-request arithmetic (A1 strategy, A2 score, ingest).

Each test checks the oracle against something other than itself: a value the
paper (or SPEC, derived from it) prints, a closed form, a special case that
reduces to a textbook formula, an invariant, or brute force.
"Oracle pins" for the map from oracle function to pin.
"""
import math
import random
from decimal import ROUND_HALF_UP, Decimal
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from gen.configs import KV_BYTES_PER_TOKEN, PROFILES


def mkcfg(**over):
    d = dict(capacity=16, block_tokens=16, tau=1, A1=0, A2=0, S0=0, S1=0, SH=0, c_other=0,
             ticks_per_second=1e6, starvation_threshold=100, max_batch=16,
             kv_capacity_blocks=1 << 40, score_bits=40, id_bits=23)
    d.update(over)
    return O.make_cfg(d)


# ------------------------------------------------------------------ ingest
def test_quantize_paper_pins(golden):
    for row in golden["spec_examples"]["quantize"]:
        rc, t = O.quantize(row["seconds"], 1e6)
        assert rc == O.OK and t == row["expect"], row


def _ref_round(x: float) -> int:
    # exact decimal expansion of the double, then round half away from zero
    return int(Decimal(x).quantize(Decimal(1), rounding=ROUND_HALF_UP))


def test_quantize_brute_force_half_cases():
    rng = random.Random(1)
    vals = []
    for _ in range(20000):
        s = rng.uniform(0, 100.0)
        vals.append(s)
        k = rng.randrange(0, 10 ** 7)
        h = (k + 0.5) / 1e6           # lands next to an x.5 tick boundary
        vals += [h, math.nextafter(h, 0), math.nextafter(h, 1e9)]
    for s in vals:
        rc, t = O.quantize(s, 1e6)
        x = s * 1e6
        assert rc == O.OK and t == _ref_round(x), (s, t)
    # exact halves round away from zero
    for s, e in ((0.5, 1), (1.5, 2), (2.5, 3), (np.nextafter(2.5, 0), 2)):
        assert O.quantize(float(s), 1.0) == (O.OK, e)


def test_quantize_rejects():
    for s in (float("nan"), float("inf"), -1.0, -1e-300, 4294.9673, 1e30):
        assert O.quantize(s, 1e6)[0] == O.EINVAL, s
    assert O.quantize(4294.967295, 1e6) == (O.OK, 4294967295)
    assert O.quantize(1.0, float("nan"))[0] == O.EINVAL
    assert O.quantize(1.0, 0.0)[0] == O.EINVAL


def test_blk_brute_force():
    for B in (1, 2, 16, 64):
        for n in range(0, 300):
            k = 0
            while k * B < n:
                k += 1
            assert O.blk(n, B) == k


def test_kv_bytes_formula_matches_paper():
    # "GPT-3 175B ... around 2.3 GB ... for a sequence length of 512 tokens"
    gb = KV_BYTES_PER_TOKEN["gpt3"] * 512 / 1e9
    assert abs(gb - 2.3) < 0.15


# ------------------------------------------------------------------ Eq. (1)
def test_waste_preserve_spec_examples(golden):
    c = mkcfg()
    for row in golden["spec_examples"]["waste_preserve"]:
        if "api_seconds" in row:
            rc, ticks = O.quantize(row["api_seconds"], row["ticks_per_second"])
            assert rc == O.OK
            W = O.wastes(c, row["ctx"], row["pre_rem"], ticks)
            assert W[0] == row["expect"] and 2 * W[0] == row["expect_times_m2"]
        else:
            assert O.wastes(c, row["ctx"], row["pre_rem"], row["api_ticks"])[0] == row["expect"], row


def test_waste_preserve_linear():
    # waste_preserve is linear in each argument
    c = mkcfg()
    rng = random.Random(2)
    for _ in range(500):
        a, ctx, pre, k = rng.randrange(10 ** 6), rng.randrange(10 ** 4), rng.randrange(500), rng.randrange(1, 50)
        assert O.wastes(c, ctx, pre, k * a)[0] == k * O.wastes(c, ctx, pre, a)[0]


# ------------------------------------------------------------------ Eq. (2)
def test_waste_discard_spec_examples(golden):
    for row in golden["spec_examples"]["waste_discard"]:
        if row.get("property") == "c_squared":
            c = mkcfg(A1=1 << 16, SH=16)
            for x in range(0, 301):
                assert O.wastes(c, x, 0, 0)[1] == x * x
        else:
            c = mkcfg(A1=row["A1"], A2=row["A2"], SH=row["SH"], c_other=row["c_other"])
            assert O.wastes(c, row["c_i"], 0, 0)[1] == row["expect"]


def test_waste_discard_other_requests_term():
    # Eq. (2): the recompute delays the other requests' C_other tokens too
    c = mkcfg(A1=1 << 16, SH=16, c_other=300)
    for x in (1, 7, 100):
        assert O.wastes(c, x, 0, 0)[1] == x * x + x * 300


def test_t_fwd_appendix_prefill(golden):
    row = golden["spec_examples"]["t_fwd"][0]
    SH = row["SH"]
    A2 = round(row["k1"] * row["d"] * 2 ** SH)
    c = mkcfg(A2=A2, SH=SH)
    got = O.t_fwd(c, row["c"])
    assert abs(got - row["expect_real"]) < 1.0 and got == math.floor(row["expect_real"])


def test_t_fwd_counts_attention_pairs():
    # prefill self-attention is O(n^2 d): with A2 = 2^SH, T_fwd(n)
    # equals the number of (query, key) pairs of an n-token prompt without a
    # causal mask, counted by brute force.
    c = mkcfg(A2=1 << 16, SH=16)
    for n in range(0, 60):
        pairs = sum(1 for q in range(n) for k in range(n))
        assert O.t_fwd(c, n) == pairs


def test_t_fwd_shift_floor_brute_force():
    rng = random.Random(3)
    for _ in range(2000):
        A1, A2, SH = rng.randrange(1 << 30), rng.randrange(1 << 20), rng.randrange(0, 40)
        cval = rng.randrange(1 << 25)
        c = mkcfg(A1=A1, A2=A2, SH=SH)
        exact = Fraction(A1 * cval + A2 * cval * cval, 2 ** SH)
        assert O.t_fwd(c, cval) == min(math.floor(exact), 2 ** 64 - 1)


# ------------------------------------------------------------------ Eq. (3)
def test_waste_swap_spec_examples(golden):
    r1, r2 = golden["spec_examples"]["waste_swap"]
    c = mkcfg(S0=r1["S0"], S1=r1["S1"], SH=r1["SH"], c_other=r1["c_other"])
    W = O.wastes(c, r1["c_i"], 0, 0)
    assert W[2] == r1["expect_units"] * r1["ticks_per_unit"]
    c = mkcfg(S0=r2["S0"], S1=r2["S1"], SH=r2["SH"], c_other=r2["c_other"])
    assert O.wastes(c, 0, 0, 0)[2] == 0 and O.t_swap(c, 0) == 0
    assert O.t_swap(c, 1) == (12345 + 65536) >> 16


def test_wastes_saturate():
    c = mkcfg(A1=(1 << 48) - 1, A2=(1 << 48) - 1, S0=(1 << 48) - 1, S1=(1 << 48) - 1,
              c_other=(1 << 32) - 1)
    W = O.wastes(c, (1 << 32) - 1, (1 << 32) - 1, (1 << 32) - 1)
    assert W == [2 ** 64 - 1] * 3
    W = O.wastes(c, 1000, 0, 12345)
    assert W[0] == 12345000 and W[1] == W[2] == 2 ** 64 - 1


# ------------------------------------------------------------------ argmin
def test_argmin_brute_force_with_ties():
    rng = random.Random(4)
    for _ in range(10000):
        pool = [rng.randrange(5) for _ in range(2)] + [rng.randrange(1 << 62)]
        W = [rng.choice(pool) for _ in range(3)]
        best = min(range(3), key=lambda k: (W[k], k))
        assert O.argmin3(W) == best


def test_chosen_strategy_is_minimal_waste():
    c = O.make_cfg(dict(capacity=16, **{k: v for k, v in PROFILES["gptj"].items()},
                        starvation_threshold=100, max_batch=16, kv_capacity_blocks=1 << 40,
                        score_bits=40, id_bits=23))
    rng = random.Random(5)
    for _ in range(3000):
        W = O.wastes(c, rng.randrange(4096), rng.randrange(600), rng.randrange(1 << 27))
        s = O.argmin3(W)
        assert all(W[s] <= W[k] for k in range(3))


def _gptj():
    return O.make_cfg(dict(capacity=16, **PROFILES["gptj"], starvation_threshold=100,
                           max_batch=16, kv_capacity_blocks=1 << 40, score_bits=40, id_bits=23))


def test_rule_of_thumb_discard_then_swap():
    # for a long API, "If the pre-API portion ... is ... short, Discard
    # is beneficial. Otherwise, Swap".  Sweep C_i at a 28.6 s Chatbot API.
    c = _gptj()
    labels = [O.argmin3(O.wastes(c, x, 0, 28_600_000)) for x in range(1, 4000)]
    assert labels[0] == O.D and labels[-1] == O.S
    first_s = labels.index(O.S)
    assert all(l == O.D for l in labels[:first_s]) and all(l == O.S for l in labels[first_s:])


def test_rule_of_thumb_preserve_for_short_api():
    # "For brief API calls, the Preserve strategy may be advantageous";
    # Table 2 Math API (9e-5 s) -> Preserve at any context; W_P grows linearly in T_INT
    c = _gptj()
    for x in (16, 256, 2048):
        assert O.argmin3(O.wastes(c, x, 0, 90)) == O.P
        labels = [O.argmin3(O.wastes(c, x, 0, t)) for t in range(0, 100_000_000, 250_000)]
        k = next(i for i, l in enumerate(labels) if l != O.P)
        assert all(l == O.P for l in labels[:k]) and all(l != O.P for l in labels[k:])


# ------------------------------------------------------------------ Table 1
@pytest.mark.parametrize("fx", ["a", "b"])
def test_table1_labels_and_scores(golden, fx):
    t1 = golden["table1"]
    f = t1["fixtures"][fx]
    cm = t1["common"]
    c = mkcfg(block_tokens=cm["block_tokens"], tau=f["tau"], A1=cm["A1"], A2=f["A2"],
              S0=cm["S0"], S1=f["S1"], SH=cm["SH"], c_other=cm["c_other"])
    for name, rq in t1["requests"].items():
        api_ticks = rq["api_iters"] * f["tau"]
        W = O.wastes(c, 0, rq["api_after"], api_ticks)
        exp = f["expect"][name]
        assert W == exp["W"], (name, W)
        lab = O.argmin3(W)
        assert "PDS"[lab] == rq["label"]
        sc = O.score(c, ctx=0, pre_rem=rq["api_after"], api_ticks=api_ticks,
                     resp_len=cm["resp_len"], post_len=rq["post"], strategy=lab)
        assert sc == exp["score"], (name, sc)


def test_table1_literal_integral_order_contradicts_narrative(golden):
    # Reading R16: the paper's narrative order R3 < R2 < R1 is
    # not what the literal integral gives; the oracle follows the definition.
    for f in golden["table1"]["fixtures"].values():
        s = {k: v["score"] for k, v in f["expect"].items()}
        assert s["R2"] < s["R3"] < s["R1"]


# ------------------------------------------------------------------ score
def _F(n, B):
    # sum_{j=1..n} ceil(j/B) in closed form, n = Q*B + R
    Q, R = divmod(n, B)
    return B * Q * (Q + 1) // 2 + R * (Q + 1)


def test_score_spec_arithmetic_series(golden):
    row = golden["spec_examples"]["score"][0]
    c = mkcfg(block_tokens=row["B"], tau=row["tau"])
    assert O.score(c, ctx=row["ctx"], pre_rem=row["pre_rem"], has_api=0) == row["expect"]
    for L in range(0, 200):
        assert O.score(c, ctx=0, pre_rem=L, has_api=0) == L * (L + 1) // 2


@pytest.mark.parametrize("B", [1, 2, 16])
def test_score_ramp_closed_form(B):
    c = mkcfg(block_tokens=B, tau=7)
    rng = random.Random(6)
    for _ in range(300):
        c0, L = rng.randrange(3000), rng.randrange(600)
        assert O.score(c, ctx=c0, pre_rem=L, has_api=0) == 7 * (_F(c0 + L, B) - _F(c0, B))


def test_score_pending_rectangle():
    c = mkcfg(block_tokens=16, tau=5)
    assert O.score(c, ctx=33, pre_rem=0, pending=1000, has_api=0) == 3 * 1000


def test_score_api_phase_per_strategy():
    # A2's strategy phase (R7-R9) against hand values, B=16, tau=0 to isolate it
    c = mkcfg(block_tokens=16, tau=0, A1=3 << 4, A2=0, S0=5 << 4, S1=2 << 4, SH=4)
    # C_i = 30+5 = 35 tokens -> 3 blocks; resp 20 -> 55 tokens -> 4 blocks
    kw = dict(ctx=30, pre_rem=5, api_ticks=1000, resp_len=20, post_len=9)
    assert O.score(c, **kw, strategy=O.P) == 3 * 1000
    assert O.score(c, **kw, strategy=O.D) == 4 * (3 * 55)
    assert O.score(c, **kw, strategy=O.S) == 2 * 3 * (5 + 2 * 35)
    assert O.score(c, **kw, strategy=O.NONE) == 0
    # post ramp starts after the response: tau=1, no api time
    c2 = mkcfg(block_tokens=16, tau=1)
    assert O.score(c2, ctx=30, pre_rem=0, api_ticks=0, resp_len=20, post_len=9, strategy=O.P) == \
        (_F(59, 16) - _F(50, 16))


def test_score_monotone_in_lengths():
    # strictly increasing in the predicted lengths
    c = _gptj()
    for s in (O.P, O.D, O.S):
        prev = -1
        for L in range(0, 400, 7):
            v = O.score(c, ctx=100, pre_rem=L, api_ticks=500_000, resp_len=64, post_len=50, strategy=s)
            assert v > prev
            prev = v
        prev = -1
        for L in range(0, 400, 7):
            v = O.score(c, ctx=100, pre_rem=20, api_ticks=500_000, resp_len=64, post_len=L, strategy=s)
            assert v > prev
            prev = v


def test_score_no_api_is_sjf_order():
    # with no APIs and equal ctx/pending, LAMPS order = SJF order
    c = _gptj()
    rng = random.Random(7)
    L = [rng.randrange(1, 500) for _ in range(200)]
    sc = [O.score(c, ctx=300, pre_rem=x, has_api=0, pending=40_000) for x in L]
    assert sorted(range(200), key=lambda i: (sc[i], i)) == sorted(range(200), key=lambda i: (L[i], i))


def test_score_order_scale_invariant():
    # multiplying every time constant by k scales all scores by k (SH=0)
    rng = random.Random(8)
    base = dict(tau=3, A1=5, A2=1, S0=7, S1=2, SH=0, c_other=50, block_tokens=16)
    for k in (2, 5):
        c1 = mkcfg(**base)
        c2 = mkcfg(**{**base, **{n: base[n] * k for n in ("tau", "A1", "A2", "S0", "S1")}})
        for _ in range(200):
            kw = dict(ctx=rng.randrange(2000), pre_rem=rng.randrange(300), resp_len=rng.randrange(100),
                      post_len=rng.randrange(200), pending=rng.randrange(10 ** 5))
            api = rng.randrange(10 ** 6)
            s1 = O.argmin3(O.wastes(c1, kw["ctx"], kw["pre_rem"], api))
            s2 = O.argmin3(O.wastes(c2, kw["ctx"], kw["pre_rem"], api * k))
            assert s1 == s2
            v1 = O.score(c1, **kw, api_ticks=api, strategy=s1)
            v2 = O.score(c2, **{**kw, "pending": kw["pending"] * k}, api_ticks=api * k, strategy=s2)
            assert v2 == k * v1


def test_score_saturates():
    c = mkcfg(block_tokens=1, tau=1 << 40, score_bits=20)
    assert O.score(c, ctx=0, pre_rem=5, has_api=0) == (1 << 20) - 1
    c = mkcfg(block_tokens=1, tau=1, score_bits=3)
    assert O.score(c, ctx=0, pre_rem=3, has_api=0) == 6
    assert O.score(c, ctx=0, pre_rem=4, has_api=0) == 7
