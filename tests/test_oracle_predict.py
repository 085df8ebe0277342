"""Oracle pins for SURVEY row F4: predictor ingest (bins of 10 tokens) and the
paper's error injection error ~ N(0, p*m), reading R27 (integer,
counter-based normal draw; include/lamps.h lamps_noise).

Pinned against: published splitmix64 output vectors, the exact Binomial(1024, 1/2)
law, the standard normal CDF, the paper's bin midpoints and p values, closed-form
rounding cases -- not against a retyped copy of the oracle's formula."""
import math

import numpy as np
import pytest

import gen
import oracle as O

LIMIT = 1 << 24


def truth_array(d: dict) -> np.ndarray:
    n = len(d["key"])
    a = np.zeros(n, O.TRUTH_DTYPE)
    for f in ("key", "prompt_len", "pre_len", "pre_bin", "resp_len", "post_len", "api_ticks", "has_api"):
        a[f] = d[f]
    return a


def single(m_pre=100, m_post=50, api=1_000_000, key=0, has=1, b=O.NO_BIN, resp=7, prompt=11):
    return truth_array(dict(key=[key], prompt_len=[prompt], pre_len=[m_pre], pre_bin=[b], resp_len=[resp],
                            post_len=[m_post], api_ticks=[api], has_api=[has]))


def test_splitmix64_published_vectors():
    """splitmix64 (Steele, Lea & Flood 2014; Vigna's reference splitmix64.c): the widely
    published first outputs for seeds 1234567 and 0."""
    assert [O.splitmix_output(1234567, n) for n in range(1, 6)] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
        16408922859458223821]
    assert [O.splitmix_output(0, n) for n in range(1, 4)] == [
        0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_no_error_is_identity_and_bins_are_midpoints():
    """p = 0: predictions equal the measured values (Noisy(0) == Oracle);
    bin b -> 10 b + 5 tokens, the midpoint of the bin's 10 tokens."""
    d = gen.truths("C3", 500, seed=1)
    rc, p = O.predict(truth_array(d))
    assert rc == O.OK
    has = d["has_api"] == 1
    assert np.array_equal(p["pre_len"], d["pre_len"])
    assert np.array_equal(p["post_len"], np.where(has, d["post_len"], 0))
    assert np.array_equal(p["api_ticks"], np.where(has, d["api_ticks"], 0))
    assert np.array_equal(p["resp_len"], np.where(has, d["resp_len"], 0))
    db = gen.truths("C4", 500, seed=2, bins=True)
    rc, pb = O.predict(truth_array(db))
    assert rc == O.OK
    for b, v in zip(db["pre_bin"], pb["pre_len"]):
        assert 10 * b <= v <= 10 * b + 9 and v == 10 * b + 5
    assert pb["pre_len"].min() >= 5 and pb["pre_len"].max() <= 495  # 50 bins


def test_binomial_law_of_the_popcount_sum():
    """X = Z // 2^16 + 512 must follow Binomial(1024, 1/2) exactly; the dither
    (Z mod 2^16) must be uniform.  Chi-square against the exact pmf."""
    N = 40000
    Z = np.array([O.normal_q20(99, k, k % 3) for k in range(N)], np.int64)
    X = (Z + 32768) // 65536 + 512
    U = (Z + 32768) % 65536
    assert X.min() >= 0 and X.max() <= 1024
    # exact pmf, cells of width 4 around the centre, tails pooled
    lo, hi = 512 - 48, 512 + 48
    edges = list(range(lo, hi + 1, 4))
    from fractions import Fraction
    pmf = np.array([float(Fraction(math.comb(1024, x), 1 << 1024)) for x in range(1025)])
    obs, exp = [], []
    obs.append((X < lo).sum()); exp.append(pmf[:lo].sum() * N)
    for a, b in zip(edges[:-1], edges[1:]):
        obs.append(((X >= a) & (X < b)).sum()); exp.append(pmf[a:b].sum() * N)
    obs.append((X >= hi).sum()); exp.append(pmf[hi:].sum() * N)
    obs, exp = np.array(obs, float), np.array(exp)
    chi2 = ((obs - exp) ** 2 / exp).sum()
    dof = len(obs) - 1  # 25
    assert chi2 < dof + 6 * math.sqrt(2 * dof), chi2
    hu, _ = np.histogram(U, bins=16, range=(0, 65536))
    chi2u = ((hu - N / 16) ** 2 / (N / 16)).sum()
    assert chi2u < 15 + 6 * math.sqrt(30), chi2u


def test_normal_draw_matches_standard_normal():
    """z = Z / 2^20: mean 0, variance 1 + 1/(12*256) (binomial + one-step dither),
    Kolmogorov-Smirnov distance to Phi small."""
    N = 40000
    z = np.array([O.normal_q20(7, k, 2) for k in range(N)], float) / 2.0 ** 20
    assert abs(z.mean()) < 5 / math.sqrt(N)
    assert abs(z.var() - (1 + 1 / 3072)) < 6 * math.sqrt(2 / N)
    zs = np.sort(z)
    phi = np.array([0.5 * (1 + math.erf(v / math.sqrt(2))) for v in zs])
    ks = max(np.max(np.arange(1, N + 1) / N - phi), np.max(phi - np.arange(N) / N))
    assert ks < 1.95 / math.sqrt(N) + 0.004, ks
    # symmetric, and the two sides of 0 are balanced
    assert abs((z > 0).mean() - 0.5) < 5 * 0.5 / math.sqrt(N)


@pytest.mark.parametrize("p", [0.05, 0.10, 0.30])
def test_error_scale_is_p_times_m(p):
    """error ~ N(0, p * m) -- the standard deviation of the error is p*m.
    The paper's p values 5, 10, 30 %; m large so rounding is negligible."""
    N, m = 6000, 10_000
    d = dict(key=np.arange(N), prompt_len=np.full(N, 10), pre_len=np.full(N, m), pre_bin=np.full(N, O.NO_BIN),
             resp_len=np.zeros(N), post_len=np.full(N, m), api_ticks=np.full(N, m * 100), has_api=np.ones(N))
    rc, pr = O.predict(truth_array(d), seed=3, len_error_ppm=int(p * 1e6), api_error_ppm=int(p * 1e6))
    assert rc == O.OK
    for f, mm in (("pre_len", m), ("post_len", m), ("api_ticks", m * 100)):
        e = pr[f].astype(float) - mm
        assert abs(e.mean()) < 5 * p * mm / math.sqrt(N), f
        assert abs(e.std() / (p * mm) - 1) < 0.05, (f, e.std() / (p * mm))
    # the three fields draw independent errors
    c = np.corrcoef(pr["pre_len"].astype(float), pr["post_len"].astype(float))[0, 1]
    assert abs(c) < 5 / math.sqrt(N)
    c = np.corrcoef(pr["pre_len"].astype(float), pr["api_ticks"].astype(float))[0, 1]
    assert abs(c) < 5 / math.sqrt(N)


def test_clamp_at_zero_fraction():
    """p = 50 %: predicted = max(0, m + e) is 0 exactly when z <= -2 (up to
    rounding), i.e. with probability Phi(-2) = 2.28 %."""
    N, m = 20000, 1000
    d = dict(key=np.arange(N), prompt_len=np.full(N, 10), pre_len=np.full(N, m), pre_bin=np.full(N, O.NO_BIN),
             resp_len=np.zeros(N), post_len=np.zeros(N), api_ticks=np.zeros(N), has_api=np.zeros(N))
    rc, pr = O.predict(truth_array(d), seed=11, len_error_ppm=500_000)
    assert rc == O.OK
    frac = (pr["pre_len"] == 0).mean()
    phi_m2 = 0.5 * (1 + math.erf(-2 / math.sqrt(2)))
    assert abs(frac - phi_m2) < 5 * math.sqrt(phi_m2 / N), frac


def test_rounding_half_away_from_zero_closed_forms():
    """error = p m z rounded half away from zero: with p = 1 (10^6 ppm) and
    z = +-1/2 (Z = +-2^19) the error of m = 1 is +-0.5 -> +-1; m = 3: +-1.5 -> +-2;
    z just below 1/2 rounds toward 0."""
    H = 1 << 19
    assert O.perturb(1, 1_000_000, H, LIMIT) == 2
    assert O.perturb(1, 1_000_000, -H, LIMIT) == 0
    assert O.perturb(3, 1_000_000, H, LIMIT) == 5
    assert O.perturb(3, 1_000_000, -H, LIMIT) == 1
    assert O.perturb(1, 1_000_000, H - 1, LIMIT) == 1
    assert O.perturb(1, 1_000_000, -(H - 1), LIMIT) == 1
    assert O.perturb(10, 500_000, 1 << 20, LIMIT) == 15          # p m z = 0.5 * 10 * 1
    assert O.perturb(10, 500_000, -(1 << 21), LIMIT) == 0        # 10 - 10
    assert O.perturb(10, 500_000, -(3 << 20), LIMIT) == 0        # clamp at 0
    assert O.perturb(LIMIT - 1, 10_000_000, 1 << 22, LIMIT) == LIMIT  # clamp at the ingest limit
    assert O.perturb(0xFFFFFFFF, 10_000_000, 1 << 22, 0xFFFFFFFF) == 0xFFFFFFFF
    assert O.perturb(12345, 0, 1 << 22, LIMIT) == 12345


def test_determinism_and_streams():
    """Same (seed, key) -> same prediction whatever the batch; different seed or key ->
    (almost always) different draws; a bin and a measured m of the same value draw alike."""
    d = gen.truths("C2", 300, seed=5)
    a = truth_array(d)
    rc, p1 = O.predict(a, seed=42, len_error_ppm=100_000, api_error_ppm=100_000)
    rc2, p2 = O.predict(a[::-1].copy(), seed=42, len_error_ppm=100_000, api_error_ppm=100_000)
    assert rc == rc2 == O.OK
    assert np.array_equal(p1, p2[::-1])
    rc3, p3 = O.predict(a, seed=43, len_error_ppm=100_000, api_error_ppm=100_000)
    has = d["has_api"] == 1
    assert (p3["api_ticks"] != p1["api_ticks"])[has].mean() > 0.9
    bb = single(m_pre=0, b=7, key=5)
    mm = single(m_pre=75, key=5)
    _, pb = O.predict(bb, seed=1, len_error_ppm=300_000)
    _, pm = O.predict(mm, seed=1, len_error_ppm=300_000)
    assert pb["pre_len"][0] == pm["pre_len"][0]


def test_validation():
    assert O.predict(single(has=2))[0] == O.EINVAL
    assert O.predict(single(b=50))[0] == O.EINVAL
    assert O.predict(single(key=1 << 57))[0] == O.EINVAL
    assert O.predict(single(), len_error_ppm=10_000_001)[0] == O.EINVAL
    a = single(); a["reserved"] = 1
    assert O.predict(a)[0] == O.EINVAL
    rc, p = O.predict(single(has=0, m_post=9, api=9, resp=9))
    assert rc == O.OK and p["post_len"][0] == 0 and p["api_ticks"][0] == 0 and p["resp_len"][0] == 0
