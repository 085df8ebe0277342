"""GPU <-> oracle parity for SURVEY row F4 (lamps_predict / k_predict): bin -> tokens
 and error injection N(0, p*m) (reading R27), bit-exact on the
same seeded truths; and the predict -> submit chain quantises back to the same ticks."""
import numpy as np
import pytest

import gen
import oracle as O
from test_oracle_predict import truth_array

pytestmark = pytest.mark.gpu


def sched(cname="C3"):
    from paper_2410_18248_b200 import Scheduler
    return Scheduler(gen.lib_config(cname))


def compare(seg, pred, truth):
    assert np.array_equal(seg["pre_len"], pred["pre_len"])
    assert np.array_equal(seg["post_len"], pred["post_len"])
    assert np.array_equal(seg["resp_len"], pred["resp_len"])
    assert np.array_equal(seg["has_api"], truth["has_api"])
    assert np.array_equal(seg["prompt_len"], truth["prompt_len"])
    ticks = np.array([O.quantize(float(x), 1e6)[1] for x in seg["api_seconds"]], np.int64)
    assert np.array_equal(ticks, pred["api_ticks"].astype(np.int64))


@pytest.mark.parametrize("bins", [False, True])
@pytest.mark.parametrize("len_ppm,api_ppm", [(0, 0), (50_000, 0), (100_000, 100_000), (300_000, 500_000),
                                             (500_000, 300_000), (10_000_000, 10_000_000)])
def test_predict_parity(bins, len_ppm, api_ppm):
    s = sched()
    for n, seed in ((1, 0), (257, 1), (70_001, 2)):  # one record, a ragged block, > one staging chunk
        t = truth_array(gen.truths("C4", n, seed=seed, bins=bins, key0=seed * 1_000_003))
        seg = s.predict(t, seed=0xC0FFEE + seed, len_error_ppm=len_ppm, api_error_ppm=api_ppm)
        rc, pred = O.predict(t, seed=0xC0FFEE + seed, len_error_ppm=len_ppm, api_error_ppm=api_ppm)
        assert rc == O.OK
        compare(seg, pred, t)
    s.close()


def test_predict_extreme_keys_and_values():
    s = sched()
    n = 4096
    rng = np.random.default_rng(5)
    d = dict(key=rng.integers(0, 1 << 57, n, dtype=np.uint64), prompt_len=rng.integers(0, 1 << 20, n),
             pre_len=rng.integers(0, 1 << 32, n, dtype=np.uint64), pre_bin=np.full(n, O.NO_BIN),
             resp_len=rng.integers(0, 1 << 32, n, dtype=np.uint64),
             post_len=rng.integers(0, 1 << 32, n, dtype=np.uint64),
             api_ticks=rng.integers(0, 1 << 32, n, dtype=np.uint64), has_api=rng.integers(0, 2, n))
    t = truth_array(d)
    for ppm in (1, 999_999, 10_000_000):
        seg = s.predict(t, seed=(1 << 64) - 1 - ppm, len_error_ppm=ppm, api_error_ppm=ppm)
        rc, pred = O.predict(t, seed=(1 << 64) - 1 - ppm, len_error_ppm=ppm, api_error_ppm=ppm)
        assert rc == O.OK
        compare(seg, pred, t)
    s.close()


def test_predict_errors_match_oracle():
    from paper_2410_18248_b200.lamps import LAMPS_EINVAL
    s = sched()
    base = truth_array(gen.truths("C2", 4, seed=9))
    for mut in ("has", "bin", "key", "reserved"):
        t = base.copy()
        if mut == "has": t["has_api"][2] = 2
        if mut == "bin": t["pre_bin"][1] = 50
        if mut == "key": t["key"][3] = 1 << 57
        if mut == "reserved": t["reserved"][0] = 1
        assert s.predict_rc(t)[0] == LAMPS_EINVAL
        assert O.predict(t)[0] == O.EINVAL
    assert s.predict_rc(base, len_error_ppm=10_000_001)[0] == LAMPS_EINVAL
    rc, seg = s.predict_rc(base, noise=False)
    assert rc == 0
    compare(seg, O.predict(base)[1], base)
    s.close()


def test_predict_then_submit_pool_matches_oracle():
    """The predicted segments feed lamps_submit; the pool the GPU builds from them equals
    the oracle's pool built from the oracle's predictions (ticks survive the seconds
    round trip exactly)."""
    cfg = gen.lib_config("C3")
    s = sched()
    t = truth_array(gen.truths("C3", 1500, seed=3))
    seg = s.predict(t, seed=77, len_error_ppm=300_000, api_error_ppm=300_000)
    ids = s.submit(seg)
    rc, pred = O.predict(t, seed=77, len_error_ppm=300_000, api_error_ppm=300_000)
    o = O.OraclePool(cfg)
    rows = [dict(prompt_len=int(a), pre_len=int(p["pre_len"]), resp_len=int(p["resp_len"]),
                 post_len=int(p["post_len"]), api_seconds=float(p["api_ticks"]) / 1e6, has_api=int(h))
            for a, p, h in zip(t["prompt_len"], pred, t["has_api"])]
    rc, oids = o.submit(O.segments(rows))
    assert rc == O.OK and np.array_equal(ids, oids)
    e = s.export_pool()
    for f in ("ctx", "pre_rem", "api_ticks", "resp_len", "post_len", "pending", "has_api"):
        assert np.array_equal(e[f].astype(np.int64), o.pool[f].astype(np.int64)), f
    s.close()
