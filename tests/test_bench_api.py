"""bench_model / bench_iso_latency / bench_csv mirrors (lutham.cpp:852-951)
and the reference acceptance check 6 (iso-latency across grid resolutions,
acceptance.cpp:387-421) on the device."""
import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200.lutham import _MT19937_64, _percentile


def test_mt19937_64_matches_the_standard():
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64
    r = _MT19937_64(5489)
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042


def test_bench_csv_schema_and_percentile():
    rows = [hq.BenchRow(5, 0.1 + 0.2, 1.25, 2.0), hq.BenchRow(128, 3.0, 2.5, 3.5)]
    assert hq.bench_csv(rows) == "G,median_us,p25_us,p75_us\n5,0.30000000000000004,1.25,2\n128,3,2.5,3.5\n"
    v = sorted([5.0, 1.0, 3.0, 2.0, 4.0])
    assert (_percentile(v, 0.5), _percentile(v, 0.25), _percentile(v, 0.75)) == (3.0, 2.0, 4.0)


@pytest.mark.gpu
def test_iso_latency_g5_vs_g128_on_device():
    """acceptance.cpp:387-421: {2,16,1}, K=16, G in {5, 128}: median latency
    ratio <= 1.5 and one interpolation per edge-sample at both resolutions."""
    models, edges = [], 2 * 16 + 16 * 1
    for G in (5, 128):
        m = oracle.ref_random([2, 16, 1], G, 0.4, 90, 16, False)
        models.append(hq.upload([t.to_runtime() for t in m.tables()]))
    rows = hq.bench_iso_latency(models, hq.BenchConfig(batch=64, repeats=151, warmup=20))
    ratio = max(r.median_us for r in rows) / min(r.median_us for r in rows)
    assert ratio <= 1.5, hq.bench_csv(rows)
    for m in models:
        ws = hq.make_workspace(m, 32)
        y = np.zeros(32)
        hq.compressed_forward(m, np.full(64, 0.1), 32, y, ws)
        assert ws.interp_ops == 32 * edges
