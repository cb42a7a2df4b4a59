"""GPU backend of the reference CLI's run/bench/inspect (main.cpp:265-345):
outputs.csv bitwise the reference forward (%.17g), manifest fields, bench
CSV schema and stdout lines, exit codes; parsing errors on CPU."""
import os

import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import cli, synthetic


def test_cli_usage_and_parse_errors(tmp_path):
    assert cli.main([]) == 1
    assert cli.main(["bogus"]) == 1
    p = tmp_path / "x.csv"
    p.write_text("1,2\n\n3, 4 \n")
    assert cli._parse_input_csv(str(p), 2).tolist() == [[1.0, 2.0], [3.0, 4.0]]
    p.write_text("1,2\n3,x\n")
    with pytest.raises(hq.errors.ValueError, match="row 2: cannot parse 'x' as a number"):
        cli._parse_input_csv(str(p), 2)
    p.write_text("1,2,3\n")
    with pytest.raises(hq.errors.ValueError, match="row 1: expected 2 values, got 3"):
        cli._parse_input_csv(str(p), 2)
    assert cli.main(["inspect", "--model", str(tmp_path / "missing.skan")]) == 2


@pytest.mark.gpu
def test_cli_run_bench_inspect(tmp_path, capsys):
    cn = synthetic.synthetic_head(dims=(48, 24, 6), k=256, grid=10, int8=True, seed=3)
    ref = oracle.ref_build(cn)
    mpath = tmp_path / "m.skan"
    mpath.write_bytes(ref.serialize())
    x = synthetic.synthetic_inputs(4, 48, seed=2).reshape(4, 48)
    (tmp_path / "in.csv").write_text("".join(",".join("%.17g" % v for v in row) + "\n" for row in x))
    out = tmp_path / "out"
    assert cli.main(["run", "--model", str(mpath), "--input", str(tmp_path / "in.csv"), "--out-dir", str(out)]) == 0
    want, _ = oracle.port_forward(ref.tables(), x.reshape(-1), 4)
    got = np.array([[float(v) for v in line.split(",")] for line in (out / "outputs.csv").read_text().split("\n") if line])
    assert np.array_equal(got.reshape(-1), want)
    man = (out / "manifest.txt").read_text()
    assert "command = run" in man and "rows = 4" in man and "outputs = outputs.csv" in man
    assert "wrote 4 output rows" in capsys.readouterr().out
    # bench: G=5 vs G=10 heads of the same topology
    m2 = tmp_path / "g5.skan"
    m2.write_bytes(oracle.ref_build(synthetic.synthetic_head(dims=(48, 24, 6), k=256, grid=5, int8=True,
                                                             seed=4)).serialize())
    assert cli.main(["bench", "--model", str(m2), "--model", str(mpath), "--batch", "8", "--repeats", "5",
                     "--warmup", "1", "--out-dir", str(out)]) == 0
    text = capsys.readouterr().out
    assert "G=5: median " in text and "G=10: median " in text and "max/min median ratio: " in text
    assert (out / "bench.csv").read_text().splitlines()[0] == hq.bench_csv([]).splitlines()[0]
    assert cli.main(["bench", "--model", str(mpath), "--out-dir", str(out)]) == 1  # ConfigError
    assert cli.main(["inspect", "--model", str(mpath)]) == 0
    assert "layer 0: 48->24 G=10 K=256" in capsys.readouterr().out
