"""Batch build/query from key files (harness.cpp:247-304) and the sizing model
(model.cpp) — parity with the reference."""
import hashlib
import io
import json
import os
import sys

import numpy as np
import pytest

from paper_2101_01719_b200 import tools as T

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "frontend.json")) as fh:
        return json.load(fh)


def write_lines(path, lines, trailing_newline=True):
    data = b"\n".join(lines) + (b"\n" if trailing_newline and lines else b"")
    with open(path, "wb") as fh:
        fh.write(data)


def test_read_key_lines_semantics(tmp_path):
    p = tmp_path / "k"
    for content, want in ((b"", []), (b"\n", [b""]), (b"a\nb\n", [b"a", b"b"]), (b"a\nb", [b"a", b"b"]),
                          (b"a\n\nb\n", [b"a", b"", b"b"])):
        p.write_bytes(content)
        assert T.read_key_lines(str(p)) == want


def test_model_matches_reference(reference):
    for a in (0.0, 0.5, 5.0, 20.0, 24.4140625, 30.517578125, 52.0, 1000.0):
        assert T.sbbf_fpp(a) == reference.lib.ref_sbbf_fpp(a)
    for ndv in (1, 17, 1000, 100_000, 10_000_000):
        for fpp in (0.5, 0.1, 0.01, 0.001, 1e-5):
            assert T.size_for(ndv, fpp) == reference.lib.ref_size_for(ndv, fpp), (ndv, fpp)


@pytest.mark.gpu
@pytest.mark.parametrize("fpp", ["0.01", "0.001", "0.2"])
def test_build_and_query_match_reference(cuda, oracle, golden, tmp_path, fpp):
    import make_golden
    keys, probes = make_golden.build_query_inputs()
    kf, pf, out = tmp_path / "keys", tmp_path / "probes", tmp_path / "f.sbbf"
    write_lines(kf, keys)
    write_lines(pf, probes, trailing_newline=False)
    g = golden["build_query"]
    r = T.run_build(str(kf), str(out), float(fpp))
    assert r["keys_read"] == g["keys_read"] and r["distinct_hashes"] == g["distinct"]
    run = g["runs"][fpp]
    assert r["num_buckets"] == run["num_buckets"]
    img = out.read_bytes()
    assert int.from_bytes(img[-4:], "little") == run["image_crc"]
    rc, blocks, hid = oracle.deserialize(img)                    # the reference's image format
    assert rc == 0 and hid == 1 and blocks.shape[0] == run["num_buckets"]
    sink = io.StringIO()
    q = T.run_query(str(out), str(pf), out=sink)
    lines = sink.getvalue().splitlines()
    ans = np.array([1 if x == "maybe" else 0 for x in lines], np.uint8)
    assert q["maybe"] == run["maybe"] and len(lines) == len(probes)
    assert hashlib.sha256(ans.tobytes()).hexdigest() == run["answers_sha256"]


def test_size_cli(reference, capsys):
    """`sbbf size` (main.cpp cmd_size): bit-exact sizing, output format,
    efficient-range warning, usage errors -> exit 1."""
    from paper_2101_01719_b200 import tools
    assert tools.main(["size", "--ndv", "1000000", "--fpp", "0.01"]) == 0
    out = capsys.readouterr()
    nb = tools.size_for(1_000_000, 0.01)
    assert out.out.strip() == (f"ndv=1000000 target_fpp=0.01 -> buckets={nb} bytes={nb * 32} "
                               f"(a={1_000_000 / nb:.3f}, predicted fpp={tools.sbbf_fpp(1_000_000 / nb):.6f})")
    assert out.err == ""
    assert tools.main(["size", "--ndv", "1000", "--fpp", "0.5"]) == 0
    assert "outside the efficient range" in capsys.readouterr().err
    assert tools.main(["size", "--ndv", "1000", "--fpp", "1.5"]) == 1
    r = tools.sizing(123_457, 0.02)
    assert r["num_buckets"] == reference.lib.ref_size_for(123_457, 0.02)


def test_model_cli_matches_reference(reference, capsys, tmp_path):
    """`sbbf model` (run_model / within_2x_report): every row bit-exact with
    the reference's standard_bloom_fpp / optimal_bloom_k / sbbf_fpp."""
    from paper_2101_01719_b200 import tools
    r = tools.run_model()
    assert len(r["rows"]) == 65
    for row in r["rows"]:
        bpk = 256.0 / row["a"]
        k = reference.lib.ref_optimal_bloom_k(bpk)
        assert tools.optimal_bloom_k(bpk) == k
        assert row["standard_fpp"] == reference.lib.ref_standard_bloom_fpp(bpk, k)
        assert row["sbbf_fpp"] == reference.lib.ref_sbbf_fpp(row["a"])
    assert r["max_ratio"] <= tools.WITHIN_2X_BOUND
    csv = tmp_path / "m.csv"
    assert tools.main(["model", "--assert-2x", "--csv", str(csv)]) == 0
    assert csv.read_text().splitlines()[0] == "a,bits_per_key,sbbf_fpp,standard_fpp,ratio"
    assert capsys.readouterr().out.splitlines()[-1] == f"max ratio: {r['max_ratio']:.4f}"
    assert tools.main(["model", "--a-min", "5", "--a-max", "1"]) == 1
    assert tools.main(["model", "--a-min", "60", "--a-max", "200", "--steps", "9", "--assert-2x"]) in (0, 3)
