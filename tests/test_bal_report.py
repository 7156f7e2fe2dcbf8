"""BAL text I/O, the schema-1 run report and the `dba` front end (SURVEY.md §8f
rows f2, f3). KATs restated from tests/test_problem.cpp:16-80 and
tests/test_generator_report.cpp:12-135 of the reference; number parsing is
checked token by token against libc strtod / strtoll, which the reference
calls (dba/bal_io.hpp:41-61)."""
import ctypes
import ctypes.util
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from paper_2112_01349_b200 import report as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MINIMAL = b"1 1 1\n0 0 0.0 0.0\n0\n0\n0\n0\n0\n0\n1\n0\n0\n0\n0\n1\n"


def test_parse_minimal_well_formed():  # test_problem.cpp:24-33
    p = dba.parse_bal(MINIMAL)
    assert (p.num_cameras, p.num_points, p.num_observations) == (1, 1, 1)
    assert p.arrays()[0][0, 6] == 1.0
    assert list(p.arrays()[1][0]) == [0.0, 0.0, 1.0]
    assert p.validate() == []


def test_parse_rejects_out_of_range_index_with_line():  # test_problem.cpp:35-44
    with pytest.raises(dba.ParseError) as e:
        dba.parse_bal(b"2 1 1\n5 0 0 0\n")
    assert e.value.line == 2
    assert "camera index 5" in str(e.value)
    assert str(e.value).startswith("line 2: ")
    with pytest.raises(dba.ParseError, match=r"line 3: point index 1 out of range \[0, 1\)"):
        dba.parse_bal(b"1 1 2\n0 0 1 2\n0 1 3 4\n")


@pytest.mark.parametrize("text, msg", [
    (b"1 1 1\n0 0 0.0\n", "unexpected end of input"),            # truncated
    (b"1 1 1\n0 0 0.0 xyz\n", "expected number, got 'xyz'"),     # garbage
    (b"1 1 1\n0 0 0.0 nan\n", "non-finite value 'nan'"),         # non-finite
    (b"1 1 1\n0 0 0.0 1e999\n", "non-finite value '1e999'"),     # overflow -> inf
    (b"1 1 x\n", "expected integer, got 'x'"),
    (b"1 1 1.5\n", "expected integer, got '1.5'"),
    (b"1 -1 1\n", "negative count in header"),
    (b"", "unexpected end of input"),
])
def test_parse_rejects_bad_input(text, msg):  # test_problem.cpp:46-55
    with pytest.raises(dba.ParseError, match=msg):
        dba.parse_bal(text)


def test_non_positive_focal_warns_but_parses():  # test_problem.cpp:57-68
    w = []
    p = dba.parse_bal(b"1 1 1\n0 0 0.0 0.0\n0\n0\n0\n0\n0\n0\n-2\n0\n0\n0\n0\n1\n", warnings=w)
    assert p.arrays()[0][0, 6] == -2.0
    assert len(w) == 1 and "non-positive focal" in w[0]


def test_tokens_follow_strtod_strtoll():
    libc = ctypes.CDLL(ctypes.util.find_library("c"))
    libc.strtod.restype = ctypes.c_double
    libc.strtod.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    reals = [b"0.1", b"+1.5", b"-2.25e-3", b"0x1p3", b"1E+02", b"3.", b".5", b"7", b"-0", b"4.9e-324",
             b"1.7976931348623157e308", b"2.2250738585072014e-308", b"123456789012345678901234567890"]
    body = b"\t".join(reals[:9]) + b"\r\n" + b"  ".join(reals[9:])
    text = b"1 1 1\n0 0 " + reals[0] + b" " + reals[1] + b"\n" + b" ".join(reals[2:11]) + b"\n" + b" ".join(reals[11:13]) + b" 1\n"
    p = dba.parse_bal(text)
    got = list(p.arrays()[0].reshape(-1)) + list(p.arrays()[1].reshape(-1))
    want = [libc.strtod(t, None) for t in reals[2:13]] + [1.0]
    assert [x.hex() for x in got] == [x.hex() for x in want]
    assert p.arrays()[4][0] == libc.strtod(reals[0], None) and p.arrays()[5][0] == 1.5
    assert body  # tabs / CRLF separate tokens too
    q = dba.parse_bal(b"+1\t1\r\n001\n0 0 1 2\n" + b"0\n" * 6 + b"1\n0\n0\n0\n0\n1\n")
    assert q.num_cameras == 1 and q.num_observations == 1


def test_round_trip_preserves_values_exactly():  # test_problem.cpp:70-80
    rng = np.random.default_rng(7)
    m, n, N = 3, 5, 9
    cams = rng.normal(size=(m, 9)) * [1, 1, 1, 1, 1, 1, 500, 0.1, 0.1]
    pts = rng.normal(size=(n, 3))
    cid = rng.integers(0, m, N).astype(np.int32)
    pid = rng.integers(0, n, N).astype(np.int32)
    pix = rng.normal(size=(N, 2)) * 300
    p = dba.BAProblem.from_arrays(cams, pts, cid, pid, pix)
    text = dba.format_bal(p)
    q = dba.parse_bal(text)
    for a, b in zip(p.arrays(), q.arrays()):
        assert np.array_equal(a, b)
    assert dba.format_bal(q) == text
    # the reference's "%.16e" line format
    line = text.split(b"\n")[1].split(b" ")
    assert line[2] == (b"%.16e" % pix[0, 0])


def test_fp32_parse_casts_like_parse_bal_float():
    p = dba.parse_bal(MINIMAL.replace(b"0 0 0.0 0.0", b"0 0 0.1 0.2"), dtype=np.float32)
    assert p.dtype == np.float32 and p.arrays()[4][0] == np.float32(0.1)


def test_generator_counts_header_determinism_and_parse_back():  # test_generator_report.cpp:12-70
    g = dba.generate_synthetic(dba.SyntheticOptions(cameras=20, points=80, obs_per_point=10))
    text = dba.format_bal(g)
    assert text.split(b"\n")[0] == b"20 80 800"
    assert g.validate() == []
    o = dba.SyntheticOptions(cameras=5, points=9, obs_per_point=3, seed=4)
    assert dba.format_bal(dba.generate_synthetic(o)) == dba.format_bal(dba.generate_synthetic(o))
    o2 = dba.SyntheticOptions(cameras=5, points=9, obs_per_point=3, seed=5)
    assert dba.format_bal(dba.generate_synthetic(o)) != dba.format_bal(dba.generate_synthetic(o2))
    w = []
    q = dba.parse_bal(dba.format_bal(dba.generate_synthetic(dba.SyntheticOptions(cameras=7, points=15,
                                                                                  obs_per_point=3))), warnings=w)
    assert (q.num_cameras, q.num_points, q.num_observations) == (7, 15, 45) and w == []


# ------------------------------------------------------------------ report --

def _sample_report():
    its = [dba.IterationRecord(1, 1234.5, 1.5e-07, 1e-4, 17, True, 0.0123, [45, 45], [900, 900]),
           dba.IterationRecord(2, 1e15, 0.0001, 3.3333333333333335e-05, 0, False, 1.0, [45, 45], [0, 0]),
           dba.IterationRecord(3, 100.0, 1e-05, 1e+32, 500, True, 123456.789, [1], [2])]
    cfg = dba.SolverConfig(workers=2, max_iterations=3)
    state = dba.SolverState(np.zeros(9), np.zeros(3), 1e-4, 2.0, 3, 100.0, "max_iterations", its)
    return R.make_report("sample", cfg, state, 90)


def test_report_round_trips_byte_identically():  # test_generator_report.cpp:105-115
    r = _sample_report()
    once = dba.serialize_report(r)
    parsed = dba.report_from_json(once)
    assert dba.serialize_report(parsed) == once
    assert parsed.schema == 1 and parsed.dataset == "sample" and len(parsed.iterations) == 3
    assert json.loads(once)["config"]["damping"] == "diagonal"


def test_report_key_order_and_number_format():
    """dba/report.hpp:81-119 key order; nlohmann::json float output."""
    d = json.loads(dba.serialize_report(_sample_report()))
    assert list(d) == ["schema", "dataset", "workers", "precision", "config", "iterations", "final_cost", "final_mse",
                       "final_mse_alternate", "termination"]
    assert list(d["config"]) == ["max_iterations", "pcg_tol", "pcg_max_iters", "lambda0", "lambda_max", "rel_tol",
                                 "step_tol", "damping", "mse_convention", "jacobian"]
    assert list(d["iterations"][0]) == ["iteration", "cost", "mse", "lambda", "pcg_iterations", "accepted",
                                        "wall_seconds", "worker_edges", "worker_block_ops"]
    f = R._fmt_double
    assert [f(x) for x in (1e-06, 100.0, 1e+32, 0.0001, 1e-05, 1e15, 1e14, 1.5, -0.0, 0.1, 123456.789,
                           1.2345678901234568e+17, 2.5e-300, float("inf"))] == [
        "1e-06", "100.0", "1e+32", "0.0001", "1e-05", "1e+15", "100000000000000.0", "1.5", "-0.0", "0.1",
        "123456.789", "1.2345678901234568e+17", "2.5e-300", "null"]
    text = dba.serialize_report(_sample_report())
    assert text.startswith('{\n  "schema": 1,\n  "dataset": "sample",\n') and text.endswith("}\n")
    assert '"worker_edges": [\n        45,\n        45\n      ],' in text


def test_report_mse_under_both_conventions():  # test_generator_report.cpp:117-135
    r = _sample_report()
    assert r.final_mse == dba.dba.mse_from_cost(100.0, 90, dba.dba.MSE_HALF_PER_OBSERVATION)
    assert r.final_mse_alternate == dba.dba.mse_from_cost(100.0, 90, dba.dba.MSE_PER_OBSERVATION)


def test_report_rejects_other_schema():
    d = json.loads(dba.serialize_report(_sample_report()))
    d["schema"] = 2
    with pytest.raises(dba.ParseError, match="unsupported report schema 2"):
        dba.report_from_json(json.dumps(d))


# --------------------------------------------------------------------- CLI --

def _cli(*args, **kw):
    return subprocess.run([sys.executable, "-m", "paper_2112_01349_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=300, **kw)


def test_cli_generate_and_parse_errors(tmp_path):  # tools/dba_main.cpp:45-60, 173-225
    out = tmp_path / "ring.txt"
    r = _cli("generate", "--cameras", "6", "--points", "12", "--obs-per-point", "3", "--output", str(out))
    assert r.returncode == 0, r.stderr
    assert "generated 6 cameras, 12 points, 36 observations (seed 1)" in r.stderr
    assert out.read_bytes().startswith(b"6 12 36\n")
    bad = tmp_path / "bad.txt"
    bad.write_bytes(b"2 1 1\n5 0 0 0\n")
    r = _cli("solve", "--input", str(bad))
    assert r.returncode == 2 and "error: " in r.stderr and "line 2: camera index 5" in r.stderr
    r = _cli("solve", "--input", str(tmp_path / "missing.txt"))
    assert r.returncode == 2 and "cannot open" in r.stderr
    r = _cli("solve", "--input", str(out), "--damping", "bogus")
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_solve_report(tmp_path):
    bal = tmp_path / "ring.txt"
    assert _cli("generate", "--cameras", "10", "--points", "60", "--obs-per-point", "4", "--pixel-noise", "0.5",
                "--output", str(bal)).returncode == 0
    rep = tmp_path / "report.json"
    r = _cli("solve", "--input", str(bal), "--max-iters", "4", "--output", str(rep))
    assert r.returncode == 0, r.stderr
    text = rep.read_text()
    d = json.loads(text)
    assert d["dataset"] == "ring" and d["precision"] == "fp64" and len(d["iterations"]) == 4
    assert dba.serialize_report(dba.report_from_json(text)) == text
    # the same solve through the API: identical cost trajectory
    p = dba.parse_bal(bal.read_bytes())
    s = dba.lm_solve(p, dba.SolverConfig(max_iterations=4))
    assert [it["cost"] for it in d["iterations"]] == [it.cost for it in s.history]
    assert "iter 1" in r.stderr and "final mse" in r.stderr


NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp"


@pytest.mark.skipif(not os.path.exists(NLOHMANN), reason="nlohmann/json single header not in this image")
def test_report_text_matches_nlohmann_dump(tmp_path):
    """The reference serialises with nlohmann::ordered_json::dump(2)
    (dba/report.hpp:165-167): emit the sample report's document through the
    real library and compare byte for byte."""
    doc = R.to_json(_sample_report())
    vals = [1e-06, 100.0, 1e+32, 0.0001, 1e-05, 1e15, 1e14, 1.5, -0.0, 0.1, 123456.789, 1.2345678901234568e+17,
            2.5e-300, 3.3333333333333335e-05, 5e-324, 1.7976931348623157e308, 0.30000000000000004]
    doc["probe"] = vals
    # The cudnn_frontend copy of nlohmann 3.11.3 prints integer arrays on one
    # line ("Custom from FE"); restore the stock serializer the reference
    # links (one element per line) in a private copy.
    hdr = open(NLOHMANN).read()
    custom = ("if (pretty_print && (elementType != value_t::number_integer) &&\n"
              "                    (elementType != value_t::number_unsigned))")
    hdr = hdr.replace(custom, "if (pretty_print)")
    (tmp_path / "json.hpp").write_text(hdr)
    src = tmp_path / "dump.cpp"
    src.write_text('#include <iostream>\n#include "json.hpp"\nint main() {\n'
                   '  auto j = nlohmann::ordered_json::parse(std::cin);\n  std::cout << j.dump(2) << "\\n";\n}\n')
    exe = tmp_path / "dump"
    subprocess.run(["g++", "-O0", "-std=c++17", "-I", str(tmp_path), str(src), "-o", str(exe)], check=True,
                   timeout=300)
    ours = R._dump(doc, 0) + "\n"
    theirs = subprocess.run([str(exe)], input=ours, capture_output=True, text=True, check=True).stdout
    assert ours == theirs
