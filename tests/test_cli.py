"""The CLI front-end (tools/fpb200_cli.cpp) against the reference CLI's contract (tests/test_cli.cpp).

Each reference TEST_CASE is restated here with the same arguments and assertions, plus parity
checks the reference cannot make: generated inputs bit-identical to the reference generators
(golden fixtures), containers byte-identical to the reference writer, and CLI outputs equal to the
oracle on the same inputs.  Paths that fail before any device call (usage, format, io, shape
validation, `gen`) run on CPU; the rest are marked gpu.
"""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from tests._util import read_fpt, write_fpt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session")
def cli():
    from paper_2603_06199_b200 import build as b
    return b.build_cli()


def run(cli, args, cwd=None):
    r = subprocess.run([cli, *args.split()], capture_output=True, text=True, timeout=600, cwd=cwd)
    return r.returncode, r.stdout, r.stderr


def strip_timings(rep):
    rep = dict(rep)
    rep.pop("timings_ms", None)
    if "cells" in rep:
        rep["cells"] = [{k: v for k, v in c.items() if k != "timings_ms"} for c in rep["cells"]]
    return rep


# ============================================================================ CPU (no device call)
def test_usage_errors_exit_1(cli):  # test_cli.cpp:272-277
    for args in ["", "discover", "sweep --gen vertical", "frobnicate",
                 "discover --gen vertical --method nonsense", "discover --gen heavy-tail",
                 "select --topk notanumber", "attend --alpha", "gen --gen vertical",
                 "sweep --gen vertical --alphas 0.1 --bogus 1", "discover --format xml"]:
        code, _, err = run(cli, args)
        assert code == 1, (args, code, err)
        assert "usage error" in err


def test_help_exits_0(cli):
    code, out, _ = run(cli, "--help")
    assert code == 0 and "discover" in out


def test_malformed_container_exits_3(cli, tmp_path):  # test_cli.cpp:292-300
    g = tmp_path / "garbage.fpt"
    g.write_bytes(b"not a tensor container")
    code, _, err = run(cli, f"discover --q {g} --k {g}")
    assert code == 3 and "format error" in err


def test_missing_input_exits_3_and_writes_nothing(cli, tmp_path):  # test_cli.cpp:117-124
    prefix = tmp_path / "missing_out"
    code, _, err = run(cli, f"discover --q /nonexistent/q.fpt --k /nonexistent/k.fpt --out {prefix}")
    assert code == 3 and err
    assert not os.path.exists(f"{prefix}.score.fpt") and not os.path.exists(f"{prefix}.report.json")


def test_container_format_errors(cli, tmp_path):
    """tensor.hpp load_tensor rejections: each malformed variant exits 3, non-finite exits 2."""
    good = tmp_path / "good.fpt"
    write_fpt(good, np.ones((1, 1, 8, 4), np.float32))
    raw = good.read_bytes()
    cases = {
        "badmagic": b"FPT2" + raw[4:],
        "version": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "ndim0": raw[:8] + (0).to_bytes(4, "little") + raw[12:],
        "ndim9": raw[:8] + (9).to_bytes(4, "little") + raw[12:],
        "zerodim": raw[:12] + (0).to_bytes(8, "little") + raw[20:],
        "dtype": raw[:44] + (1).to_bytes(4, "little") + raw[48:],
        "truncated": raw[:-4],
        "trailing": raw + b"\0",
        "header_only": raw[:10],
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.fpt"
        p.write_bytes(blob)
        code, _, err = run(cli, f"discover --q {p} --k {good}")
        assert code == 3, (name, code, err)
    nan = tmp_path / "nan.fpt"
    a = np.ones((1, 1, 8, 4), np.float32)
    a[0, 0, 3, 1] = np.nan
    write_fpt(nan, a)
    code, _, err = run(cli, f"discover --q {nan} --k {good}")
    assert code == 2 and "non-finite" in err


def test_shape_mismatch_exits_2(cli, tmp_path):  # test_cli.cpp:279-290
    rng = np.random.default_rng(13)
    write_fpt(tmp_path / "mis.q.fpt", rng.standard_normal((1, 1, 8, 4)).astype(np.float32))
    write_fpt(tmp_path / "mis.k.fpt", rng.standard_normal((1, 1, 16, 4)).astype(np.float32))
    code, _, err = run(cli, f"discover --q {tmp_path}/mis.q.fpt --k {tmp_path}/mis.k.fpt -B 4")
    assert code == 2 and "validation error" in err


def test_fpt_writer_matches_reference_bytes(tmp_path):
    z = np.load(os.path.join(GOLD, "cli.npz"))
    for name in ("f32", "i32"):
        p = tmp_path / f"{name}.fpt"
        write_fpt(p, z[f"fpt_{name}_array"])
        assert p.read_bytes() == z[f"fpt_{name}_bytes"].tobytes()
        np.testing.assert_array_equal(read_fpt(p), z[f"fpt_{name}_array"])


GEN_CASES = [  # golden planted cases (tests/golden/gen_golden.py): name, pattern, target
    ("vertical_L1000_d32", "vertical", "3"),
    ("slash_L2048_d32", "slash", "300"),
    ("block_L777_B64_d16", "block", "9,4"),
    ("needle_L1500_d32", "needle", "1234"),
]


@pytest.mark.parametrize("name,pattern,target", GEN_CASES)
def test_gen_matches_reference_generator(cli, port, tmp_path, name, pattern, target):
    """`gen` reproduces the reference generate_planted bit-for-bit (golden gt + port oracle q/k/v)."""
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    kind, strength, a, b, noise, seed, Z, H, L, d, B, _ = z["params"]
    prefix = tmp_path / "w"
    code, out, err = run(cli, f"gen --gen {pattern} --target {target} --strength {strength} "
                              f"--noise {noise} --seed {int(seed)} --Z {int(Z)} --H {int(H)} "
                              f"--L {int(L)} --d {int(d)} -B {int(B)} --out {prefix}")
    assert code == 0, err
    rep = json.loads(out)
    assert rep["command"] == "gen" and rep["shape"] == {"Z": Z, "H": H, "L": L, "d": d}
    assert rep["config"]["rng_seed"] == seed
    q, k, v = (read_fpt(f"{prefix}.{t}.fpt") for t in "qkv")
    gt = read_fpt(f"{prefix}.gt.fpt")
    np.testing.assert_array_equal(gt, z["gt"].astype(np.int32))
    sums = [x.astype(np.float64).sum() for x in (q, k, v)]
    np.testing.assert_array_equal(np.array(sums), z["q_sum"])
    rq, rk, rv, _ = port.generate_planted(int(kind), float(strength), int(a), int(b), float(noise),
                                          int(seed), int(Z), int(H), int(L), int(d), int(B))
    for x, y in ((q, rq), (k, rk), (v, rv)):
        np.testing.assert_array_equal(x, y)
    # the report file equals stdout
    assert open(f"{prefix}.report.json").read() == out


def test_gen_alt_slash_matches_reference(cli, tmp_path):
    z = np.load(os.path.join(GOLD, "cli.npz"))
    s, off, noise, seed, Z, H, L, d, B = z["alt_params"]
    prefix = tmp_path / "alt"
    code, _, err = run(cli, f"gen --gen alt-slash --target {int(off)} --strength {s} --noise {noise} "
                            f"--seed {int(seed)} --Z {int(Z)} --H {int(H)} --L {int(L)} --d {int(d)} "
                            f"-B {int(B)} --out {prefix}")
    assert code == 0, err
    for t in "qkv":
        np.testing.assert_array_equal(read_fpt(f"{prefix}.{t}.fpt"), z[f"alt_{t}"])
    np.testing.assert_array_equal(read_fpt(f"{prefix}.gt.fpt"), z["alt_gt"].astype(np.int32))


def test_gen_default_targets_and_config_hash(cli, tmp_path):
    """Default targets (bsattn_main.cpp:105-137) and the config echo / FNV-1a hash (report.hpp)."""
    code, out, _ = run(cli, f"gen --gen block --L 1024 -B 128 --d 8 --out {tmp_path}/b")
    assert code == 0
    gt = read_fpt(f"{tmp_path}/b.gt.fpt")[0, :, :, 0]
    off_diag = [(i, j) for i, j in zip(*np.nonzero(gt)) if i != j]
    assert off_diag == [(4, 2)]  # (M/2, M/4) with M = 8
    rep = json.loads(out)
    echo = json.dumps(rep["config"], separators=(",", ":"))
    h = 0xcbf29ce484222325
    for c in echo.encode():
        h = ((h ^ c) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert rep["config_hash"] == f"{h:016x}"
    assert list(rep["config"]) == ["block_size", "alpha", "sink_tokens", "window_tokens", "scale",
                                   "epsilon", "rng_seed"]


# ============================================================================ GPU
@pytest.mark.gpu
def test_discover_generated_workload_report(cli, fp, port, tmp_path):  # test_cli.cpp:90-105
    prefix = tmp_path / "disc"
    code, out, err = run(cli, f"discover --gen vertical --L 2048 --B 128 --seed 7 --out {prefix}")
    assert code == 0, err
    rep = json.loads(out)
    assert rep["command"] == "discover" and rep["method"] == "approx"
    assert rep["metrics"]["recall"] >= 0.95
    assert rep["config"]["rng_seed"] == 7
    assert os.path.exists(f"{prefix}.report.json")
    score = read_fpt(f"{prefix}.score.fpt")
    assert score.ndim == 4 and score.shape[2] == 16
    # parity: the same workload through the oracle
    q, k, _, _ = port.generate_planted(0, 2.5, 4, 0, 0.5, 7, 1, 1, 2048, 64, 128,
                                       float(1 / np.sqrt(np.float32(64))))
    en, lm, sc = port.discover(q, k, 128, float(1 / np.sqrt(np.float32(64))))
    np.testing.assert_array_equal(read_fpt(f"{prefix}.localmax.fpt"), lm)
    np.testing.assert_allclose(read_fpt(f"{prefix}.energy.fpt"), en, rtol=1e-5, atol=0)
    np.testing.assert_allclose(score, sc, rtol=1e-5, atol=1e-7)


@pytest.mark.gpu
def test_discover_methods_dispatch(cli, fp, tmp_path):  # test_cli.cpp:107-115
    for method in ("approx", "pool-both", "exact"):
        code, out, err = run(cli, f"discover --gen vertical --L 512 --B 64 --d 32 --seed 1 "
                                  f"--method {method} --compare-exact")
        assert code == 0, err
        rep = json.loads(out)
        assert rep["method"] == method
        if method != "exact":
            assert rep["metrics"]["rank_corr_exact"] > 0.0


@pytest.mark.gpu
def test_attend_check_alpha0_matches_dense(cli, fp):  # test_cli.cpp:126-136
    code, out, err = run(cli, "attend --gen slash --L 512 --B 64 --d 32 --seed 9 --check --alpha 0 "
                              "--sink-tokens 0 --window-tokens 1")
    assert code == 0, err
    m = json.loads(out)["metrics"]
    assert m["density"] == 1.0
    assert m["err_max_abs"] <= 1e-4 and m["lse_err_max_abs"] <= 1e-4
    assert m["block_visits"] == m["visit_count"]


@pytest.mark.gpu
def test_attend_dense_single_token_returns_value(cli, fp, tmp_path):  # test_cli.cpp:138-158
    rng = np.random.default_rng(11)
    for t in "qkv":
        write_fpt(tmp_path / f"one.{t}.fpt", rng.standard_normal((1, 1, 1, 4)).astype(np.float32))
    code, _, err = run(cli, f"attend --dense --q {tmp_path}/one.q.fpt --k {tmp_path}/one.k.fpt "
                            f"--v {tmp_path}/one.v.fpt -B 64 --out {tmp_path}/one_out")
    assert code == 0, err
    np.testing.assert_allclose(read_fpt(f"{tmp_path}/one_out.out.fpt")[0, 0, 0],
                               read_fpt(f"{tmp_path}/one.v.fpt")[0, 0, 0], rtol=1e-5)


@pytest.mark.gpu
def test_corrupted_plan_exits_2(cli, fp, port, tmp_path):  # test_cli.cpp:160-181
    M = 4
    idx, counts = port.full_causal_plan(1, 1, M)
    idx[0, 1, 0, 0] = M  # the fill value inside the valid prefix
    write_fpt(tmp_path / "bad.idx.fpt", idx)
    write_fpt(tmp_path / "bad.cnt.fpt", counts)
    q, k, v, _ = port.generate_planted(0, 0.0, 0, 0, 1.0, 2, 1, 1, 256, 8, 64)
    for t, x in zip("qkv", (q, k, v)):
        write_fpt(tmp_path / f"bad.{t}.fpt", x)
    code, _, err = run(cli, f"attend --q {tmp_path}/bad.q.fpt --k {tmp_path}/bad.k.fpt "
                            f"--v {tmp_path}/bad.v.fpt -B 64 --plan {tmp_path}/bad")
    assert code == 2 and "plan" in err


@pytest.mark.gpu
def test_sweep_density_monotone(cli, fp):  # test_cli.cpp:183-197
    code, out, err = run(cli, "sweep --gen vertical --L 1024 --B 128 --d 32 --seed 4 --sink-tokens 0 "
                              "--window-tokens 1 --alphas 0,0.05,0.12,0.5,1")
    assert code == 0, err
    cells = json.loads(out)["cells"]
    assert len(cells) == 5
    dens = [c["density"] for c in cells]
    assert all(b <= a + 1e-12 for a, b in zip(dens, dens[1:]))
    assert dens[0] == 1.0
    assert cells[0]["err_max_abs"] <= 1e-4  # alpha 0 == dense


@pytest.mark.gpu
def test_heavy_tail_sweep(cli, fp, port):  # test_cli.cpp:199-217
    code, out, err = run(cli, "sweep --gen heavy-tail --L 8192 --B 128 --seed 6 --sink-tokens 0 "
                              "--window-tokens 1 --alphas 0.2 --topks 8 --topps 0.9")
    assert code == 0, err
    cells = {c["method"]: c for c in json.loads(out)["cells"]}
    assert len(cells) == 3
    assert cells["max"]["head_retention"] == 1.0
    assert cells["max"]["density"] < cells["topk"]["density"]
    assert cells["max"]["density"] < cells["topp"]["density"]
    # parity: the same selectors on the reference's own heavy-tail map (golden) through the oracle
    z = np.load(os.path.join(GOLD, "cli.npz"))
    score = z["heavy_score"]
    M = score.shape[2]
    mask, _ = port.max_threshold_mask(score, 128, 0.2, 0, 1)
    _, cnt = port.compress_indices(mask)
    assert cells["max"]["visit_count"] == port.visit_count(cnt)
    for method, param in (("topk", 8), ("topp", 0.9)):
        m2 = port.sort_select(score, method, param, 128, 0, 1)
        _, c2 = port.compress_indices(m2)
        assert cells[method]["visit_count"] == port.visit_count(c2), method
        assert cells[method]["density"] == pytest.approx(port.density(c2, M), abs=0)


@pytest.mark.gpu
def test_reports_deterministic(cli, fp):  # test_cli.cpp:219-226
    args = "discover --gen block --L 512 --B 64 --d 16 --seed 12"
    r1, r2 = run(cli, args), run(cli, args)
    assert r1[0] == 0 and r2[0] == 0
    assert strip_timings(json.loads(r1[1])) == strip_timings(json.loads(r2[1]))


@pytest.mark.gpu
def test_json_csv_agree(cli, fp, tmp_path):  # test_cli.cpp:228-256
    args = "sweep --gen vertical --L 512 --B 64 --d 16 --seed 3 --alphas 0.05,0.2 --topks 4"
    cj, oj, ej = run(cli, args + " --format json")
    cc, oc, ec = run(cli, args + f" --format csv --out {tmp_path}/sw")
    assert cj == 0 and cc == 0, ej + ec
    rep = json.loads(oj)
    rows = [ln.split(",") for ln in oc.splitlines() if ln]
    assert len(rows) == len(rep["cells"]) + 1
    hdr = rows[0]
    for r, cell in enumerate(rep["cells"]):
        for col in ("density", "visit_count", "recall"):
            assert rows[r + 1][hdr.index(col)] == json.dumps(cell[col]) or \
                float(rows[r + 1][hdr.index(col)]) == cell[col]
    assert open(f"{tmp_path}/sw.csv").read() == oc


@pytest.mark.gpu
def test_lse_natural(cli, fp, tmp_path):  # test_cli.cpp:258-270
    base = "attend --gen vertical --L 256 --B 64 --d 16 --seed 8 --alpha 0 "
    assert run(cli, base + f"--out {tmp_path}/lse2")[0] == 0
    assert run(cli, base + f"--lse-natural --out {tmp_path}/lsee")[0] == 0
    l2, le = read_fpt(f"{tmp_path}/lse2.lse.fpt"), read_fpt(f"{tmp_path}/lsee.lse.fpt")
    np.testing.assert_allclose(le, l2 * 0.6931471805599453, atol=1e-5, rtol=0)


@pytest.mark.gpu
def test_discover_select_attend_chain_matches_oracle(cli, fp, port, tmp_path):
    """discover -> select -> attend --plan through containers equals the oracle pipeline."""
    name = "slash_L2048_d32"
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    kind, strength, a, b, noise, seed, Z, H, L, d, B, _ = z["params"]
    q, k, v, _ = port.generate_planted(int(kind), float(strength), int(a), int(b), float(noise),
                                       int(seed), int(Z), int(H), int(L), int(d), int(B))
    for t, x in zip("qkv", (q, k, v)):
        write_fpt(tmp_path / f"{t}.fpt", x)
    code, _, err = run(cli, f"discover --q {tmp_path}/q.fpt --k {tmp_path}/k.fpt -B {int(B)} "
                            f"--out {tmp_path}/d")
    assert code == 0, err
    np.testing.assert_allclose(read_fpt(f"{tmp_path}/d.score.fpt"), z["score"], rtol=1e-5, atol=1e-7)
    # select on the REFERENCE score map -> plan must equal the golden plan bit-for-bit
    write_fpt(tmp_path / "ref_score.fpt", z["score"])
    code, out, err = run(cli, f"select --scores {tmp_path}/ref_score.fpt -B {int(B)} --alpha 0.12 "
                              f"--out {tmp_path}/p")
    assert code == 0, err
    rep = json.loads(out)
    assert rep["selector"] == "max"
    assert rep["metrics"]["score_comparisons"] == int(z["cmp_a012"][0])
    np.testing.assert_array_equal(read_fpt(f"{tmp_path}/p.idx.fpt"), z["idx_a012"])
    np.testing.assert_array_equal(read_fpt(f"{tmp_path}/p.cnt.fpt"), z["counts_a012"])
    code, out, err = run(cli, f"attend --q {tmp_path}/q.fpt --k {tmp_path}/k.fpt --v {tmp_path}/v.fpt "
                              f"-B {int(B)} --plan {tmp_path}/p --out {tmp_path}/o")
    assert code == 0, err
    rep = json.loads(out)
    assert rep["metrics"]["block_visits"] == int(z["visits"][0])
    np.testing.assert_allclose(read_fpt(f"{tmp_path}/o.out.fpt"), z["out_sparse"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(read_fpt(f"{tmp_path}/o.lse.fpt"), z["lse_sparse"], atol=1e-5, rtol=0)
    # top-k / top-p selectors on the reference map equal the reference baselines
    for flag, key in (("--topk 4", "topk4"), ("--topp 0.9", "topp09")):
        code, _, err = run(cli, f"select --scores {tmp_path}/ref_score.fpt -B {int(B)} {flag} "
                                f"--out {tmp_path}/s")
        assert code == 0, err
        _, ref_cnt = port.compress_indices(z[key])
        np.testing.assert_array_equal(read_fpt(f"{tmp_path}/s.cnt.fpt"), ref_cnt)
