"""The cli module's file plumbing and its GPU bench:
MCAM bit-exact round trips (Python and the C++ header), the format / domain
error contract, cmd_attn_import, and cmd_bench over mca_forward_attn (the
layer on a given attention matrix) checked against the fp64 oracle."""
import os
import struct
import subprocess
import warnings

import numpy as np
import pytest

from paper_2201_12854_b200 import cli, mcam

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------- MCAM (CPU)
def test_mcam_layout_is_bit_exact(tmp_path):
    m = np.random.default_rng(0).standard_normal((8, 8))
    p = str(tmp_path / "m.mcam")
    mcam.write_mcam(p, m)
    raw = open(p, "rb").read()
    assert raw == b"MCAM" + struct.pack("<IQQ", 1, 8, 8) + m.astype("<f8").tobytes()
    back = mcam.read_mcam(p)
    assert back.tobytes() == m.tobytes()


def test_mcam_errors(tmp_path):
    p = str(tmp_path / "m.mcam")
    full = mcam.encode_mcam(np.eye(3))
    open(p, "wb").write(full[:-5])                        # truncated payload: expected vs actual
    with pytest.raises(mcam.FormatError, match=f"expected {len(full)} bytes .* got {len(full) - 5}"):
        mcam.read_mcam(p)
    with pytest.raises(mcam.FormatError) as e:
        mcam.decode_mcam(b"MCAX" + full[4:])
    assert e.value.offset == 0
    with pytest.raises(mcam.FormatError) as e:
        mcam.decode_mcam(full[:4] + struct.pack("<I", 2) + full[8:])
    assert e.value.offset == 4
    bad = bytearray(full)
    bad[24 + 8 * 4: 24 + 8 * 5] = struct.pack("<d", float("nan"))
    with pytest.raises(mcam.FormatError) as e:
        mcam.decode_mcam(bytes(bad))
    assert e.value.offset == 24 + 8 * 4


def test_csv_import_and_attention_checks(tmp_path):
    p = tmp_path / "i2.csv"
    p.write_text("1,0\n0,1\n")
    assert np.array_equal(mcam.attn_import(str(p), "csv"), np.eye(2))
    p.write_text("1,0\n0,1,0\n")
    with pytest.raises(mcam.FormatError, match="ragged"):
        mcam.read_csv(str(p))
    p.write_text("1,x\n")
    with pytest.raises(mcam.FormatError, match="not a number"):
        mcam.read_csv(str(p))
    p.write_text("0.5,-0.5\n0,1\n")
    with pytest.raises(mcam.DomainError):
        mcam.attn_import(str(p), "csv")
    p.write_text("2,2\n0,1\n")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        a = mcam.attn_import(str(p), "csv")                                            # renormalised
    assert w and np.allclose(a.sum(axis=1), 1.0) and np.allclose(a[0], [0.5, 0.5])


def test_cpp_header_round_trip(tmp_path):
    exe = str(tmp_path / "mcam_roundtrip")
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "mcam_roundtrip.cpp"), "-o", exe], check=True)
    a, b = str(tmp_path / "a.mcam"), str(tmp_path / "b.mcam")
    mcam.write_mcam(a, np.abs(np.random.default_rng(3).standard_normal((5, 7))))
    r = subprocess.run([exe, a, b], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.split() == ["5", "7"]
    assert open(a, "rb").read() == open(b, "rb").read()                                # C++ <-> Python bitwise
    open(a, "wb").write(mcam.encode_mcam(np.eye(2))[:30])
    r = subprocess.run([exe, a, b], capture_output=True, text=True)
    assert r.returncode == 2 and "format_error offset=30" in r.stdout and "expected 56 bytes" in r.stdout
    mcam.write_mcam(a, np.array([[1.0, -0.1], [0.0, 1.0]]))
    r = subprocess.run([exe, a, b], capture_output=True, text=True)
    assert r.returncode == 2 and r.stdout.startswith("domain_error")


def test_cli_import_exit_codes(tmp_path, capsys):
    p = tmp_path / "i2.csv"
    p.write_text("1,0\n0,1\n")
    out = str(tmp_path / "i2.mcam")
    assert cli.main(["import", "--input", str(p), "--format", "csv", "--out", out]) == 0
    assert np.array_equal(mcam.read_mcam(out), np.eye(2))
    assert "2,2,1,1" in capsys.readouterr().out
    p.write_text("1,-1\n0,1\n")
    assert cli.main(["import", "--input", str(p), "--format", "csv"]) == 2
    assert cli.main(["import", "--input", str(tmp_path / "missing.mcam")]) == 2
    assert cli.main(["bench", "--alpha", "1.5"]) == 2
    assert cli.main(["bench", "--dims", "bogus"]) == 2


def test_synthetic_attention_generators():
    for kind in ("uniform", "peaked", "gaussian"):
        a = cli.synthetic_attention(kind, 32, seed=1)
        assert a.shape == (32, 32) and np.all(a >= 0) and np.allclose(a.sum(axis=1), 1.0, atol=1e-12)
    assert np.array_equal(cli.synthetic_attention("gaussian", 16, 5), cli.synthetic_attention("gaussian", 16, 5))
    p = cli.synthetic_attention("peaked", 32, 0, eps=0.1)
    assert np.allclose(p[:, 0], 0.9)


# ------------------------------------------------------- the GPU bench path
def _oracle_given_attn(orc, attn, x, w, heads, alpha, seed, mode="approx"):
    """attention module composition on a given A per head:
    Eq. 9 from A's column maxima, approx_encode_row / exact rows, A . H~."""
    n, d = x.shape
    ys, budgets = [], []
    for h in range(heads):
        wh = w[:, 64 * h: 64 * h + 64]
        dist = orc.weight_probs(wh)
        b, e = orc.sample_budgets(attn, alpha, d)
        if mode == "regular":
            e = np.ones_like(e, dtype=bool)
        hh = np.empty((n, 64))
        for j in range(n):
            hh[j] = x[j] @ wh if e[j] else orc.approx_encode_row(x[j], wh, dist, int(b[j]), seed, h * n + j, 0)
        ys.append(attn @ hh)
        budgets.append(np.where(e, d, b))
    return np.concatenate(ys, axis=1), np.stack(budgets)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gaussian", "peaked", "uniform"])
def test_forward_given_attention_matches_oracle(orc, kind):
    import torch
    from paper_2201_12854_b200 import api
    n, d, heads, seed = 40, 128, 2, 9
    attn = cli.synthetic_attention(kind, n, seed=3, temperature=0.3)
    x, w = cli.synthetic_inputs(n, d, heads, seed)
    weights = api.AttentionWeights(torch.from_numpy(w).float().cuda(), heads=heads)
    xt = torch.from_numpy(x).float().cuda()[None]
    at = torch.from_numpy(attn).cuda()[None, None].expand(1, heads, n, n).contiguous()
    xf, wf = x.astype(np.float32).astype(np.float64), w.astype(np.float32).astype(np.float64)
    for alpha in (0.2, 1.0):
        out = api.forward_given_attention(weights, at, xt, api.McaConfig(alpha=alpha), seed=seed, return_plan=True,
                                          flops=True)
        ref_y, ref_b = _oracle_given_attn(orc, attn, xf, wf, heads, alpha, seed)
        assert np.array_equal(out.budgets[0].cpu().numpy(), ref_b)                      # Eq. 9 bitwise
        got = out.y[0].double().cpu().numpy()
        rel = np.linalg.norm(got - ref_y, axis=1) / np.maximum(np.linalg.norm(ref_y, axis=1), 1e-30)
        assert rel.max() <= 1e-5
        assert out.flops.samples == int(out.budgets[out.exact_mask == 0].sum())
    reg = api.forward_given_attention(weights, at, xt, api.McaConfig(mode="regular"), seed=seed, flops=True)
    exact = attn @ (xf @ wf)
    assert np.abs(reg.y[0].double().cpu().numpy() - exact).max() <= 1e-5 * np.abs(exact).max()
    assert reg.flops.reduction_factor == 1.0


@pytest.mark.gpu
def test_forward_given_attention_bf16(orc):
    """bf16 inputs (fp16 H~, bf16 y) on a given attention matrix: budgets
    bitwise (the dump is fp64 either way), y within the bf16 tolerance."""
    import torch
    from paper_2201_12854_b200 import api
    n, d, heads, seed = 64, 256, 4, 2
    attn = cli.synthetic_attention("gaussian", n, seed=8, temperature=0.25)
    x, w = cli.synthetic_inputs(n, d, heads, seed)
    weights = api.AttentionWeights(torch.from_numpy(w).to(torch.bfloat16).cuda(), heads=heads)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()[None]
    at = torch.from_numpy(attn).cuda()[None, None].expand(1, heads, n, n).contiguous()
    xf = xt[0].double().cpu().numpy()
    wf = torch.from_numpy(w).to(torch.bfloat16).double().numpy()
    out = api.forward_given_attention(weights, at, xt, api.McaConfig(alpha=0.3), seed=seed, return_plan=True)
    ref_y, ref_b = _oracle_given_attn(orc, attn, xf, wf, heads, 0.3, seed)
    assert np.array_equal(out.budgets[0].cpu().numpy(), ref_b)
    got = out.y[0].double().cpu().numpy()
    rel = np.linalg.norm(got - ref_y, axis=1) / np.maximum(np.linalg.norm(ref_y, axis=1), 1e-30)
    assert rel.max() <= 2e-2


@pytest.mark.gpu
def test_cli_bench_csv(capsys, tmp_path):
    # uniform attention, alpha = 1: every budget is 1, so the reduction is
    # 2 d_in d_h / (2 d_h + 3) exactly (SPEC.md:458 with d_h = 64 heads)
    assert cli.main(["bench", "--synthetic", "uniform", "--alpha", "1.0", "--dims", "32x128", "--seed", "4"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "alpha,n,d,reduction_factor,total_reduction,mean_row_error,max_row_error"
    f = rows[1].split(",")
    assert float(f[3]) == pytest.approx(2 * 128 * 64 / (2 * 64 + 3), rel=1e-9)
    # regular mode: reduction 1, error 0
    assert cli.main(["bench", "--synthetic", "gaussian", "--mode", "regular", "--alpha", "0.4", "--seed", "4"]) == 0
    f = capsys.readouterr().out.strip().splitlines()[1].split(",")
    assert float(f[3]) == 1.0 and float(f[5]) == 0.0 and float(f[6]) == 0.0
    # a sink-column (CoLA-like) dump beats a uniform (RTE-like) one at equal alpha
    p = str(tmp_path / "peaked.mcam")
    mcam.write_mcam(p, cli.synthetic_attention("peaked", 32, 0))
    assert cli.main(["bench", "--input", p, "--alpha", "0.4", "--seed", "4"]) == 0
    peaked = float(capsys.readouterr().out.strip().splitlines()[1].split(",")[3])
    assert cli.main(["bench", "--synthetic", "uniform", "--alpha", "0.4", "--dims", "32x128", "--seed", "4"]) == 0
    uniform = float(capsys.readouterr().out.strip().splitlines()[1].split(",")[3])
    assert peaked > uniform
    # determinism: same seed, byte-identical CSV
    cli.main(["bench", "--synthetic", "gaussian", "--alpha", "0.2,0.6", "--seed", "7"])
    a = capsys.readouterr().out
    cli.main(["bench", "--synthetic", "gaussian", "--alpha", "0.2,0.6", "--seed", "7"])
    assert capsys.readouterr().out == a
