"""GPU verify suites (acceptance criteria 3-6 and 10) and the
PyTorch binding."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def verify():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_12854_b200 import verify
    return verify


@pytest.mark.parametrize("suite,trials", [("lemma1", 2000), ("scaling", 1000), ("unbiased", 20000),
                                          ("theorem1", 4000), ("monotone", 1000)])
def test_verify_suite(verify, suite, trials):
    rep = verify.SUITES[suite](trials=trials)
    assert rep.passed, rep.csv()


def test_verify_cli_deterministic(verify, capsys):
    assert verify.main(["--suite", "lemma1", "--trials", "500", "--seed", "9"]) == 0
    a = capsys.readouterr().out
    assert verify.main(["--suite", "lemma1", "--trials", "500", "--seed", "9"]) == 0
    assert capsys.readouterr().out == a                      # identical CSV for the same seed


def test_torch_module_regular_matches_dense():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_12854_b200.torch_op import McaSelfAttention
    torch.manual_seed(0)
    m = McaSelfAttention(768, 12, mode="regular").cuda()
    hs = torch.randn(2, 64, 768, device="cuda")
    with torch.no_grad():
        y = m(hs)
        q, k, v = m.query(hs), m.key(hs), m.value(hs)
        sh = lambda t: t.view(2, 64, 12, 64).transpose(1, 2)   # noqa: E731
        att = torch.softmax(sh(q) @ sh(k).transpose(-1, -2) / 8.0, dim=-1)
        ref = (att @ sh(v)).transpose(1, 2).reshape(2, 64, 768)
    assert float((y - ref).norm() / ref.norm()) < 1e-5
    m.mode = "approximation"
    m.alpha = 1e-7                                            # every budget clamps to exact: the regular layer
    with torch.no_grad():
        ye = m(hs)
    assert float((ye - ref).norm() / ref.norm()) < 1e-5
    m.alpha = 0.4                                             # Monte-Carlo layer: Theorem 1's per-row bound
    with torch.no_grad():
        ya = m(hs)
        err = (ya - ref).view(2, 64, 12, 64).norm(dim=3)      # [b, j, h]
        beta = hs.double().norm(dim=2).mean(dim=1)            # per sequence
        wn = m.value.weight.t().double().reshape(768, 12, 64).norm(dim=(0, 2))
        bound = 0.4 * beta[:, None, None] * wn[None, None, :]
    assert bool(torch.isfinite(ya).all()) and bool((err.mean(dim=1) <= bound[:, 0, :]).all())


@pytest.mark.gpu
def test_torch_op_approximation_mode_matches_forward():
    """torch.ops.mca_b200.attention in approximation mode is mca_forward on the
    same tensors (same seed / layer): bitwise equal outputs."""
    import torch
    import paper_2201_12854_b200 as mca
    from paper_2201_12854_b200 import synthetic
    import paper_2201_12854_b200.torch_op  # noqa: F401
    H, n, d_in = 12, 128, 768
    w = synthetic.make_weights(d_in, H, seed=3).to(torch.bfloat16).cuda()
    inp = synthetic.make_inputs(2, n, d_in, H, seed=3)
    q, k, x = (t.to(torch.bfloat16).cuda() for t in (inp.q, inp.k, inp.x))
    y_op = torch.ops.mca_b200.attention(q, k, x, w, H, 0.4, 11, "approximation", 2)
    y_fw = mca.mca_forward(mca.AttentionWeights(w, heads=H), q, k, x, mca.McaConfig(alpha=0.4), seed=11, layer=2).y
    assert torch.equal(y_op, y_fw)


@pytest.mark.gpu
def test_torch_module_stack_uses_each_layers_weights():
    """Two McaSelfAttention layers with different value weights, and one layer
    after an in-place weight update: each call uses its own current W_V (the
    prepared-weight cache never serves another tensor's tables)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_12854_b200.torch_op import McaSelfAttention
    torch.manual_seed(1)
    hs = torch.randn(1, 32, 768, device="cuda")

    def dense(m):
        q, k, v = m.query(hs), m.key(hs), m.value(hs)
        sh = lambda t: t.view(1, 32, 12, 64).transpose(1, 2)   # noqa: E731
        att = torch.softmax(sh(q) @ sh(k).transpose(-1, -2) / 8.0, dim=-1)
        return (att @ sh(v)).transpose(1, 2).reshape(1, 32, 768)

    layers = [McaSelfAttention(768, 12, mode="regular").cuda() for _ in range(2)]
    with torch.no_grad():
        for _ in range(2):                                     # repeated calls alternate between the layers
            for m in layers:
                ref = dense(m)
                assert float((m(hs) - ref).norm() / ref.norm()) < 1e-5
        layers[0].value.weight.mul_(-2.0)                      # in place: same storage, new version
        ref = dense(layers[0])
        assert float((layers[0](hs) - ref).norm() / ref.norm()) < 1e-5
        w_a = torch.randn(768, 768, device="cuda") / 30        # functional op on temporaries of equal size
        w_b = torch.randn(768, 768, device="cuda") / 30
        q = torch.randn(1, 32, 768, device="cuda")
        for w_v in (w_a, w_b):
            y = torch.ops.mca_b200.attention(q, q, hs, w_v.clone(), 12, 1.0, 0, "regular", 0)
            att = torch.softmax(q.view(1, 32, 12, 64).transpose(1, 2) @ q.view(1, 32, 12, 64).transpose(1, 2)
                                .transpose(-1, -2) / 8.0, dim=-1)
            ref = (att @ (hs @ w_v).view(1, 32, 12, 64).transpose(1, 2)).transpose(1, 2).reshape(1, 32, 768)
            assert float((y - ref).norm() / ref.norm()) < 1e-5


@pytest.mark.parametrize("suite", ["lemma1", "scaling", "unbiased", "theorem1", "monotone"])
def test_verify_suite_bert_scale(verify, suite):
    """The same acceptance criteria at BERT-base scale (d_in = 768, 12 heads,
    synthetic BERT-init W_V, sink-model attention), 10^4 seeds per case
    (SURVEY §8(f) #2)."""
    rep = verify.SUITES[suite](scale="bert")
    print(rep.csv())
    assert rep.trials == verify.BERT_TRIALS
    assert rep.passed, rep.csv()
