"""K10 surrogate-loss head (surrogate.py / surrogate.cu) against the
reference's sample_loss_tgat / sample_loss_graphmixer and ad.backward
(golden ``surrogate.npz``, sampler.py:183-250, training.py:409-436).

Tolerances (normwise, max |err| / max |ref|): coefficients 1e-10 in f64
(the TGAT coefficient is a difference of two quotient-rule terms; the
device reassociates <dL/dh, mu> as sum_j tau_j <dL/dh, V_j>), f32 outputs
2e-6 (one f32 rounding of f64-accumulated values); f32 TGAT coefficients are
compared with the reference formula evaluated in f64 on the same inputs
(the reference's own float32 run loses up to a few % to that cancellation).
loss and d loss / d logits: 1e-12 (f64), 2e-6 (f32) given the reference's c."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
TAGS = ["s0_f64", "s1_f64", "s2_f64", "s3_f64", "s0_f32", "s1_f32", "s2_f32", "s3_f32"]


def _g(tag):
    z = load_golden("surrogate")
    return lambda k: z[f"{tag}/{k}"]


def _close(a, b, tol):
    a = a.detach().cpu().double().numpy() if hasattr(a, "detach") else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b).max() if a.size else 0.0
    assert err <= tol * max(np.abs(b).max() if b.size else 0.0, 1e-30), (err, np.abs(b).max())


def _policy(g, agg):
    from paper_2402_05396_b200.sampler import PolicyOutput
    return PolicyOutput(q=g(f"{agg}/q"), log_q=g(f"{agg}/log_q"), mask=g("mask"), selected=g(f"{agg}/selected"),
                        selected_mask=g(f"{agg}/sel_mask"))


@pytest.mark.parametrize("tag", TAGS)
def test_device_tgat_coefficients_and_logits_grad(tag):
    from paper_2402_05396_b200 import surrogate as sur
    g = _g(tag)
    f64 = tag.endswith("f64")
    c = sur.tgat_sample_coefficients(g("dL_dh"), g("tau"), g("V"), g("tgat/sel_mask"), g("contrib"))
    assert str(c.dtype) == ("torch.float64" if f64 else "torch.float32")
    _close(c, g("tgat/c64"), 1e-10 if f64 else 2e-6)
    r = sur.surrogate_grad(g("tgat/c"), _policy(g, "tgat"))
    _close(r.loss, g("tgat/loss"), 1e-12 if f64 else 2e-6)
    _close(r.dlogits, g("tgat/dlogits"), 1e-12 if f64 else 2e-6)


@pytest.mark.parametrize("tag", TAGS)
def test_device_graphmixer_coefficients_and_logits_grad(tag):
    import torch
    from paper_2402_05396_b200 import surrogate as sur
    g = _g(tag)
    f64 = tag.endswith("f64")
    tol = 1e-10 if f64 else 2e-6
    c = sur.graphmixer_message_coefficients(g("dL_dh"), g("msgs"), g("Wc1"), g("Wt1"), g("Wt2"),
                                            g("graphmixer/sel_mask"), g("contrib"))
    _close(c, g("graphmixer/c"), tol)
    # the general form, w' as the Trainer broadcasts it and as a full array
    mu = g("msgs") @ g("Wc1")
    w_row = g("w_row").astype(mu.dtype)
    wp2 = np.ascontiguousarray(np.broadcast_to(w_row[:, None], mu.shape[1:]))
    for wp in (wp2, np.ascontiguousarray(np.broadcast_to(wp2, mu.shape))):
        c = sur.graphmixer_sample_coefficients(g("dL_dh"), wp, mu, g("graphmixer/sel_mask"), g("contrib"))
        _close(c, g("graphmixer/c"), tol if f64 else 2e-5)
    r = sur.sample_loss_graphmixer(g("dL_dh"), torch.as_tensor(wp2).cuda(), mu, _policy(g, "graphmixer"),
                                   sel_mask=g("graphmixer/sel_mask"), contrib_mask=g("contrib"))
    _close(r.loss, g("graphmixer/loss"), 1e-10 if f64 else 2e-5)
    _close(r.dlogits, g("graphmixer/dlogits"), 1e-10 if f64 else 2e-5)


def test_device_tgat_nonpositive_normalizer_raises():
    """FloatingPointError for an active row with lam <= 0 (sampler.py:202-203);
    the same row with contrib False is fine and gets zero coefficients."""
    from paper_2402_05396_b200 import surrogate as sur
    B, n, d = 5, 4, 7
    rng = np.random.default_rng(3)
    tau = np.exp(rng.normal(size=(B, n)))
    tau[3] = 0.0
    args = (rng.normal(size=(B, d)), tau, rng.normal(size=(B, n, d)), np.ones((B, n), bool))
    with pytest.raises(FloatingPointError):
        sur.tgat_sample_coefficients(*args, np.ones(B, bool))
    contrib = np.ones(B, bool)
    contrib[3] = False
    c = sur.tgat_sample_coefficients(*args, contrib)
    assert (c[3] == 0).all() and (c[:3] != 0).any()


def test_device_surrogate_empty_and_no_picks():
    """B = 0 is a no-op with an exact zero loss; rows without picks (or without
    valid slots) get zero coefficients and zero logits gradient."""
    import torch
    from paper_2402_05396_b200 import surrogate as sur
    from paper_2402_05396_b200.sampler import PolicyOutput
    c = sur.tgat_sample_coefficients(np.zeros((0, 3)), np.zeros((0, 2)), np.zeros((0, 2, 3)))
    assert tuple(c.shape) == (0, 2)
    pol = PolicyOutput(q=np.zeros((0, 5)), log_q=np.zeros((0, 5)), mask=np.zeros((0, 5), bool),
                       selected=np.zeros((0, 2), np.int64), selected_mask=np.zeros((0, 2), bool))
    r = sur.surrogate_grad(np.zeros((0, 2)), pol)
    assert float(r.loss) == 0.0 and tuple(r.dlogits.shape) == (0, 5)
    q = np.zeros((2, 5))
    q[1, :2] = 0.5
    pol = PolicyOutput(q=q, log_q=np.where(q > 0, np.log(np.maximum(q, 1e-300)), -1e30), mask=q > 0,
                       selected=np.array([[-1, -1], [1, -1]]), selected_mask=np.array([[False, False], [True, False]]))
    r = sur.surrogate_grad(np.array([[0.0, 0.0], [2.0, 0.0]]), pol)
    assert torch.equal(r.dlogits[0].cpu(), torch.zeros(5, dtype=torch.float64))
    np.testing.assert_allclose(r.dlogits[1].cpu().numpy(), [-1.0, 1.0, 0, 0, 0])
    assert float(r.loss) == pytest.approx(2.0 * np.log(0.5))


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_device_adam_bit_exact_vs_reference(tag):
    """tg_adam_step (one launch for the whole store) equals ParamStore.adam_step
    bit for bit over three steps (golden adam.npz): float64 and float32 stores,
    a float64 gradient on a float32 parameter, a parameter without gradient."""
    import torch
    from paper_2402_05396_b200.optim import AdamState
    z = load_golden("adam")
    keys = ["a", "b", "c", "d"]
    params = {k: torch.as_tensor(z[f"{tag}/init/{k}"].copy()).cuda() for k in keys}
    opt = AdamState(params)
    for s in range(3):
        lr, b1, b2, eps = (float(x) for x in z[f"{tag}/s{s}/hp"])
        grads = {k: (z[f"{tag}/s{s}/g/{k}"] if z[f"{tag}/s{s}/g/{k}"].size else None) for k in keys}
        opt.step(grads, lr, beta1=b1, beta2=b2, eps=eps)
        for k in keys:
            for name, arr in (("p", params[k]), ("m", opt.m[k]), ("v", opt.v[k])):
                ref = z[f"{tag}/s{s}/{name}/{k}"]
                got = arr.cpu().numpy()
                assert got.dtype == ref.dtype and got.tobytes() == ref.tobytes(), (s, k, name)


def test_device_surrogate_large_batch_matches_oracle():
    """More roots than the grid holds (grid-stride paths): B = 5000, f64,
    against the oracle restatement (itself pinned to the reference)."""
    import torch
    from oracle import surrogate as osur
    from paper_2402_05396_b200 import surrogate as sur
    from paper_2402_05396_b200.sampler import PolicyOutput
    rng = np.random.default_rng(11)
    B, m, n, d, dm, ht = 5000, 25, 10, 24, 40, 12
    sel = rng.random((B, n)) < 0.9
    contrib = rng.random(B) < 0.95
    g = rng.normal(size=(B, d))
    tau = np.exp(rng.normal(size=(B, n)))
    V = rng.normal(size=(B, n, d))
    c_ref = osur.tgat_coefficients(g, tau, V, sel, contrib)
    c = sur.tgat_sample_coefficients(g, tau, V, sel, contrib).cpu().numpy()
    assert np.abs(c - c_ref).max() <= 1e-10 * np.abs(c_ref).max()
    msgs = rng.normal(size=(B, n, dm))
    Wc1, Wt1, Wt2 = rng.normal(size=(dm, d)), rng.normal(size=(n, ht)), rng.normal(size=(ht, n))
    c2_ref = osur.graphmixer_from_messages(g, msgs, Wc1, Wt1, Wt2, sel, contrib)
    c2 = sur.graphmixer_message_coefficients(g, msgs, Wc1, Wt1, Wt2, sel, contrib).cpu().numpy()
    assert np.abs(c2 - c2_ref).max() <= 1e-10 * np.abs(c2_ref).max()
    mask = rng.random((B, m)) < 0.8
    logits = rng.normal(size=(B, m))
    e = np.where(mask, np.exp(logits - np.where(mask, logits, -np.inf).max(axis=1, keepdims=True)), 0.0)
    z = e.sum(axis=1, keepdims=True)
    q = np.divide(e, z, out=np.zeros_like(e), where=z > 0)
    log_q = np.where(mask, np.log(np.maximum(q, 1e-300)), -1e30)
    selected = np.stack([rng.permutation(m)[:n] for _ in range(B)])
    sm = sel & np.take_along_axis(mask, selected, axis=1)
    selected = np.where(sm, selected, -1)
    pol = PolicyOutput(q=q, log_q=log_q, mask=mask, selected=selected, selected_mask=sm)
    loss_ref, dl_ref = osur.logq_grad(c_ref, q, log_q, mask, selected, sm)
    r = sur.surrogate_grad(torch.as_tensor(c_ref).cuda(), pol)
    assert abs(float(r.loss) - loss_ref) <= 1e-12 * max(abs(loss_ref), 1.0) * 10
    assert np.abs(r.dlogits.cpu().numpy() - dl_ref).max() <= 1e-12 * np.abs(dl_ref).max()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_device_adam_large_tensors_bit_exact(dtype):
    """Tensors larger than one grid pass (3M elements), several sizes in one
    launch, bit-identical to the numpy update (oracle.surrogate.adam_step)."""
    import torch
    from oracle import surrogate as osur
    from paper_2402_05396_b200.optim import AdamState
    rng = np.random.default_rng(5)
    dt = np.float64 if dtype == "float64" else np.float32
    shapes = {"w": (3_000_001,), "b": (17,), "t": (512, 300)}
    host = {k: rng.normal(size=s).astype(dt) for k, s in shapes.items()}
    m = {k: np.zeros_like(v) for k, v in host.items()}
    v = {k: np.zeros_like(v) for k, v in host.items()}
    params = {k: torch.as_tensor(a.copy()).cuda() for k, a in host.items()}
    opt = AdamState(params)
    for step in range(1, 3):
        grads = {k: (rng.normal(size=s) * 1e-3).astype(dt) for k, s in shapes.items()}
        opt.step(grads, 1e-3)
        for k in shapes:
            osur.adam_step(host[k], grads[k], m[k], v[k], step, 1e-3)
            assert params[k].cpu().numpy().tobytes() == host[k].tobytes(), (step, k)
            assert opt.v[k].cpu().numpy().tobytes() == v[k].tobytes(), (step, k)
