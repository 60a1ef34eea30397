"""Sampler backward on the device: the scoring
network's parameter gradients from d loss / d logits, against the
reference's own ad.backward (golden sampler_grad.npz, made by
tests/golden/make_golden.py from tgadapt: forward -> WOR -> surrogate loss
sum(c * selected_log_q) -> backward).

Tolerances: f64 (the reference's default precision) <= 1e-10 normwise per
parameter; f32 <= 2e-4 normwise against the same f64 reference gradients
(the f32 path's own rounding, ~1e-6 per op through a d=325 mixer)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

CASES = [f"g{i}" for i in range(8)]


def _case(z, tag, precision="float64"):
    import torch
    from paper_2402_05396_b200.params import ScoringModel, sampler_params
    d_v, d_e, enc, m, B, store_seed, n = (int(x) for x in z[f"{tag}/meta"])
    dec = str(z[f"{tag}/decoder"])
    alpha, beta, _ = (float(x) for x in z[f"{tag}/ab"])
    params = sampler_params(store_seed, enc, m, d_v, d_e, dec)
    for k in z.files:
        if k.startswith(f"{tag}/param/"):
            params[k[len(tag) + 7:]] = z[k]
    model = ScoringModel(params, dec, enc, m, d_v, d_e, alpha, beta, precision=precision)
    dev = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)  # noqa: E731
    inp = {"ids": dev(z[f"{tag}/ids"], torch.int64), "dts": dev(z[f"{tag}/dts"], torch.float64),
           "mask": dev(z[f"{tag}/mask"], torch.bool)}
    if d_v:
        inp["node_rows"] = dev(z[f"{tag}/node_rows"], torch.float32)
        inp["tgt_rows"] = dev(z[f"{tag}/tgt_rows"], torch.float32)
    if d_e:
        inp["edge_rows"] = dev(z[f"{tag}/edge_rows"], torch.float32)
    grads = {k[len(tag) + 6:]: z[k] for k in z.files if k.startswith(f"{tag}/grad/")}
    return model, inp, grads, (B, m, n)


def _err(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("tag", CASES)
def test_device_sampler_backward_f64_matches_reference(tag):
    import torch
    from paper_2402_05396_b200.scoring import SamplerGrad, score_policy
    z = load_golden("sampler_grad")
    model, inp, ref, _ = _case(z, tag)
    q, _ = score_policy(model, inp["ids"], inp["dts"], inp["mask"], inp.get("node_rows"), inp.get("edge_rows"),
                        inp.get("tgt_rows"))
    np.testing.assert_allclose(q.cpu().numpy(), z[f"{tag}/q"], rtol=1e-11, atol=1e-14)
    sg = SamplerGrad(model)
    dl = torch.as_tensor(z[f"{tag}/dlogits"]).cuda()
    sg.backward(dlogits=dl, **inp)
    torch.cuda.synchronize()
    assert set(ref) == set(sg.grads), (sorted(ref), sorted(sg.grads))
    for name, g in ref.items():
        got = sg.grad(name).cpu().numpy()
        assert got.shape == g.shape, name
        if not np.any(g):
            assert not np.any(got), f"{name}: reference gradient is zero"
            continue
        assert _err(got, g) <= 1e-10, (tag, name, _err(got, g))


@pytest.mark.parametrize("tag", ["g0", "g1", "g3", "g7"])
def test_device_sampler_backward_f32_close_to_reference(tag):
    import torch
    from paper_2402_05396_b200.scoring import SamplerGrad
    z = load_golden("sampler_grad")
    model, inp, ref, _ = _case(z, tag, precision="float32")
    sg = SamplerGrad(model)
    sg.backward(dlogits=torch.as_tensor(z[f"{tag}/dlogits"]).cuda().float(), **inp)
    torch.cuda.synchronize()
    for name, g in ref.items():
        if np.any(g):
            got = sg.grad(name).double().cpu().numpy()
            assert _err(got, g) <= 2e-4, (tag, name, _err(got, g))


@pytest.mark.parametrize("tag", ["g1", "g4", "g5"])
def test_device_sampler_update_chain(tag):
    """score_policy -> (reference picks, c) -> K10 surrogate_grad -> backward
    accumulated over two layers' worth of calls -> update_sampler (device
    Adam): gradients are 2x the reference's, the parameters move exactly as
    ParamStore.adam_step moves them for those gradients."""
    import torch
    from paper_2402_05396_b200.optim import AdamState
    from paper_2402_05396_b200.sampler import PolicyOutput
    from paper_2402_05396_b200.scoring import SamplerGrad, score_policy, update_sampler
    from paper_2402_05396_b200.surrogate import surrogate_grad
    z = load_golden("sampler_grad")
    model, inp, ref, (B, m, n) = _case(z, tag)
    q, lq = score_policy(model, inp["ids"], inp["dts"], inp["mask"], inp.get("node_rows"), inp.get("edge_rows"),
                         inp.get("tgt_rows"))
    pol = PolicyOutput(q=q, log_q=lq, mask=inp["mask"], selected=torch.as_tensor(z[f"{tag}/selected"]).cuda(),
                       selected_mask=torch.as_tensor(z[f"{tag}/sel_mask"]).cuda())
    sgr = surrogate_grad(torch.as_tensor(z[f"{tag}/c"]).cuda(), pol)
    np.testing.assert_allclose(sgr.dlogits.cpu().numpy(), z[f"{tag}/dlogits"], rtol=1e-11, atol=1e-13)
    sg = SamplerGrad(model)
    before = {k: v.clone() for k, v in model.named_params().items()}
    adam = AdamState(model.named_params())
    for _ in range(2):  # two adaptive layers' terms of one surrogate loss
        sg.backward(dlogits=sgr.dlogits, **inp)
    torch.cuda.synchronize()
    for name, g in ref.items():
        if np.any(g):
            assert _err(sg.grad(name).cpu().numpy(), 2 * g) <= 1e-10, name
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    update_sampler(sg, adam, lr)
    torch.cuda.synchronize()
    for name, p0 in before.items():
        g = 2 * ref[name].reshape(-1)
        mm, vv = (1 - b1) * g, (1 - b2) * g * g
        exp = p0.cpu().numpy() - lr * (mm / (1 - b1)) / (np.sqrt(vv / (1 - b2)) + eps)
        got = model.named_params()[name].cpu().numpy()
        np.testing.assert_allclose(got, exp, rtol=0, atol=1e-9, err_msg=name)
    assert all(not torch.any(g) for g in sg.grads.values())


def test_device_sampler_backward_validation():
    import torch
    from paper_2402_05396_b200.scoring import SamplerGrad
    z = load_golden("sampler_grad")
    model, inp, _, (B, m, _) = _case(z, "g0")
    sg = SamplerGrad(model)
    with pytest.raises(ValueError):
        sg.backward(dlogits=torch.zeros((B, m + 1), dtype=torch.float64, device="cuda"), **inp)
    empty = {k: v[:0] for k, v in inp.items()}
    sg.backward(dlogits=torch.zeros((0, m), dtype=torch.float64, device="cuda"), **empty)
    assert all(not torch.any(g) for g in sg.grads.values())
