"""Adapter optimizer: the fp64 AdamW oracle pinned to torch.optim.AdamW
(CPU), and the CUDA kernel against the oracle (GPU, fp32 path tolerance 1e-5)."""
import numpy as np
import pytest

from oracle import optim as O

HP = [dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01),
      dict(lr=3e-4, beta1=0.8, beta2=0.99, eps=1e-6, weight_decay=0.0),
      dict(lr=5e-3, beta1=0.95, beta2=0.9999, eps=1e-8, weight_decay=0.1)]


def test_oracle_matches_torch_adamw():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    n = 101
    p0 = rng.standard_normal(n)
    group = rng.integers(0, 3, size=n)
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    params = [torch.tensor(p0[group == k], dtype=torch.float64, requires_grad=True) for k in range(3)]
    opt = torch.optim.AdamW([dict(params=[params[k]], lr=HP[k]["lr"], betas=(HP[k]["beta1"], HP[k]["beta2"]),
                                  eps=HP[k]["eps"], weight_decay=HP[k]["weight_decay"]) for k in range(3)])
    for step in range(1, 6):
        g = rng.standard_normal(n)
        p, m, v = O.adamw_step(p, g, m, v, group, HP, step)
        for k in range(3):
            params[k].grad = torch.tensor(g[group == k], dtype=torch.float64)
        opt.step()
        for k in range(3):
            assert np.allclose(p[group == k], params[k].detach().numpy(), rtol=1e-12, atol=1e-14)


def test_oracle_per_group_step_matches_torch_for_a_late_group():
    """A group that joins after 3 steps (its own torch param group created then) is the
    oracle with hparams[k]["step"] = its own count."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    n = 64
    p0 = rng.standard_normal(n)
    group = (np.arange(n) % 2).astype(np.int64)
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    t0 = torch.tensor(p0[group == 0], dtype=torch.float64, requires_grad=True)
    t1 = torch.tensor(p0[group == 1], dtype=torch.float64, requires_grad=True)
    opt0 = torch.optim.AdamW([t0], lr=1e-3, weight_decay=0.01)
    opt1 = torch.optim.AdamW([t1], lr=1e-3, weight_decay=0.01)
    hp = [dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01) for _ in range(2)]
    for step in range(1, 7):
        g = rng.standard_normal(n)
        if step <= 3:                       # group 1 not trained yet: zero gradient, no step
            g[group == 1] = 0.0
            p, m, v = O.adamw_step(p, g, m, v, group, hp[:1], step)   # group 1 not in hparams
        else:
            hp[1]["step"] = step - 3
            hp[0]["step"] = step
            p, m, v = O.adamw_step(p, g, m, v, group, hp, step)
            t1.grad = torch.tensor(g[group == 1], dtype=torch.float64)
            opt1.step()
        t0.grad = torch.tensor(g[group == 0], dtype=torch.float64)
        opt0.step()
        assert np.allclose(p[group == 0], t0.detach().numpy(), rtol=1e-12, atol=1e-14)
        assert np.allclose(p[group == 1], t1.detach().numpy(), rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_gpu_adamw_matches_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(1)
    n = 1_000_003                       # ragged tail beyond the float4 body
    p0 = rng.standard_normal(n).astype(np.float32)
    group = rng.integers(0, 3, size=n).astype(np.uint8)
    P = torch.from_numpy(p0.copy()).to(dev)
    M = torch.zeros(n, device=dev)
    V = torch.zeros(n, device=dev)
    Gi = torch.from_numpy(group).to(dev)
    Pb = torch.empty(n, dtype=torch.bfloat16, device=dev)
    p, m, v = p0.astype(np.float64), np.zeros(n), np.zeros(n)
    for step in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32)
        _lib.lobra_adamw_step(P, torch.from_numpy(g).to(dev), M, V, HP, step, group=Gi, params_bf16=Pb,
                              grad_scale=0.5)
        p, m, v = O.adamw_step(p, g, m, v, group, HP, step, grad_scale=0.5)
        # feed the oracle the GPU's fp32 state rounding-free: compare per step
        torch.cuda.synchronize()
        got = P.cpu().numpy().astype(np.float64)
        assert np.max(np.abs(got - p)) / np.max(np.abs(p)) < 1e-5
        assert np.max(np.abs(M.cpu().numpy() - m)) / np.max(np.abs(m)) < 1e-5
        assert torch.equal(Pb.cpu(), P.cpu().to(torch.bfloat16))
