"""GPU: one Llama decoder layer's fine-tuning step (paper_2509_01193_b200/
decoder.py) against the fp64 oracle (oracle/decoder.py) on the same bf16 parameters and
inputs: Y, dX and every projection's per-task dA / dB.

Tolerance (reading Q27): the GPU layer rounds ~12 intermediate tensors to bf16
(h1, q/k/v after RoPE, the attention output, o, x2, h2, gate/up, act, down, and in the
backward their gradients) and FlashAttention rounds its probabilities to bf16 before
P V; each rounding contributes <= 2^-9 relative to its tensor, ~12 * 2^-9 ~ 2.3e-2 end
to end; the test uses 3e-2.  That bound assumes O(1) attention logits: softmax amplifies
a relative error e of q, k into an absolute logit error e |q||k| / sqrt(D).  The input
recipe therefore scales the adapters' B_t to N(0, 1/(16 r_t)) (logit std ~2, the spread
of a trained model); with B_t ~ N(0, 1/r_t) the logits reach std 5 / max 36 and the bf16
rounding of q, k alone moves outputs by several percent (measured: attention on the
GPU's own bf16 q / k / v still agrees with the oracle to 0.3%; tools/debug_decoder.py).
The attention stage is also checked on its own inputs (test_attention_stage_*).
"""
import numpy as np
import pytest

from oracle import decoder as Dd
from oracle import lora as O

pytestmark = pytest.mark.gpu
TOL = 3e-2

SMALL = [("q", 256, 256, "col", "attn"), ("k", 256, 256, "col", "attn"), ("v", 256, 256, "col", "attn"),
         ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
         ("down", 512, 256, "row", "down_in")]


# grouped-query attention (Llama-2-70B style): 4 query heads of 64, 2 kv heads (k, v: 256 -> 128)
SMALL_GQA = [("q", 256, 256, "col", "attn"), ("k", 256, 128, "col", "attn"), ("v", 256, 128, "col", "attn"),
             ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
             ("down", 512, 256, "row", "down_in")]
ARCH = {"mha": (SMALL, 2), "gqa": (SMALL_GQA, 4)}


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _backend(name):
    if name != "lobra":                                     # "lobra": own tcgen05 forward + backward
        pytest.importorskip(name)
    return name


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _run(group_inputs=True, seed=0, backend="flash_attn", arch="mha"):
    torch = _torch()
    shapes, heads = ARCH[arch]
    from paper_2509_01193_b200.decoder import DecoderLayer
    ranks, scales = [16, 8, 16], [2.0, 0.5, 1.0]
    lens = np.array([1, 300, 57, 129, 200, 33], np.int32)
    tasks = np.array([0, 0, 1, 1, 2, 2], np.int32)
    layer = DecoderLayer(shapes, n_heads=heads, ranks=ranks, scales=scales, seed=seed, group_inputs=group_inputs,
                         deterministic_attn=True, attn_backend=_backend(backend))
    for p in layer.lora.projs:          # B_t ~ N(0, 1/(16 r)): O(1) attention logits (see above)
        p.B.mul_(0.25)
    T = int(lens.sum())
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 1)
    X = torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16)
    dY = torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16)
    Y = layer.forward(lens, tasks, X).clone()
    dX = layer.backward(dY).clone()
    torch.cuda.synchronize()
    return layer, lens, tasks, ranks, scales, X, dY, Y, dX


@pytest.mark.parametrize("arch", ["mha", "gqa"])
@pytest.mark.parametrize("backend", ["cudnn", "flash_attn", "lobra"])
def test_decoder_layer_matches_oracle(backend, arch):
    if backend == "lobra" and arch == "gqa":
        pytest.skip("own attention kernel is head_dim 128; this GQA layer has 64 (GQA at 128: test_gpu_attn)")
    layer, lens, tasks, ranks, scales, X, dY, Y, dX = _run(backend=backend, arch=arch)
    P = {"g_attn": _f64(layer.g_attn), "g_mlp": _f64(layer.g_mlp)}
    for p in layer.lora.projs:
        P[p.name] = (_f64(p.W), _f64(p.A), _f64(p.B))
    cfg = {"n_heads": layer.n_heads, "eps": layer.eps, "theta": layer.theta}
    Yo, cache = Dd.layer_fwd(_f64(X), P, cfg, ranks, scales, lens, tasks)
    dXo, grads = Dd.layer_bwd(_f64(dY), P, cfg, ranks, scales, lens, tasks, cache)
    errs = {"Y": O.max_rel_err(_f64(Y), Yo), "dX": O.max_rel_err(_f64(dX), dXo)}
    fg = layer.lora.flat_grad.cpu().numpy().astype(np.float64)
    R = int(sum(ranks))
    roff = np.concatenate([[0], np.cumsum(ranks)])
    for p in layer.lora.projs:
        dA = fg[p.dA_off:p.dA_off + R * p.d_in].reshape(R, p.d_in)
        dB = fg[p.dB_off:p.dB_off + p.d_out * R].reshape(p.d_out, R)
        for t in range(len(ranks)):
            a, b = roff[t], roff[t + 1]
            errs[f"dA_{p.name}{t}"] = O.max_rel_err(dA[a:b], grads[p.name][0][a:b])
            errs[f"dB_{p.name}{t}"] = O.max_rel_err(dB[:, a:b], grads[p.name][1][:, a:b])
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, f"tolerance {TOL} exceeded: {bad}; all: {errs}"


def test_decoder_layer_grouped_equals_ungrouped():
    """The projection-group path and the per-projection path give the same layer
    (bitwise: deterministic FlashAttention backward, group == single calls)."""
    torch = _torch()
    a = _run(group_inputs=True, seed=3)
    b = _run(group_inputs=False, seed=3)
    assert torch.equal(a[7], b[7]) and torch.equal(a[8], b[8])
    assert torch.equal(a[0].lora.flat_grad, b[0].lora.flat_grad)


@pytest.mark.parametrize("backend", ["cudnn", "flash_attn", "lobra"])
def test_attention_stage_on_its_own_inputs(backend):
    """The library attention inside the layer (forward and backward) against the oracle
    evaluated on the GPU's own bf16 q / k / v / dO: isolates that stage from the rounding
    of its inputs (valid for any logit scale; the layer here uses the unscaled B_t)."""
    torch = _torch()
    from paper_2509_01193_b200.decoder import DecoderLayer
    lens = np.array([1, 300, 57, 129, 200, 33], np.int32)
    tasks = np.array([0, 0, 1, 1, 2, 2], np.int32)
    layer = DecoderLayer(SMALL, n_heads=2, ranks=[16, 8, 16], scales=[2.0, 0.5, 1.0], seed=5,
                         deterministic_attn=True, attn_backend=_backend(backend))
    T = int(lens.sum())
    g = torch.Generator(device="cuda")
    g.manual_seed(6)
    X = torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16)
    dY = torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16)
    layer.forward(lens, tasks, X)
    layer.backward(dY)
    torch.cuda.synchronize()
    c = layer.cache
    view = lambda n: _f64(c[n][:T * 256].view(T, 2, 128))
    q, k, v = view("q"), view("k"), view("v")
    ao, Ps = Dd.attention(q, k, v, lens)
    assert O.max_rel_err(_f64(layer.saved["att"]), ao) <= 1e-2
    dO = view("d_att")
    dq, dk, dv = Dd.attention_bwd(dO, q, k, v, Ps, lens)
    # the layer applies the inverse RoPE to dq, dk in place after the attention backward
    pos = Dd.positions(lens)
    dq = Dd.rope(dq, pos, layer.theta, inverse=True)
    dk = Dd.rope(dk, pos, layer.theta, inverse=True)
    assert O.max_rel_err(view("dq"), dq) <= 1e-2
    assert O.max_rel_err(view("dk"), dk) <= 1e-2
    assert O.max_rel_err(view("dv"), dv) <= 1e-2
