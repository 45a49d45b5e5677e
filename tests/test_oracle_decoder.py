"""Pins of the fp64 decoder-layer oracle (oracle/decoder.py), CPU only.

Each pin is fixed by something other than the oracle's own formulas:
  * HF transformers' LlamaDecoderLayer (an independent implementation of the public Llama
    layer) equals the oracle with zero LoRA expand (B = 0), per sequence (to 1e-6: HF
    evaluates the rotary angles and the softmax in fp32);
  * the backward equals central finite differences of <Y, R> for dX and sampled dA / dB of
    every projection;
  * closed forms: RMSNorm scale invariance and unit RMS, RoPE (identity at position 0,
    norm-preserving, relative-position property, inverse), causal attention (first token
    = its own value; equal keys = prefix mean of values), SiLU;
  * packing: the packed batch equals each sequence run alone (block-diagonal attention,
    positions restart per sequence).
"""
import numpy as np
import pytest

from oracle import decoder as Dd

CFG = {"n_heads": 2, "eps": 1e-5, "theta": 10000.0}
H_, F_ = 16, 24
SHAPES = {"q": (H_, H_), "k": (H_, H_), "v": (H_, H_), "o": (H_, H_), "gate": (H_, F_), "up": (H_, F_),
          "down": (F_, H_)}


def _params(seed, ranks, zero_B=False, shapes=None):
    rng = np.random.default_rng(seed)
    R = int(sum(ranks))
    P = {"g_attn": 1.0 + 0.1 * rng.standard_normal(H_), "g_mlp": 1.0 + 0.1 * rng.standard_normal(H_)}
    for p, (i, o) in (shapes or SHAPES).items():
        W = rng.standard_normal((o, i)) / np.sqrt(i)
        A = rng.standard_normal((R, i)) / np.sqrt(i)
        B = np.zeros((o, R)) if zero_B else rng.standard_normal((o, R)) / 2
        P[p] = (W, A, B)
    return P


BATCH = dict(ranks=[2, 3], scales=[1.5, 0.5], seq_lens=np.array([3, 5, 2]), seq_task=np.array([0, 1, 0]))


# grouped-query attention (Llama-2-70B style): 2 query heads share 1 kv head (k, v: 16 -> 8)
GQA = dict(SHAPES, k=(H_, H_ // 2), v=(H_, H_ // 2))


def _run(P, X, b=BATCH):
    return Dd.layer_fwd(X, P, CFG, b["ranks"], b["scales"], b["seq_lens"], b["seq_task"])


@pytest.mark.parametrize("kv_heads", [2, 1])
def test_matches_hf_llama_layer_with_zero_lora(kv_heads):
    """MHA (Llama-2-7B) and grouped-query attention (Llama-2-70B: kv heads shared)."""
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    from transformers.models.llama import modeling_llama as M
    cfg = tr.LlamaConfig(hidden_size=H_, intermediate_size=F_, num_attention_heads=2, num_key_value_heads=kv_heads,
                         rms_norm_eps=CFG["eps"], rope_theta=CFG["theta"], attention_bias=False, mlp_bias=False)
    cfg._attn_implementation = "eager"
    layer = M.LlamaDecoderLayer(cfg, 0).double()
    rot = M.LlamaRotaryEmbedding(cfg).double()
    P = _params(1, BATCH["ranks"], zero_B=True, shapes=SHAPES if kv_heads == 2 else GQA)
    names = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj", "o": "self_attn.o_proj",
             "gate": "mlp.gate_proj", "up": "mlp.up_proj", "down": "mlp.down_proj"}
    sd = {f"{names[p]}.weight": torch.from_numpy(P[p][0]) for p in names}
    sd["input_layernorm.weight"] = torch.from_numpy(P["g_attn"])
    sd["post_attention_layernorm.weight"] = torch.from_numpy(P["g_mlp"])
    layer.load_state_dict(sd)
    rng = np.random.default_rng(2)
    X = rng.standard_normal((int(BATCH["seq_lens"].sum()), H_))
    Y, _ = _run(P, X)
    off = 0
    for n in BATCH["seq_lens"]:
        x = torch.from_numpy(X[off:off + n])[None]
        pos = torch.arange(n)[None]
        mask = torch.full((n, n), float("-inf"), dtype=torch.float64).triu(1)[None, None]
        ref = layer(x, attention_mask=mask, position_ids=pos, position_embeddings=rot(x, pos))
        ref = (ref[0] if isinstance(ref, tuple) else ref)[0].detach().numpy()
        # HF's eager path takes the rotary cos/sin and the softmax in fp32 even for a double
        # model: agreement at fp32 level; a convention error would be O(1)
        assert np.allclose(Y[off:off + n], ref, rtol=1e-6, atol=1e-6)
        off += n


@pytest.mark.parametrize("shapes", [SHAPES, GQA], ids=["mha", "gqa"])
def test_backward_equals_finite_differences(shapes):
    P = _params(3, BATCH["ranks"], shapes=shapes)
    rng = np.random.default_rng(4)
    T = int(BATCH["seq_lens"].sum())
    X = rng.standard_normal((T, H_))
    Rm = rng.standard_normal((T, H_))
    Y, cache = _run(P, X)
    dX, grads = Dd.layer_bwd(Rm, P, CFG, BATCH["ranks"], BATCH["scales"], BATCH["seq_lens"],
                             BATCH["seq_task"], cache)
    f = lambda Pp, Xx: float(np.sum(_run(Pp, Xx)[0] * Rm))
    eps = 1e-6
    num = np.zeros_like(X)
    for i in range(T):
        for j in range(H_):
            Xp, Xm = X.copy(), X.copy()
            Xp[i, j] += eps
            Xm[i, j] -= eps
            num[i, j] = (f(P, Xp) - f(P, Xm)) / (2 * eps)
    assert np.max(np.abs(num - dX)) <= 1e-6 * max(1.0, np.max(np.abs(dX)))
    for p in Dd.PROJS:
        for which in (1, 2):                       # A_p, B_p
            M = P[p][which]
            for _ in range(4):
                a, b = int(rng.integers(M.shape[0])), int(rng.integers(M.shape[1]))
                vals = []
                for sgn in (1, -1):
                    Q = dict(P)
                    Mm = M.copy()
                    Mm[a, b] += sgn * eps
                    Q[p] = tuple(Mm if k == which else P[p][k] for k in range(3))
                    vals.append(f(Q, X))
                g = (vals[0] - vals[1]) / (2 * eps)
                got = grads[p][which - 1][a, b]
                assert abs(g - got) <= 1e-6 * max(1.0, abs(got)), (p, which, a, b, g, got)


def test_rmsnorm_closed_forms():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 32))
    y1, _ = Dd.rmsnorm(x, np.ones(32), 0.0)
    y2, _ = Dd.rmsnorm(7.5 * x, np.ones(32), 0.0)
    assert np.allclose(y1, y2, rtol=1e-13)                       # scale invariance (eps = 0)
    assert np.allclose(np.mean(y1 * y1, axis=-1), 1.0, rtol=1e-13)  # unit RMS


def test_rope_closed_forms():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((6, 2, 8))
    pos = np.array([0, 1, 2, 3, 7, 100])
    y = Dd.rope(x, pos, 10000.0)
    assert np.allclose(y[0], x[0], rtol=0, atol=0)               # position 0: identity
    pair = lambda z: z[..., :4] ** 2 + z[..., 4:] ** 2
    assert np.allclose(pair(y), pair(x), rtol=1e-13)               # rotation of each (j, j+D/2) pair
    assert np.allclose(Dd.rope(y, pos, 10000.0, inverse=True), x, rtol=1e-12, atol=1e-12)
    q, k = x[1:2], x[2:3]
    dot = lambda m, n: np.sum(Dd.rope(q, [m], 1e4) * Dd.rope(k, [n], 1e4))
    assert abs(dot(3, 1) - dot(13, 11)) < 1e-12                    # depends on m - n only
    # angle of pair j at position p is p * theta^(-2j/D): check one value by hand
    j, p = 1, 7
    ang = p * 10000.0 ** (-2 * j / 8)
    e = np.zeros((1, 1, 8))
    e[0, 0, j] = 1.0
    r = Dd.rope(e, [p], 10000.0)
    assert np.isclose(r[0, 0, j], np.cos(ang)) and np.isclose(r[0, 0, j + 4], np.sin(ang))


def test_attention_closed_forms():
    rng = np.random.default_rng(7)
    lens = [4, 3]
    q = rng.standard_normal((7, 2, 8))
    v = rng.standard_normal((7, 2, 8))
    k = np.broadcast_to(rng.standard_normal((1, 2, 8)), (7, 2, 8)).copy()   # equal keys
    O, _ = Dd.attention(q, k, v, lens)
    off = 0
    for n in lens:
        for i in range(n):
            assert np.allclose(O[off + i], v[off:off + i + 1].mean(axis=0), rtol=1e-12)  # prefix mean
        off += n
    O, _ = Dd.attention(q, rng.standard_normal((7, 2, 8)), v, lens)
    assert np.allclose(O[0], v[0]) and np.allclose(O[4], v[4])     # first token sees itself only


def test_silu_closed_forms():
    assert Dd.silu(0.0) == 0.0
    assert np.isclose(Dd.silu(40.0), 40.0) and abs(Dd.silu(-40.0)) < 1e-15
    assert np.isclose(Dd.silu(1.0), 1.0 / (1.0 + np.exp(-1.0)))


def test_packed_equals_sequences_alone():
    P = _params(8, BATCH["ranks"])
    rng = np.random.default_rng(9)
    T = int(BATCH["seq_lens"].sum())
    X = rng.standard_normal((T, H_))
    Y, _ = _run(P, X)
    off = 0
    for n, t in zip(BATCH["seq_lens"], BATCH["seq_task"]):
        b = dict(BATCH, seq_lens=np.array([n]), seq_task=np.array([t]))
        y, _ = _run(P, X[off:off + n], b)
        assert np.allclose(Y[off:off + n], y, rtol=1e-13, atol=1e-13)
        off += n
