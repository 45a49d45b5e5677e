"""Debug: per-sequence errors of the decoder layer's forward intermediates vs the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import decoder as Dd, lora as O
from paper_2509_01193_b200.decoder import DecoderLayer
SMALL = [("q", 256, 256, "col", "attn"), ("k", 256, 256, "col", "attn"), ("v", 256, 256, "col", "attn"),
         ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
         ("down", 512, 256, "row", "down_in")]

f64 = lambda t: t.float().cpu().numpy().astype(np.float64)
ranks, scales = [16, 8, 16], [2.0, 0.5, 1.0]
lens = np.array([1, 300, 57, 129, 200, 33], np.int32)
tasks = np.array([0, 0, 1, 1, 2, 2], np.int32)
layer = DecoderLayer(SMALL, n_heads=2, ranks=ranks, scales=scales, seed=0, deterministic_attn=True)
T = int(lens.sum())
g = torch.Generator(device="cuda"); g.manual_seed(1)
X = torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16)
Y = layer.forward(lens, tasks, X)
torch.cuda.synchronize()
P = {"g_attn": f64(layer.g_attn), "g_mlp": f64(layer.g_mlp)}
for p in layer.lora.projs:
    P[p.name] = (f64(p.W), f64(p.A), f64(p.B))
cfg = {"n_heads": 2, "eps": layer.eps, "theta": layer.theta}
Yo, c = Dd.layer_fwd(f64(X), P, cfg, ranks, scales, lens, tasks)
C = layer.cache
def get(n, w): return f64(C[n][:T * w].view(T, w))
pairs = [("h1", get("h1", 256), c["h1"]), ("q_rot", get("q", 256), c["qr"].reshape(T, 256)),
         ("k_rot", get("k", 256), c["kr"].reshape(T, 256)), ("v", get("v", 256), c["v"]),
         ("att", f64(layer.saved["att"].view(T, 256)), c["att"]), ("x2", get("x2", 256), c["x2"]),
         ("h2", get("h2", 256), c["h2"]), ("gate", get("gate", 512), c["gate"]), ("act", get("act", 512), c["act"]),
         ("Y", f64(Y), Yo)]
off = np.concatenate([[0], np.cumsum(lens)])
for name, a, b in pairs:
    per = [O.max_rel_err(a[off[i]:off[i+1]], b[off[i]:off[i+1]]) for i in range(len(lens))]
    print(f"{name:6s} all {O.max_rel_err(a, b):.4f} per-seq " + " ".join(f"{x:.4f}" for x in per))
# q before rope: recompute oracle q vs gpu q un-roped
qo = c["q"]
qg = f64(C["q"][:T*256].view(T,256))
qg_unrot = Dd.rope(qg.reshape(T,2,128), Dd.positions(lens), 1e4, inverse=True).reshape(T,256)
print("q unrot", O.max_rel_err(qg_unrot, qo), [round(O.max_rel_err(qg_unrot[off[i]:off[i+1]], qo[off[i]:off[i+1]]),4) for i in range(len(lens))])
# attention alone on the GPU's own bf16 inputs
qg = f64(C["q"][:T*256].view(T, 2, 128)); kg = f64(C["k"][:T*256].view(T, 2, 128)); vg = f64(C["v"][:T*256].view(T, 2, 128))
ao, _ = Dd.attention(qg, kg, vg, lens)
ag = f64(layer.saved["att"].view(T, 256))
print("attn on gpu inputs", O.max_rel_err(ag, ao.reshape(T, 256)), [round(O.max_rel_err(ag[off[i]:off[i+1]], ao.reshape(T,256)[off[i]:off[i+1]]),4) for i in range(len(lens))])
# logit scale
S = np.einsum("thd,shd->hts", qg[1:301], kg[1:301]) / np.sqrt(128)
print("logit std", S.std(), "max", S.max())
