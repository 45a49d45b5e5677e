import torch, math
from flash_attn import flash_attn_interface as fa
T, H, D = 300, 4, 128
lens = [100, 200]
cu = torch.tensor([0, 100, 300], dtype=torch.int32, device="cuda")
q, k, v = (torch.randn(T, H, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o, lse, _, _ = fa._flash_attn_varlen_forward(q, k, v, cu, cu, 200, 200, 0.0, 1 / math.sqrt(D), True)
print("lse", lse.shape, lse.dtype, lse.stride())
# reference lse for head 0, token 5 of seq 0 and token 150 (seq 1, pos 50)
for tok, s0 in ((5, 0), (150, 100)):
    z = (q[tok, 0].float() @ k[s0:tok + 1, 0].float().T) / math.sqrt(D)
    print(tok, float(torch.logsumexp(z, 0)), float(lse[0, tok]))
