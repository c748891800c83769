import sys, torch
sys.path.insert(0, '.')
import paper_2604_26256_b200 as G
from paper_2604_26256_b200 import _lib as L
torch.manual_seed(0)
dev = torch.device('cuda')
for (n, d, V) in [(128, 64, 256), (300, 192, 1000), (1024, 512, 4096)]:
    X = (torch.randn(n, d, device=dev)).bfloat16()
    W = (torch.randn(V, d, device=dev) * 0.1).bfloat16()
    ld = (V + 7) // 8 * 8
    out = torch.zeros(n, ld, dtype=torch.bfloat16, device=dev)
    L.grpo_async_lmhead_logits(X, W, n, d, V, out, ld)
    torch.cuda.synchronize()
    ref = (X.float() @ W.float().T)
    err = (out[:, :V].float() - ref).abs().max().item()
    print(n, d, V, 'max abs err', err, 'ref max', ref.abs().max().item(), flush=True)
