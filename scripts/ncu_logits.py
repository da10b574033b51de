"""Two calls of the fp32 output layer (config 4 shapes) for an outer ncu: the second
call's first pair-GEMM launch is the logits GEMM with the softmax-statistics epilogue.
    ncu --set full -k regex:gemm_bf16_tc2 --launch-skip 3 -c 1 python scripts/ncu_logits.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200.output import OutputCE
B, T, D, V = 256, 60, 1000, 20000
out = OutputCE(B, T, D, V, precision=os.environ.get("PREC", "fp32"))
x = torch.randn(B, T, D, device="cuda") * 0.1
W = torch.randn(D, V, device="cuda") * 0.03
b = torch.randn(V, device="cuda") * 0.1
tg = torch.randint(0, V, (B, T), device="cuda", dtype=torch.int32)
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
for _ in range(2):
    out.forward_backward(x, tg, lens, W, b)
torch.cuda.synchronize()
print("loss", float(out.loss))
