"""Per-tensor errors of the config-4 training step (bench shape) vs the fp64
restatement (oracle/torch_model.py), for our fp32 / bf16 modes and for a plain
fp32 evaluation of the same formulas (torch autograd, FP32 GEMMs, no TF32) —
the error an fp32 reference itself has on each tensor."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import oracle
from oracle import torch_model
from test_fullsize_gpu import _model_tensors, rel
from paper_1805_05225_b200.model import Seq2SeqAttention
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
L, B, T, emb, H, V = 6, int(os.environ.get("B", 256)), 60, 620, 1000, 20000
out = {}
for prec in ("fp32", "bf16"):
    m = Seq2SeqAttention(L, B, T, T, emb, H, V, V, V, device="cuda", precision=prec)
    m.init_uniform(seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    src = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    trg = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    lens = torch.randint(T // 2, T + 1, (B,), device="cuda", generator=g, dtype=torch.int32)
    lens[0] = T
    loss = m.forward_backward(src, lens, trg)
    torch.cuda.synchronize()
    readout = m.readout.clone()
    ctr = int(m.dropout_counter().item())
    keep = torch.as_tensor(oracle.dropout_mask_np(oracle.dropout_key(1, "output/output_prob", 0, ctr), B, T, H, 0.3),
                           device="cuda")
    P = {k: v.detach().double() for k, v in _model_tensors(m, "p").items()}
    G = {k: v.detach().clone() for k, v in _model_tensors(m, "g").items()}
    del m
    torch.cuda.empty_cache()
    r_loss, r_ro, r_g = torch_model.loss_and_grads(P, src, lens, trg, lens, L, keep=keep, relu_mask=readout > 0)
    out[prec] = {n: rel(G[n], r_g[n]) for n in G}
    out[prec]["_loss"] = abs(float(loss) - float(r_loss)) / abs(float(r_loss))
    out[prec]["_readout"] = rel(readout, r_ro)
    if prec == "fp32":  # a plain fp32 evaluation of the same formulas
        Pf = {k: v.float() for k, v in P.items()}
        leaves = {k: v.clone().requires_grad_(True) for k, v in Pf.items()}
        l32, _ = torch_model.forward_loss(leaves, src, lens, trg, lens, L, keep=keep, relu_mask=readout > 0)
        names = list(leaves)
        gr = torch.autograd.grad(l32, [leaves[n] for n in names], allow_unused=True)
        out["torch_fp32"] = {n: rel(gv, r_g[n]) for n, gv in zip(names, gr) if gv is not None}
        scale = {n: float(r_g[n].abs().max()) for n in r_g}
        out["ref_grad_absmax"] = scale
    del r_g
    torch.cuda.empty_cache()
names = sorted(out["fp32"])
print(f"{'tensor':28s} {'ours fp32':>10s} {'torch fp32':>10s} {'ours bf16':>10s} {'|g|max':>10s}")
for n in names:
    print(f"{n:28s} {out['fp32'][n]:10.2e} {out['torch_fp32'].get(n, float('nan')):10.2e} {out['bf16'][n]:10.2e} "
          f"{out['ref_grad_absmax'].get(n, float('nan')):10.2e}")
json.dump(out, open("gpurun_out/fullsize_errors.json", "w"), indent=1)
