"""Whole-grid step trace of the CTA-pair forward recurrence (rec_tc_pair.cu).

    python scripts/trace_all.py [--D 2000] [--B 256] [--H 1000]

Every CTA records its per-step phase timestamps (slots as in trace_report.py);
this prints, per step, when the last CTA of each batch tile published, how
long the consumers took to see it, and which CTAs straggle and why.
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--T", type=int, default=60)
ap.add_argument("--D", type=int, default=2000)
ap.add_argument("--H", type=int, default=1000)
ap.add_argument("--nd", type=int, default=2)
ap.add_argument("--prec", default="bf16")
a = ap.parse_args()
B, T, D, H, nd = a.B, a.T, a.D, a.H, a.nd
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(B, T, D, device="cuda", generator=g) * 2 - 1
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
s = H ** -0.5
W = [(torch.rand(D, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
R = [(torch.rand(H, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
b = [(torch.rand(4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
layer = lstm.LSTMLayer(B, T, D, H, nd, 1, a.prec)
for _ in range(2):
    layer.forward(x, lens, W, R, b)
torch.cuda.synchronize()
grid = 2 * ((H + 31) // 32) * nd
L = lstm.lib()
L.sl_debug_set_flags(int(os.environ.get("SL_FLAGS", "0")))
buf = torch.zeros(grid * T * 48, dtype=torch.int64, device="cuda")
L.sl_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), -1)
layer.forward(x, lens, W, R, b)
torch.cuda.synchronize()
L.sl_debug_set_trace(None, 0)
L.sl_debug_set_flags(0)
t = buf.view(grid, T, 48).cpu().double() / 1000.0  # us
t0 = t[:, 1, 0].min()
t = t - t0
tile = torch.arange(grid) % 2
steps = range(3, T - 3)
rows = []
for st in steps:
    for r in (0, 1):
        m = tile == r
        pub = t[m, st, 6]
        nxt = t[m, st + 1, 0]  # producers saw the counter for step st+1
        last = pub.max().item()
        rows.append((last - pub.min().item(), (nxt - last).median().item(), (nxt - last).max().item(),
                     int(torch.nonzero(m)[pub.argmax()].item())))
rows_t = torch.tensor([r[:3] for r in rows])
print(f"grid {grid}: per step and tile (median over steps) | publish spread {rows_t[:,0].median():.2f} us | "
      f"last publish -> consumer start: median {rows_t[:,1].median():.2f} max {rows_t[:,2].median():.2f} us")
period = (t[:, T - 4, 6] - t[:, 4, 6]) / (T - 8)
print(f"period (all CTAs) median {period.median():.2f} us")
from collections import Counter
c = Counter(r[3] for r in rows)
print("most frequent last publishers (cta: count):", c.most_common(8))
# phase durations per CTA, median over steps (leader CTAs hold the MMA slots 1, 2)
sl = slice(3, T - 3)
w2f = (t[:, sl, 1] - t[:, sl, 0]).median(dim=1).values
stream = (t[:, sl, 2] - t[:, sl, 1]).median(dim=1).values
m2p = (t[:, sl, 6] - t[:, sl, 8]).median(dim=1).values
tfw = (t[:, sl, 8] - t[:, sl, 12]).median(dim=1).values
lead = tile == 0
print(f"leaders: wait->first median {w2f[lead].median():.2f} max {w2f[lead].max():.2f} | "
      f"stream median {stream[lead].median():.2f} max {stream[lead].max():.2f} (cta {int(stream[lead].argmax())*2})")
print(f"all: tfull->publish median {m2p.median():.2f} max {m2p.max():.2f} (cta {int(m2p.argmax())})")
raw = buf.view(grid, T, 48).cpu().double()
polls = raw[:, sl, 14]
spin = (raw[:, sl, 0] - raw[:, sl, 13]) / 1000.0
rtt = spin.sum() / polls.clamp(min=1).sum()
print(f"counter spin: median {spin.median():.2f} us, {polls.median():.0f} polls; mean poll round trip {rtt:.3f} us")
for cta in [cc for cc, _ in c.most_common(3)]:
    p = cta - cta % 2
    print(f"  cta {cta}: start {t[cta, sl, 0].mean() - t[:, sl, 0].mean(dim=0).mean():+.2f} vs mean; "
          f"pair leader stream {stream[p]:.2f}, wait->first {w2f[p]:.2f}; tfull->pub {m2p[cta]:.2f}")
qs = torch.tensor([0.0, 0.1, 0.5, 0.9, 1.0], dtype=torch.float64)
print("leader stream quantiles (0,10,50,90,100%):", [round(v, 2) for v in torch.quantile(stream[lead], qs).tolist()])
slow = torch.argsort(stream[lead], descending=True)[:6] * 2
print("slowest leaders:", slow.tolist(), [round(stream[i].item(), 2) for i in slow])
st0 = 20
for cta in slow[:3].tolist() + [0]:
    row = t[cta, st0]
    print(f"  cta {cta} step {st0}: first-issue {row[0]:.2f} first-full {row[1]:.2f} last-full {row[2]:.2f} "
          f"tfull {row[8]:.2f} publish {row[6]:.2f} | peer publish {t[cta + 1, st0, 6]:.2f}")

# per-group readiness vs issue: does a consumer wait for publishers or for ring slots?
P = (H + 31) // 32
ngrp = 8 if ((H + 63) // 64) % 2 == 0 else (H + 63) // 64
gunits = ((H + 63) // 64 // ngrp) * 64
cta_pair = (torch.arange(grid) // 2) % P
cta_dir = (torch.arange(grid) // 2) // P
cta_grp = cta_pair * 32 // gunits
slk, lag_full = [], []
for st_ in range(4, T - 4):
    for c in range(0, grid):
        r, d = c % 2, int(cta_dir[c])
        same = (tile == r) & (cta_dir == d)
        koff = int(cta_pair[c]) % ngrp
        for kq in range(ngrp):
            kg = (kq + koff) % ngrp
            pubs = t[same & (cta_grp == kg), st_ - 1, 6]
            ready = pubs.max().item()
            slk.append(t[c, st_, 16 + kq].item() - ready)
            if r == 0:
                lag_full.append(t[c, st_, 32 + kq].item() - t[c, st_, 16 + kq].item())
slk = torch.tensor(slk, dtype=torch.float64)
lag_full = torch.tensor(lag_full, dtype=torch.float64)
print(f"group issue - group ready: quantiles {[round(v,2) for v in torch.quantile(slk, qs).tolist()]}")
print(f"group issue -> stage full at MMA (leaders): quantiles {[round(v,2) for v in torch.quantile(lag_full, qs).tolist()]}")
c = 0
st_ = 20
print("cta 0 step 20 issue times:", [round(t[c, st_, 16 + k].item() - t[c, st_, 16].item(), 2) for k in range(ngrp)])
print("cta 0 step 20 full  times:", [round(t[c, st_, 32 + k].item() - t[c, st_, 16].item(), 2) for k in range(ngrp)])
print("cta 0 step 20 tfull/publish:", round(t[c, st_, 8].item() - t[c, st_, 16].item(), 2), round(t[c, st_, 6].item() - t[c, st_, 16].item(), 2))
sl_ = int(slow[0])
for c in (sl_, sl_ + 1, 0, 1):
    print(f"cta {c} step 20 issue:", [round(t[c, st_, 16 + k].item() - t[c, st_, 16].item(), 2) for k in range(ngrp)],
          "| full:", [round(t[c, st_, 32 + k].item() - t[c, st_, 16].item(), 2) for k in range(ngrp)] if c % 2 == 0 else "")
    print(f"   first issue at {t[c, st_, 16].item() - t[0, st_, 16].item():+.2f} vs cta 0; tfull {t[c, st_, 8].item() - t[c, st_, 16].item():.2f} publish {t[c, st_, 6].item() - t[c, st_, 16].item():.2f}")
