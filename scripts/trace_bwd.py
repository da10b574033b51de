"""Whole-grid step trace of the BPTT kernel (rec_tc_bwd.cu), one bidirectional
layer at the config-4 shape:  python scripts/trace_bwd.py [--D 2000]

Slots per (CTA, iteration): 0/3 producer past the step-counter wait (tile 0/1),
1/4 first and 2/5 last stage-full seen by the MMA issuer, 6/7 publish (tile 0/1),
and for tile 0's first epilogue warp: 12 loop start, 8 accumulator full, 9 sends
done, 10 peers' partials received, 13 partials summed, 14 math done, 11 DZ ring
stored.
"""
import argparse, ctypes, os, sys
from collections import Counter
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--T", type=int, default=60)
ap.add_argument("--D", type=int, default=2000)
ap.add_argument("--H", type=int, default=1000)
ap.add_argument("--prec", default="bf16")
a = ap.parse_args()
B, T, D, H, nd = a.B, a.T, a.D, a.H, 2
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(B, T, D, device="cuda", generator=g) * 2 - 1
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
s = H ** -0.5
W = [(torch.rand(D, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
R = [(torch.rand(H, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
b = [(torch.rand(4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
dy = torch.rand(B, T, nd * H, device="cuda", generator=g) * 2 - 1
layer = lstm.LSTMLayer(B, T, D, H, nd, 1, a.prec)
for _ in range(2):
    layer.forward(x, lens, W, R, b)
    layer.backward(dy)
torch.cuda.synchronize()
grid = 128
L = lstm.lib()
buf = torch.zeros(grid * T * 32, dtype=torch.int64, device="cuda")
layer.forward(x, lens, W, R, b)
L.sl_debug_set_flags(int(os.environ.get("SL_FLAGS", "0")))
L.sl_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), -1)
layer.backward(dy)
torch.cuda.synchronize()
L.sl_debug_set_trace(None, 0)
L.sl_debug_set_flags(0)
t = buf.view(grid, T, 32).cpu().double() / 1000.0
t = t - t[:, 1, 0].min()
sl = slice(3, T - 3)
med = lambda v: round(float(v.median()), 2)
per = (t[:, T - 4, 6] - t[:, 4, 6]) / (T - 8)
print(f"period median {med(per)} us")
for tile in (0, 1):
    pub = t[:, sl, 6 + tile]
    spread = pub.max(dim=0).values - pub.min(dim=0).values
    nxt = t[:, 4:T - 2, 0 + 3 * tile]
    print(f"tile {tile}: publish spread median {med(spread)} us; last publishers:",
          Counter(int(c) for c in pub.argmax(dim=0)).most_common(6))
w2f = (t[:, sl, 1] - t[:, sl, 0]).median(dim=1).values
stream = (t[:, sl, 2] - t[:, sl, 1]).median(dim=1).values
q = torch.tensor([0.0, 0.1, 0.5, 0.9, 1.0], dtype=torch.float64)
print("tile0 stream quantiles:", [round(v, 2) for v in torch.quantile(stream, q).tolist()],
      "wait->first:", [round(v, 2) for v in torch.quantile(w2f, q).tolist()])
ph = {"tfull-wait": (12, 8), "sends": (8, 9), "recv-wait": (9, 10), "sum": (10, 13), "math": (13, 14),
      "ring-store": (14, 11), "sync+pub": (11, 6)}
print("tile0 epilogue (median over CTAs of per-CTA medians):",
      {k: med((t[:, sl, j] - t[:, sl, i]).median(dim=1).values) for k, (i, j) in ph.items()})
slow = torch.argsort(stream, descending=True)[:4].tolist()
print("slowest streams:", slow, [round(float(stream[i]), 2) for i in slow])
for dd in (0, 1):
    cs = slice(dd * 64, dd * 64 + 64)
    pub = t[cs, sl, 6]
    spread = pub.max(dim=0).values - pub.min(dim=0).values
    lastc = Counter(int(c) + dd * 64 for c in pub.argmax(dim=0)).most_common(4)
    print(f"dir {dd}: tile-0 publish spread median {med(spread)} us; last: {lastc}")
st_ = 20
for c in [lastc[0][0], lastc[0][0] ^ 1, 0]:
    r = t[c, st_]
    base = r[12]
    print(f"  cta {c} it {st_}: start {float(r[0] - t[0, st_, 0]):+.2f} vs cta0 | first-full {float(r[1]-r[0]):.2f} "
          f"last-full {float(r[2]-r[0]):.2f} | epi: loop {float(r[12]-r[0]):+.2f} tfull {float(r[8]-base):.2f} "
          f"sends {float(r[9]-base):.2f} recv {float(r[10]-base):.2f} sum {float(r[13]-base):.2f} "
          f"math {float(r[14]-base):.2f} ring {float(r[11]-base):.2f} pub {float(r[6]-base):.2f}")

# lateness vs placement: mean tile-0 publish time relative to the step's median, per CTA
raw = buf.view(grid, T, 32).cpu()
smid = raw[:, 0, 31].tolist()
late = (t[:, sl, 6] - t[:, sl, 6].median(dim=0).values).mean(dim=1)
order = torch.argsort(late, descending=True).tolist()
print("latest CTAs (cta, smid, mean lateness us):", [(c, int(smid[c]), round(float(late[c]), 2)) for c in order[:12]])
print("earliest CTAs:", [(c, int(smid[c]), round(float(late[c]), 2)) for c in order[-8:]])
import statistics
lo = [float(late[c]) for c in range(grid) if smid[c] < 74]
hi = [float(late[c]) for c in range(grid) if smid[c] >= 74]
print(f"mean lateness smid<74: {statistics.mean(lo) if lo else 0:.2f} ({len(lo)}), smid>=74: {statistics.mean(hi) if hi else 0:.2f} ({len(hi)})")

rawd = buf.view(grid, T, 32).cpu().double() / 1000.0
for mt in (0, 1):
    lastiss = (t[:, sl, 16 + mt] - t[:, sl, 3 * mt])  # first ready/issue -> last issue
    waitful = rawd[:, sl, 18 + mt]                     # summed waits for a free slot
    lastfull = t[:, sl, 2 + 3 * mt] - t[:, sl, 16 + mt]
    print(f"tile {mt}: first->last issue median {float(lastiss.median()):.2f} us; ring-full waits {float(waitful.median()):.2f} us; last issue->last full {float(lastfull.median()):.2f} us")
for mt in (0, 1):
    lat = t[:, sl, 22 + mt] - t[:, sl, 20 + mt]
    print(f"tile {mt}: mid-box issue -> full at the MMA: median {float(lat.median()):.2f} us, 90% {float(torch.quantile(lat.flatten(), 0.9)):.2f}")
# epilogue phases by die (smid < 74 / >= 74)
die = torch.tensor([1 if sm >= 74 else 0 for sm in smid])
for dd in (0, 1):
    m = die == dd
    row = {k: round(float((t[m][:, sl, j] - t[m][:, sl, i]).median()), 2) for k, (i, j) in ph.items()}
    strm = float((t[m][:, sl, 2] - t[m][:, sl, 1]).median())
    print(f"die {dd} ({int(m.sum())} CTAs): stream {strm:.2f}", row)
