"""Per-kernel GPU time of one config-4 training step (torch.profiler / CUPTI
activity records: warm caches, the kernels as they run inside the step).

    python scripts/kprof_step.py [--precision fp32|bf16] [--graph]
"""
import argparse
import collections
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1805_05225_b200.model import Seq2SeqAttention

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp32")
ap.add_argument("--graph", action="store_true")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--no-prof", action="store_true", help="just run the steps (for an outer ncu)")
a = ap.parse_args()
L, B, T, D0, H, V = 6, 256, 60, 620, 1000, 20000
dev = torch.device("cuda:0")
m = Seq2SeqAttention(L, B, T, T, D0, H, V, V, V, device=dev, precision=a.precision)
m.init_uniform(seed=1)
g = torch.Generator(device=dev).manual_seed(100)
x = torch.randint(0, V, (B, T), device=dev, generator=g, dtype=torch.int32)
y = torch.randint(0, V, (B, T), device=dev, generator=g, dtype=torch.int32)
lens = torch.full((B,), T, dtype=torch.int32, device=dev)
step = lambda: m.step(x, lens, y)
for _ in range(3):
    step()
torch.cuda.synchronize()
run = step
if a.graph:
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    gr.replay()
    torch.cuda.synchronize()
    run = gr.replay
if a.no_prof:
    run()
    torch.cuda.synchronize()
    sys.exit(0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
span = [float("inf"), 0.0]
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    n = e.name.replace("sl::(anonymous namespace)::", "").replace("sl::<unnamed>::", "")
    n = re.sub(r"^void ", "", re.sub(r"\(.*", "", n))
    agg[n[:70]][0] += 1
    agg[n[:70]][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(t for _, t in agg.values())
rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
for n, (c, t) in rows[:a.top]:
    print(f"{n:70s} {c:6d} {t / 1e3:9.3f} ms {t / c:9.2f} us/call {100 * t / tot:5.1f}%")
print(f"kernel total {tot / 1e3:.2f} ms over {sum(c for c, _ in agg.values())} launches")
# per (kernel, grid): separates the shapes of one kernel (e.g. per-step vs hoisted GEMMs)
trace = os.path.join("gpurun_out", f"kprof_{a.precision}.trace.json")
prof.export_chrome_trace(trace)
ev = [e for e in json.load(open(trace))["traceEvents"] if e.get("cat") == "kernel"]
byg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    n = e["name"].replace("sl::(anonymous namespace)::", "").replace("sl::<unnamed>::", "")
    n = re.sub(r"^void ", "", re.sub(r"\(.*", "", n))[:48]
    k = f"{n} grid={tuple(e['args'].get('grid', ()))}"
    byg[k][0] += 1
    byg[k][1] += e["dur"]
print("--- by (kernel, grid)")
for k, (c, t) in sorted(byg.items(), key=lambda kv: -kv[1][1])[:a.top]:
    print(f"{k:80s} {c:6d} {t / 1e3:9.3f} ms {t / c:9.2f} us/call")
# idle time between consecutive device activities (kernels + memcpy/memset), by pair
acts = sorted([e for e in json.load(open(trace))["traceEvents"]
               if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
gaps = collections.defaultdict(lambda: [0, 0.0])
nm = lambda e: re.sub(r"^void ", "", re.sub(r"\(.*", "", e["name"].replace("sl::(anonymous namespace)::", "")))[:34]
tot_gap = 0.0
for p_, n_ in zip(acts, acts[1:]):
    g = n_["ts"] - (p_["ts"] + p_["dur"])
    if g > 0:
        tot_gap += g
        k = f"{nm(p_)} -> {nm(n_)}"
        gaps[k][0] += 1
        gaps[k][1] += g
span = acts[-1]["ts"] + acts[-1]["dur"] - acts[0]["ts"]
print(f"--- span {span / 1e3:.2f} ms, idle {tot_gap / 1e3:.2f} ms over {len(acts)} activities")
for k, (c, t) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"{k:75s} {c:5d} {t / 1e3:8.3f} ms {t / c:6.2f} us")
os.remove(trace)
json.dump({n: {"calls": c, "us": t} for n, (c, t) in rows}, open(os.path.join("gpurun_out", f"kprof_{a.precision}.json"), "w"), indent=0)
