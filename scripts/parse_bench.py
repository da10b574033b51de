import json,sys
for f in sys.argv[1:]:
  for l in open(f):
    if not l.startswith('{'): continue
    d=json.loads(l); ph=d["roofline"]["phases"]
    g=lambda k: round(ph[k]["ms_per_call"]*1e3,1) if k in ph else None
    print(f.split('/')[-1], round(d["value"]), round(d["ms_per_step"],2), d["clocks"]["sm_mhz"], 'att', g("k8_attention_fwd"), g("k8_attention_bwd"), 'cell', g("k10_cell_gemm"), 'g1', g("k10_g1_gemm"), 'bf16', round(d["bf16_mode"]["value"]))
