"""Per-tensor error of the attention decoder vs the fp64 restatement (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import oracle
from test_decoder_gpu import CASES, make_case, rel, run_gpu
from paper_1805_05225_b200.decoder import NAMES

dims = CASES[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
P, enc_x, lens, ids, d_ro = make_case(sum(dims), *dims)
ro, grads, d_enc = run_gpu(dims, P, enc_x, lens, ids, d_ro)
r_ro, g, r_denc = oracle.attn_decoder_np(lens, enc_x.float().numpy(), ids, P, d_readout=d_ro,
                                         relu_mask=(ro > 0).cpu().numpy())
print(os.environ.get("SL_DEC_TANH", "0"), "readout", rel(ro, r_ro), "d_enc", rel(d_enc, r_denc))
print("  " + " ".join(f"{n}={rel(grads[n], g[n]):.4f}" for n, _ in NAMES))
