"""K3 with and without its K4 operand-image stores (experiments build, debug flag 8):
how much of the BPTT step the row-scattered DZ image stores cost.
    SL_LIB_PATH=paper_1805_05225_b200/lib_exp/libseqloom_cuda.so python scripts/k3_noimg.py"""
import ctypes, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_05225_b200 import lstm
L = lstm.lib()
L.sl_debug_set_flags.argtypes = [ctypes.c_int]
for flags in (0, 8, 0, 8):
    L.sl_debug_set_flags(flags)
    r = subprocess.run([sys.executable, "scripts/phase_layer.py", "--iters", "5", "--prec", "fp32"], capture_output=True,
                       text=True, env=dict(os.environ, SL_DEBUG_FLAGS=str(flags)))
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            d = json.loads(line)
            print(flags, {k: round(v["ms_per_call"], 3) for k, v in d["phases"].items() if k.startswith("k3") or k.startswith("k2")})
