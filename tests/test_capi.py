"""CPU tests of the C-ABI library: it loads, exports every symbol the public
header declares, and validates descriptors with the reference's error
behaviour — no compute calls (there is no GPU here)."""
import ctypes
import os
import re

import pytest

from paper_1805_05225_b200 import lstm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", "seqloom_cuda.h")]


def declared_symbols():
    names = set()
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(sl_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("sl_lstm_layer_fwd", "sl_lstm_layer_bwd", "sl_lstm_cell_fwd", "sl_lstm_cell_bwd",
              "sl_lstm_reserve_size", "sl_lstm_workspace_size", "sl_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = lstm.lib()
    for s in declared_symbols():
        assert hasattr(L, s), f"{s} declared in include/ but not exported"


def test_library_is_sm100a_only():
    # the product library carries sm_100a SASS only (no PTX / other-arch fallback)
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lstm.LIB_PATH],
                       capture_output=True, text=True)
    assert r.returncode == 0
    archs = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert archs == {"100a"}, archs


def desc(**kw):
    d = dict(batch=4, time=5, input_dim=3, hidden=8, num_dirs=1, direction=1, precision=0,
             flags=0)
    d.update(kw)
    return lstm._Layer(*[d[n] for n, _ in lstm._Layer._fields_])


def test_valid_descriptor_and_sizes():
    L = lstm.lib()
    d = desc()
    assert L.sl_lstm_layer_check(ctypes.byref(d)) == 0
    r1 = L.sl_lstm_reserve_size(ctypes.byref(d))
    w1 = L.sl_lstm_workspace_size(ctypes.byref(d))
    assert r1 > 0 and w1 > 0
    d2 = desc(num_dirs=2)
    # per-direction saves double; the fp32 mode's [X | 1] operand image is shared by both
    assert L.sl_lstm_reserve_size(ctypes.byref(d2)) > r1


@pytest.mark.parametrize("kw,code,needle", [
    (dict(direction=0), lstm.SL_ERR_INVALID_ARGUMENT, "direction must be +1 or -1"),
    (dict(direction=2), lstm.SL_ERR_INVALID_ARGUMENT, "direction must be +1 or -1"),
    (dict(time=0), lstm.SL_ERR_SHAPE, "Batch and Time"),
    (dict(batch=-1), lstm.SL_ERR_SHAPE, "Batch and Time"),
    (dict(num_dirs=3), lstm.SL_ERR_INVALID_ARGUMENT, "num_dirs"),
    (dict(precision=7), lstm.SL_ERR_UNSUPPORTED, "precision"),
])
def test_descriptor_errors_match_reference(kw, code, needle):
    # reference layers.cpp:10-16: ShapeError for missing axes, invalid_argument for direction
    L = lstm.lib()
    rc = L.sl_lstm_layer_check(ctypes.byref(desc(**kw)))
    assert rc == code
    assert needle in L.sl_last_error().decode()
    assert L.sl_lstm_reserve_size(ctypes.byref(desc(**kw))) == 0


def test_python_mirror_raises_like_reference():
    import torch
    x = torch.zeros(2, 3, 4)
    with pytest.raises(ValueError, match="direction must be"):
        lstm.lstm_sequence(x, torch.ones(2, dtype=torch.int32), torch.zeros(4, 8),
                           torch.zeros(2, 8), torch.zeros(8), direction=0)
    with pytest.raises(lstm.ShapeError):
        lstm.lstm_sequence(torch.zeros(3, 4), torch.ones(2, dtype=torch.int32),
                           torch.zeros(4, 8), torch.zeros(2, 8), torch.zeros(8), direction=1)


def test_bf16_activation_flags():
    # SL_LAYER_X_BF16 / SL_LAYER_Y_BF16: bf16 precision only, known bits only;
    # with a bf16 input the reserve no longer carries a converted copy of x
    L = lstm.lib()
    both = lstm.SL_LAYER_X_BF16 | lstm.SL_LAYER_Y_BF16
    assert L.sl_lstm_layer_check(ctypes.byref(desc(precision=1, flags=both))) == 0
    assert L.sl_lstm_layer_check(ctypes.byref(desc(precision=0, flags=1))) == lstm.SL_ERR_UNSUPPORTED
    assert "precision" in L.sl_last_error().decode()
    assert L.sl_lstm_layer_check(ctypes.byref(desc(precision=1, flags=8))) == lstm.SL_ERR_INVALID_ARGUMENT
    kw = dict(batch=64, time=30, input_dim=200, hidden=64, precision=1)
    r0 = L.sl_lstm_reserve_size(ctypes.byref(desc(**kw)))
    r1 = L.sl_lstm_reserve_size(ctypes.byref(desc(flags=lstm.SL_LAYER_X_BF16, **kw)))
    assert 0 < r1 <= r0 - 64 * 30 * 256 * 2
    for f in (1, 7, 64, 199, 2000):
        assert L.sl_lstm_bf16_pitch(f) == lstm.bf16_pitch(f) == (f + 64) // 64 * 64


def test_x3_activation_flags():
    # SL_LAYER_X_X3 / SL_LAYER_Y_X3: fp32 precision on the tensor-core path only; with
    # an x image the reserve no longer carries the layer's own [X | 1] image
    L = lstm.lib()
    both = lstm.SL_LAYER_X_X3 | lstm.SL_LAYER_Y_X3
    kw = dict(batch=64, time=30, input_dim=200, hidden=64, num_dirs=2)
    assert L.sl_lstm_layer_check(ctypes.byref(desc(precision=0, flags=both, **kw))) == 0
    assert L.sl_lstm_layer_check(ctypes.byref(desc(precision=1, flags=lstm.SL_LAYER_X_X3, **kw))) == \
        lstm.SL_ERR_UNSUPPORTED
    assert "x3" in L.sl_last_error().decode()
    r0 = L.sl_lstm_reserve_size(ctypes.byref(desc(precision=0, **kw)))
    r1 = L.sl_lstm_reserve_size(ctypes.byref(desc(precision=0, flags=lstm.SL_LAYER_X_X3, **kw)))
    assert 0 < r1 <= r0 - 2 * 64 * 30 * lstm.bf16_pitch(200) * 2


def test_attn_decoder_descriptor_validation():
    """sl_attn_decoder_workspace_size: host-only shape checks (0 + sl_last_error on bad dims)."""
    from paper_1805_05225_b200.decoder import _Desc
    L = lstm.lib()
    L.sl_attn_decoder_workspace_size.restype = ctypes.c_size_t
    L.sl_attn_decoder_workspace_size.argtypes = [ctypes.POINTER(_Desc)]
    ok = _Desc(256, 60, 60, 620, 2000, 1000, 1000, 1000, 20000)
    n = L.sl_attn_decoder_workspace_size(ctypes.byref(ok))
    assert n > 0
    small = _Desc(4, 7, 5, 12, 16, 8, 16, 8, 11)
    assert 0 < L.sl_attn_decoder_workspace_size(ctypes.byref(small)) < n
    for bad, needle in ((_Desc(4, 7, 5, 12, 16, 8, 2000, 8, 11), b"key_dim <= 1024"),
                        (_Desc(4, 7, 5, 12, 16, 9, 16, 8, 11), b"multiples of 8"),
                        (_Desc(0, 7, 5, 12, 16, 8, 16, 8, 11), b"positive"),
                        (_Desc(300, 7, 5, 12, 16, 8, 16, 8, 11), b"batch <= 256")):
        assert L.sl_attn_decoder_workspace_size(ctypes.byref(bad)) == 0
        assert needle in L.sl_last_error()


def test_fp32_layers_run_on_the_tensor_cores():
    """SL_PREC_FP32 maps to the split-bf16 tcgen05 path for every BASELINE shape
    (configs 1-5: H = 128, 1000, 1024; B up to 1024), not the SIMT kernels."""
    from paper_1805_05225_b200 import lstm
    L = lstm.lib()
    for (B, T, D, H, nd) in [(8, 20, 128, 128, 1), (128, 60, 1024, 1024, 1), (256, 60, 620, 1000, 2),
                             (256, 60, 2000, 1000, 2), (256, 60, 2620, 1000, 1), (1024, 500, 2048, 1024, 2),
                             (4, 9, 16, 24, 2)]:
        d = lstm._Layer(B, T, D, H, nd, 1, lstm.PRECISIONS["fp32"], 0)
        assert lstm.PATHS[L.sl_lstm_layer_path(ctypes.byref(d))] == "fp32_x3_tc", (B, T, D, H, nd)
        d = lstm._Layer(B, T, D, H, nd, 1, lstm.PRECISIONS["bf16"], 0)
        assert lstm.PATHS[L.sl_lstm_layer_path(ctypes.byref(d))] == "bf16_tc"
