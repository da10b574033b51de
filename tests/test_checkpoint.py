"""Checkpoint format (reference SPEC.md External Interfaces):
meta.json + params.bin of little-endian fp32 in manifest order."""
import json

import numpy as np
import pytest
import torch

from paper_1805_05225_b200 import checkpoint


class _Opt:  # the optimizer surface checkpoint.py uses (optim.Adam on the GPU)
    def __init__(self, n):
        self.m, self.v = torch.randn(n), torch.rand(n)
        self.betas, self.eps, self.clip_norm, self.lr, self._t = (0.9, 0.999), 1e-8, 5.0, 1e-3, 7

    def device_step(self):
        return self._t

    def set_device_step(self, t):
        self._t = t


def test_checkpoint_round_trip_and_layout(tmp_path):
    manifest = [("enc0_fw/W", 0, (3, 8)), ("enc0_fw/R", 24, (2, 8)), ("enc0_fw/b", 40, (8,)), ("src/W", 50, (4, 3))]
    flat = torch.randn(62)  # a gap at [48, 50): not a parameter, never written
    opt = _Opt(62)
    checkpoint.save(str(tmp_path), flat, manifest, optimizer=opt, epoch=3, best_cv=1.25)
    meta = json.load(open(tmp_path / "meta.json"))
    # the reference ParamStore's order: lexicographic by name (param_store.hpp:12), R < W < b
    assert [p["name"] for p in meta["params"]] == ["enc0_fw/R", "enc0_fw/W", "enc0_fw/b", "src/W"]
    assert meta["params"][1]["shape"] == [3, 8] and meta["epoch"] == 3 and meta["best_cv"] == 1.25
    raw = np.fromfile(tmp_path / "params.bin", dtype="<f4")  # manifest order, no gaps
    want = np.concatenate([flat[o:o + int(np.prod(s))].numpy() for _, o, s in checkpoint.ordered(manifest)])
    assert np.array_equal(raw, want)
    flat2, opt2 = torch.zeros(62), _Opt(62)
    opt2.m.zero_(), opt2.v.zero_(), opt2.set_device_step(0)
    checkpoint.load(str(tmp_path), flat2, manifest, optimizer=opt2)
    for _, o, s in manifest:
        k = int(np.prod(s))
        assert torch.equal(flat2[o:o + k], flat[o:o + k])
        assert torch.equal(opt2.m[o:o + k], opt.m[o:o + k]) and torch.equal(opt2.v[o:o + k], opt.v[o:o + k])
    assert opt2.device_step() == 7
    with pytest.raises(ValueError, match="enc0_fw/R"):  # a shape mismatch names the parameter
        bad = list(manifest)
        bad[1] = ("enc0_fw/R", 24, (8, 2))
        checkpoint.load(str(tmp_path), flat2, bad)


def test_checkpoint_order_is_the_reference_param_store_order(tmp_path):
    """The whole Listing-1 model's manifest serialises in ParamStore::manifest()
    order (the reference itself, oracle/_ref: a std::map, param_store.hpp:12)."""
    oracle = pytest.importorskip("oracle")
    try:
        ref = oracle.Reference(32)
    except FileNotFoundError:
        pytest.skip("reference build absent")
    from paper_1805_05225_b200.decoder import NAMES
    names = [f"enc{l}_{d}/{n}" for l in range(6) for d in ("fw", "bw") for n in ("W", "R", "b")]
    names += [r for _, r in NAMES] + ["output/output_prob/W", "output/output_prob/b", "src/W"]
    manifest, off = [], 0
    for n in names:
        manifest.append((n, off, (2,)))
        off += 2
    flat = torch.arange(off, dtype=torch.float32)
    checkpoint.save(str(tmp_path), flat, manifest)
    meta = json.load(open(tmp_path / "meta.json"))
    assert [p["name"] for p in meta["params"]] == ref.param_manifest_order(names)
