"""Checkpoints in the reference trainer's format (SPEC.md "External Interfaces",
SURVEY §8 f4): a directory with

  meta.json   format version, config hash, the parameter manifest (names and
              shapes, in order), epoch, lr state, pretrain stage, rng state,
              best CV score
  params.bin  little-endian 32-bit floats of every parameter, concatenated in
              manifest order

The manifest order is the reference ParamStore's: lexicographic by name
(param_store.hpp:12 — a std::map<std::string, ...>, so byte-wise order, which
"fixes the checkpoint serialization order"), whatever order the parameters
have in the flat device buffer; loading maps back by name.

Parameter names follow the reference (compiler.cpp:488-492 `{layer}/W|R|b`).
The flat device buffer is copied to the host once per save / load.  As an
extension the Adam moments and step go to `adam.bin` (same layout, m then v),
so save -> load -> continue resumes bitwise; a reader that only knows the
reference format ignores it.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import torch

FORMAT_VERSION = 1


def ordered(manifest):
    """The manifest in the reference ParamStore's iteration order (byte-wise by name)."""
    return sorted(manifest, key=lambda m: m[0].encode())


def _manifest_json(manifest):
    return [{"name": n, "shape": list(shape)} for n, _, shape in manifest]


def config_hash(manifest) -> str:
    return hashlib.sha256(json.dumps(_manifest_json(manifest), sort_keys=True).encode()).hexdigest()


def _gather(flat: torch.Tensor, manifest) -> np.ndarray:
    host = flat.detach().float().cpu().numpy()
    parts = [host[o:o + int(np.prod(shape))] for _, o, shape in manifest]
    out = np.concatenate(parts) if parts else np.zeros(0, np.float32)
    return out.astype("<f4", copy=False)


def _scatter(data: np.ndarray, flat: torch.Tensor, manifest) -> None:
    host = flat.detach().cpu().numpy().copy()
    pos = 0
    for _, o, shape in manifest:
        k = int(np.prod(shape))
        host[o:o + k] = data[pos:pos + k]
        pos += k
    flat.copy_(torch.from_numpy(host))


def save(directory: str, params: torch.Tensor, manifest, optimizer=None, epoch: int = 0, lr: float | None = None,
         pretrain_stage: int = 0, rng_state=None, best_cv: float | None = None) -> None:
    os.makedirs(directory, exist_ok=True)
    manifest = ordered(manifest)
    _gather(params, manifest).tofile(os.path.join(directory, "params.bin"))
    meta = {"format_version": FORMAT_VERSION, "config_hash": config_hash(manifest),
            "params": _manifest_json(manifest), "epoch": epoch,
            "lr": lr if lr is not None else (optimizer.lr if optimizer is not None else None),
            "pretrain_stage": pretrain_stage, "rng_state": rng_state, "best_cv": best_cv,
            "byte_order": "little", "dtype": "float32"}
    if optimizer is not None:
        np.concatenate([_gather(optimizer.m, manifest), _gather(optimizer.v, manifest)]).tofile(
            os.path.join(directory, "adam.bin"))
        meta["optimizer"] = {"file": "adam.bin", "kind": "adam", "step": optimizer.device_step(),
                             "betas": list(optimizer.betas), "eps": optimizer.eps,
                             "clip_norm": optimizer.clip_norm}
    tmp = os.path.join(directory, "meta.json.tmp")
    with open(tmp, "w") as f:
        json.dump(meta, f, indent=1)
    os.replace(tmp, os.path.join(directory, "meta.json"))


def load(directory: str, params: torch.Tensor, manifest, optimizer=None) -> dict:
    """Read a checkpoint into the flat buffer (and optimizer state when present).
    The manifest must match name for name and shape for shape, like the
    reference's loader; returns meta.json."""
    manifest = ordered(manifest)
    with open(os.path.join(directory, "meta.json")) as f:
        meta = json.load(f)
    if meta.get("format_version") != FORMAT_VERSION:
        raise ValueError(f"checkpoint format_version {meta.get('format_version')} != {FORMAT_VERSION}")
    want = _manifest_json(manifest)
    if meta["params"] != want:
        for a, b in zip(meta["params"], want):
            if a != b:
                raise ValueError(f"checkpoint parameter {a['name']} {a['shape']} does not match "
                                 f"the model's {b['name']} {b['shape']}")
        raise ValueError(f"checkpoint has {len(meta['params'])} parameters, the model {len(want)}")
    n = sum(int(np.prod(p["shape"])) for p in want)
    data = np.fromfile(os.path.join(directory, "params.bin"), dtype="<f4")
    if data.size != n:
        raise ValueError(f"params.bin holds {data.size} floats, the manifest {n}")
    _scatter(data, params, manifest)
    if optimizer is not None and "optimizer" in meta:
        mv = np.fromfile(os.path.join(directory, meta["optimizer"]["file"]), dtype="<f4")
        if mv.size != 2 * n:
            raise ValueError(f"{meta['optimizer']['file']} holds {mv.size} floats, expected {2 * n}")
        _scatter(mv[:n], optimizer.m, manifest)
        _scatter(mv[n:], optimizer.v, manifest)
        optimizer.set_device_step(int(meta["optimizer"]["step"]))
    return meta

