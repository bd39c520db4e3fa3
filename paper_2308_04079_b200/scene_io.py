"""Scene formats either side of the hot path, device-side.

Mirrors splatlab scene_io's model / checkpoint / PLY functions with the same
names, file layouts and errors:

  save_model / load_model      scene_io.py:394-414  (SPLM header + 236-B records)
  export_ply                   scene_io.py:417-439  (binary PLY, 62 floats / vertex)
  save_checkpoint / load_checkpoint  scene_io.py:442-490  (SPLC container,
                                     records + float64 Adam moments)

A model goes from file bytes to the rasterizer's device SoA tensors with one
pinned host->device copy of the packed record body and one de-interleave
kernel (gs_unpack_records), and back with gs_pack_records, so a multi-GB
scene never takes a host-side N x 59 transpose.  The files are byte-identical
to the reference's for the same float32 parameters.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .cloud import PARAM_GROUPS, GaussianCloud

MODEL_MAGIC = b"SPLM"        # scene_io.py:29
CHECKPOINT_MAGIC = b"SPLC"   # scene_io.py:30
MODEL_VERSION = 1            # scene_io.py:31
RECORD_BYTES = 236           # scene_io.py:32
PLY_NAMES = (["x", "y", "z", "nx", "ny", "nz"] + [f"f_dc_{i}" for i in range(3)]
             + [f"f_rest_{i}" for i in range(45)] + ["opacity"] + [f"scale_{i}" for i in range(3)]
             + [f"rot_{i}" for i in range(4)])


class ModelFormatError(RuntimeError):
    """Raised for malformed model or checkpoint files (scene_io.py:39-40)."""


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def pack_records(cloud: GaussianCloud, layout: int = _lib.LAYOUT_MODEL) -> torch.Tensor:
    """Device (N, 59) model records or (N, 62) PLY vertices (float32)."""
    width = _lib.MODEL_FLOATS if layout == _lib.LAYOUT_MODEL else _lib.PLY_FLOATS
    out = torch.empty((len(cloud), width), dtype=torch.float32, device=cloud.device)
    _lib.check(_lib.load().gs_pack_records(cloud.c_params(), int(layout), out.data_ptr(), _stream()),
               "pack_records")
    return out


def unpack_records(records: torch.Tensor) -> GaussianCloud:
    """Device (N, 59) model records -> GaussianCloud (device SoA)."""
    n = records.shape[0]
    dev = records.device
    z = dict(dtype=torch.float32, device=dev)
    cloud = GaussianCloud(torch.empty((n, 3), **z), torch.empty((n, 4), **z), torch.empty((n, 3), **z),
                          torch.empty(n, **z), torch.empty((n, 16, 3), **z))
    _lib.check(_lib.load().gs_unpack_records(records.contiguous().data_ptr(), cloud.c_params(), _stream()),
               "unpack_records")
    return cloud


def _to_host_bytes(t: torch.Tensor) -> bytes:
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)   # synchronous D2H (the file write needs the bytes)
    return host.numpy().astype("<f4", copy=False).tobytes()


def _records_to_device(body: memoryview, count: int, device) -> torch.Tensor:
    host = torch.frombuffer(bytearray(body), dtype=torch.float32).reshape(count, _lib.MODEL_FLOATS)
    return host.pin_memory().to(device, non_blocking=True)


def save_model(path, cloud: GaussianCloud, sh_degree: int = 3) -> None:
    """SPLM header (magic, version, count, sh_degree, reserved) + records (scene_io.py:394-398)."""
    header = MODEL_MAGIC + struct.pack("<IQII", MODEL_VERSION, len(cloud), int(sh_degree), 0)
    body = _to_host_bytes(pack_records(cloud)) if len(cloud) else b""
    with open(path, "wb") as f:
        f.write(header)
        f.write(body)


def load_model(path, device="cuda") -> tuple[GaussianCloud, int]:
    """(GaussianCloud on `device`, sh_degree); ModelFormatError for a bad
    magic, version or size, with the reference's messages (scene_io.py:401-414)."""
    data = Path(path).read_bytes()
    if len(data) < 24 or data[:4] != MODEL_MAGIC:
        raise ModelFormatError(f"'{path}' is not a splat model file")
    version, count, sh_degree, _ = struct.unpack("<IQII", data[4:24])
    if version != MODEL_VERSION:
        raise ModelFormatError(f"unsupported model version {version}")
    body = memoryview(data)[24:]
    if len(body) != count * RECORD_BYTES:
        raise ModelFormatError(
            f"truncated model: header says {count} records "
            f"({count * RECORD_BYTES} bytes) but {len(body)} bytes follow")
    if count == 0:
        return _empty_cloud(device), sh_degree
    return unpack_records(_records_to_device(body, count, device)), sh_degree


def export_ply(path, cloud: GaussianCloud) -> None:
    """Binary little-endian PLY with the de-facto splat attributes (scene_io.py:417-439)."""
    n = len(cloud)
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    header += [f"property float {name}" for name in PLY_NAMES]
    header.append("end_header")
    body = _to_host_bytes(pack_records(cloud, _lib.LAYOUT_PLY)) if n else b""
    with open(path, "wb") as f:
        f.write(("\n".join(header) + "\n").encode("ascii"))
        f.write(body)


def save_checkpoint(path, state) -> None:
    """Model records, float64 Adam moments per group and the counters
    (scene_io.py:442-457); `state` is a densify.TrainState."""
    n = len(state.cloud)
    blobs = [_to_host_bytes(pack_records(state.cloud)) if n else b""]
    for g in PARAM_GROUPS:
        for moment in (state.adam.exp_avg[g], state.adam.exp_avg_sq[g]):
            blobs.append(moment.detach().to(torch.float64).cpu().numpy().astype("<f8", copy=False).tobytes())
    header = CHECKPOINT_MAGIC + struct.pack("<IQQId", MODEL_VERSION, int(state.iteration), n,
                                            int(state.active_sh_degree), float(state.scene_extent))
    with open(path, "wb") as f:
        f.write(header)
        for blob in blobs:
            f.write(struct.pack("<Q", len(blob)))
            f.write(blob)


def load_checkpoint(path, device="cuda"):
    """(cloud, iteration, active_sh_degree, scene_extent, moments) like the
    reference (scene_io.py:460-490); cloud and moments are device tensors
    (moments float32: the device optimizer's precision)."""
    with open(path, "rb") as f:
        head = f.read(36)
        if len(head) < 36 or head[:4] != CHECKPOINT_MAGIC:
            raise ModelFormatError(f"'{path}' is not a checkpoint file")
        version, iteration, count, sh_degree, extent = struct.unpack("<IQQId", head[4:])
        if version != MODEL_VERSION:
            raise ModelFormatError(f"unsupported checkpoint version {version}")

        def blob(expect: int) -> bytes:
            raw = f.read(8)
            if len(raw) != 8:
                raise ModelFormatError("truncated checkpoint")
            (size,) = struct.unpack("<Q", raw)
            data = f.read(size)
            if len(data) != size or size != expect:
                raise ModelFormatError("truncated checkpoint")
            return data

        rec = blob(count * RECORD_BYTES)
        cloud = (unpack_records(_records_to_device(memoryview(rec), count, device)) if count
                 else _empty_cloud(device))
        shapes = {"means": (count, 3), "log_scales": (count, 3), "rotations": (count, 4),
                  "opacity_logits": (count,), "sh": (count, 16, 3)}
        moments = {}
        for g in PARAM_GROUPS:
            numel = int(np.prod(shapes[g]))
            m = np.frombuffer(blob(8 * numel), dtype="<f8").reshape(shapes[g])
            v = np.frombuffer(blob(8 * numel), dtype="<f8").reshape(shapes[g])
            moments[g] = tuple(torch.from_numpy(a.astype(np.float32)).to(device) for a in (m, v))
    return cloud, iteration, sh_degree, extent, moments


def _empty_cloud(device) -> GaussianCloud:
    z = dict(dtype=torch.float32, device=device)
    return GaussianCloud(torch.empty((0, 3), **z), torch.empty((0, 4), **z), torch.empty((0, 3), **z),
                         torch.empty(0, **z), torch.empty((0, 16, 3), **z))


def restore_train_state(path, device="cuda", seed: int = 0):
    """A densify.TrainState resumed from a checkpoint: parameters, moments,
    iteration, SH degree and scene extent (statistics start at zero, as after
    the reference's load)."""
    from .densify import TrainState
    cloud, iteration, degree, extent, moments = load_checkpoint(path, device)
    state = TrainState(cloud, extent, seed=seed)
    state.iteration = int(iteration)
    state.active_sh_degree = int(degree)
    for g in PARAM_GROUPS:
        state.adam.exp_avg[g].copy_(moments[g][0])
        state.adam.exp_avg_sq[g].copy_(moments[g][1])
    return state
