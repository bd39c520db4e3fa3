"""Model / PLY / checkpoint formats (splatlab scene_io.py:377-490).

Golden files were written by the reference itself (tests/golden/make_format_golden.py).
CPU: the record layouts restated in numpy decode the golden files to the
generating parameters, and the header checks raise the reference's errors.
GPU: the device pack/unpack kernels load the golden files bit-exactly and
write byte-identical files back.
"""
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "formats"


def golden_params():
    return dict(np.load(GOLD / "params.npz"))


def model_records(p):
    """scene_io.py:377-385 restated: mean, log_scale, rotation, opacity, SH channel-major."""
    n = p["means"].shape[0]
    rec = np.empty((n, 59), "<f4")
    rec[:, 0:3], rec[:, 3:6], rec[:, 6:10], rec[:, 10] = p["means"], p["log_scales"], p["rotations"], \
        p["opacity_logits"]
    rec[:, 11:] = p["sh"].transpose(0, 2, 1).reshape(n, 48)
    return rec


def ply_vertices(p):
    """scene_io.py:431-437 restated."""
    n = p["means"].shape[0]
    v = np.zeros((n, 62), "<f4")
    v[:, 0:3], v[:, 6:9] = p["means"], p["sh"][:, 0, :]
    v[:, 9:54] = p["sh"][:, 1:, :].transpose(0, 2, 1).reshape(n, 45)
    v[:, 54], v[:, 55:58], v[:, 58:62] = p["opacity_logits"], p["log_scales"], p["rotations"]
    return v


def test_golden_model_layout_restated():
    p = golden_params()
    data = (GOLD / "model.splat").read_bytes()
    assert data[:4] == b"SPLM" and len(data) == 24 + 23 * 236
    np.testing.assert_array_equal(np.frombuffer(data[24:], "<f4").reshape(23, 59), model_records(p))


def test_golden_ply_layout_restated():
    p = golden_params()
    data = (GOLD / "model.ply").read_bytes()
    end = data.index(b"end_header\n") + len(b"end_header\n")
    assert "element vertex 23" in data[:end].decode()
    np.testing.assert_array_equal(np.frombuffer(data[end:], "<f4").reshape(23, 62), ply_vertices(p))


@pytest.mark.parametrize("mutate,match", [(lambda d: d[:-10], "truncated"),
                                          (lambda d: d[:4] + bytes([99]) + d[5:], "version"),
                                          (lambda d: b"hello world", "not a splat model")])
def test_model_header_errors(tmp_path, mutate, match):
    from paper_2308_04079_b200.scene_io import ModelFormatError, load_model
    bad = tmp_path / "bad.splat"
    bad.write_bytes(mutate((GOLD / "model.splat").read_bytes()))
    with pytest.raises(ModelFormatError, match=match):
        load_model(bad, device="cpu")


def test_checkpoint_header_errors(tmp_path):
    from paper_2308_04079_b200.scene_io import ModelFormatError, load_checkpoint
    (tmp_path / "junk.ckpt").write_bytes(b"SPLMxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxxx")
    with pytest.raises(ModelFormatError, match="not a checkpoint"):
        load_checkpoint(tmp_path / "junk.ckpt", device="cpu")
    data = (GOLD / "state.ckpt").read_bytes()
    (tmp_path / "cut.ckpt").write_bytes(data[:100])
    with pytest.raises(ModelFormatError, match="truncated"):
        load_checkpoint(tmp_path / "cut.ckpt", device="cpu")


@pytest.mark.gpu
def test_load_save_model_bit_exact(cuda_device, tmp_path):
    from paper_2308_04079_b200.scene_io import load_model, save_model
    p = golden_params()
    cloud, degree = load_model(GOLD / "model.splat")
    assert degree == 2 and len(cloud) == 23
    for k in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        np.testing.assert_array_equal(getattr(cloud, k).cpu().numpy(), p[k])
    save_model(tmp_path / "again.splat", cloud, sh_degree=2)
    assert (tmp_path / "again.splat").read_bytes() == (GOLD / "model.splat").read_bytes()
    empty, _ = load_model(GOLD / "empty.splat")
    assert len(empty) == 0
    save_model(tmp_path / "empty.splat", empty)
    assert (tmp_path / "empty.splat").read_bytes() == (GOLD / "empty.splat").read_bytes()


@pytest.mark.gpu
def test_export_ply_byte_identical(cuda_device, tmp_path):
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.scene_io import export_ply
    p = golden_params()
    cloud = GaussianCloud.from_numpy(p["means"], p["rotations"], p["log_scales"], p["opacity_logits"], p["sh"])
    export_ply(tmp_path / "m.ply", cloud)
    assert (tmp_path / "m.ply").read_bytes() == (GOLD / "model.ply").read_bytes()


@pytest.mark.gpu
def test_checkpoint_roundtrip_byte_identical(cuda_device, tmp_path):
    from paper_2308_04079_b200.cloud import PARAM_GROUPS
    from paper_2308_04079_b200.scene_io import restore_train_state, save_checkpoint
    p = golden_params()
    state = restore_train_state(GOLD / "state.ckpt")
    assert state.iteration == 123 and state.active_sh_degree == 2 and state.scene_extent == 2.5
    for g in PARAM_GROUPS:
        np.testing.assert_array_equal(state.adam.exp_avg[g].cpu().numpy(), p[f"m_{g}"])
        np.testing.assert_array_equal(state.adam.exp_avg_sq[g].cpu().numpy(), p[f"v_{g}"])
    save_checkpoint(tmp_path / "s.ckpt", state)
    assert (tmp_path / "s.ckpt").read_bytes() == (GOLD / "state.ckpt").read_bytes()


@pytest.mark.gpu
def test_pack_unpack_identity_at_scale(cuda_device):
    import torch
    from paper_2308_04079_b200 import synthetic
    from paper_2308_04079_b200.cloud import GaussianCloud
    from paper_2308_04079_b200.scene_io import pack_records, unpack_records
    cloud = GaussianCloud.from_numpy(**synthetic.frustum_scene(1_000_003, 1920, 1080, seed=2)[0])
    rec = pack_records(cloud)
    back = unpack_records(rec)
    for k in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        assert torch.equal(getattr(back, k), getattr(cloud, k)), k
    # spot-check the layout against the numpy restatement
    idx = torch.tensor([0, 17, 500_000, 1_000_002], device="cuda")
    sub = {k: getattr(cloud, k)[idx].cpu().numpy() for k in ("means", "rotations", "log_scales", "opacity_logits",
                                                              "sh")}
    np.testing.assert_array_equal(rec[idx].cpu().numpy(), model_records(sub))
