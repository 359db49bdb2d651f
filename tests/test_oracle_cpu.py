"""CPU tests: the oracle pinned against the reference goldens, the C-ABI
library exports, and host-side logic of the drop-in package (no GPU)."""
from __future__ import annotations

import os
import re

import numpy as np
import pytest

from conftest import ROOT, cfg_from, golden_weights, load_golden

import sdf_oracle as orc


def _trace(dec, code, g, **over):
    cam = orc.Cam(int(g["res"]), int(g["res"]), g["omega"], g["t"])
    cfg = orc.Cfg(**cfg_from(g["cfg"], **over)) if "cfg" in g else orc.Cfg(**over)
    return orc.trace(lambda p: dec(p, code), cam, cfg), cam, cfg


def test_oracle_tiny64_bitexact_vs_reference():
    g = load_golden("tiny64.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    T, cam, cfg = _trace(dec, g["code"], g)
    assert T.live_counts == list(g["live_counts"])
    for a, k in [(T.status, "status"), (T.steps, "steps"), (T.d, "d"), (T.b, "b"),
                 (T.tk_d, "topk_d"), (T.tk_f, "topk_f"), (T.tk_a, "topk_absf")]:
        assert np.array_equal(a, g[k], equal_nan=True), k
    assert np.array_equal(orc.depth_map(T, cfg), g["depth"])
    assert np.array_equal(orc.soft_silhouette(T, cfg), g["silhouette"], equal_nan=True)
    assert np.array_equal(orc.normal_map(T, lambda p: dec(p, g["code"]), cfg), g["normal"])


@pytest.mark.parametrize("w,h", [(48, 20), (37, 23), (12, 100)])
def test_oracle_nonsquare_bitexact_vs_reference(w, h):
    """Non-square views with ragged ray counts (oracle/make_golden.py:nonsquare):
    the oracle's camera (fx from the width) and coarse split equal the reference."""
    g = load_golden("nonsquare.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    tag = f"v{w}x{h}_"
    cfg = orc.Cfg(**cfg_from(g[tag + "cfg"]))
    T = orc.trace(lambda p: dec(p, g["code"]), orc.Cam(w, h, g["omega"], g["t"]), cfg)
    assert T.live_counts == list(g[tag + "live_counts"])
    assert T.total_queries == int(g[tag + "total_queries"])
    for a, k in [(T.status, "status"), (T.steps, "steps"), (T.d, "d"), (T.b, "b"),
                 (T.tk_d, "topk_d"), (T.tk_a, "topk_absf")]:
        assert np.array_equal(a, g[tag + k], equal_nan=True), k
    assert np.array_equal(orc.depth_map(T, cfg), g[tag + "depth"])
    assert g[tag + "depth"].shape == (h, w)


def test_oracle_tiny64_heads_and_objective():
    g = load_golden("tiny64.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    T, cam, cfg = _trace(dec, g["code"], g)
    H = orc.heads(T, lambda p: dec(p, g["code"]), cfg, want_normals=True)
    assert np.array_equal(H.ray_index, g["h_ray_index"])
    assert np.array_equal(H.sample_f, g["h_sample_f"])
    bw = orc.heads_backward(H, dec, g["code"], cfg, g["bw_depth_seed"], g["bw_sil_seed"],
                            g["bw_normal_seed"])
    np.testing.assert_allclose(bw["code"], g["bw_code"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(bw["surface_point_grads"], g["bw_surface"], rtol=1e-12, atol=1e-14)
    tot, terms, gr, nc, q, _ = orc.objective(dec, g["code"], cam, cfg, orc.Weights(),
                                             depth=g["obs_depth"], silhouette=g["obs_sil"],
                                             normals=g["obs_normal"])
    assert tot == float(g["obj_total"]) and nc == int(g["obj_nconv"]) and q == int(g["obj_queries"])
    np.testing.assert_allclose(gr, g["obj_grad"], rtol=1e-12, atol=1e-14)


def test_oracle_complete_shape_history():
    g = load_golden("tiny64.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    cam = orc.Cam(64, 64, g["omega"], g["t"])
    cfg = orc.Cfg(k_samples=3)
    z = np.zeros(2)
    adam = orc.Adam()
    losses = []
    for _ in range(4):
        tot, _, gr, _, _, _ = orc.objective(dec, z, cam, cfg, orc.Weights(), depth=g["obs_depth"])
        losses.append(tot)
        z = adam.step(z, gr)
    assert losses == list(g["cs_losses"])


def test_oracle_ladder_golden():
    g = load_golden("ladder128.npz")
    dec = orc.Decoder(golden_weights(g), 0)
    cam = orc.Cam(128, 128, g["omega"], g["t"])
    fn = lambda p: dec(p, None)  # noqa: E731
    got = [orc.trace(fn, cam, orc.Cfg(alpha=1.0, max_steps=50, coarse_start_scale=1,
                                      use_dynamic_mask=False)).total_queries,
           orc.trace(fn, cam, orc.Cfg(alpha=1.0, max_steps=50, coarse_start_scale=1)).total_queries,
           orc.trace(fn, cam, orc.Cfg(alpha=1.5, max_steps=50, coarse_start_scale=1)).total_queries]
    T = orc.trace(fn, cam, orc.Cfg(alpha=1.5, max_steps=50, coarse_start_scale=4))
    got.append(T.total_queries)
    assert got == [819200, 168592, 139321, 73470] == list(g["ladder"])
    assert np.array_equal(T.status, g["status"]) and np.array_equal(T.d, g["d"])


@pytest.mark.parametrize("name", ["geo64.npz", "geo32s1.npz"])
def test_oracle_geometric_decoder_vs_reference(name):
    g = load_golden(name)
    dec = orc.Decoder(orc.geometric_init(256, (512,) * 8, int(g["seed"])), 256)
    T, cam, cfg = _trace(dec, g["code"], g)
    assert np.array_equal(T.status, g["status"]) and np.array_equal(T.d, g["d"])
    assert T.total_queries == int(g["total_queries"])
    tot, _, gr, nc, q, _ = orc.objective(dec, g["code"], cam, cfg, orc.Weights(), depth=g["obs_depth"])
    assert tot == float(g["obj_total"])
    np.testing.assert_allclose(gr, g["obj_grad"], rtol=1e-12, atol=1e-15)


def test_oracle_min_steps_bound_values():
    # PAPER.md:720 / test_tracer.py:324-327: 52 -> 33
    assert orc.min_steps(1.0, 1.0, np.deg2rad(10.0), 5e-5) == 52
    assert orc.min_steps(1.0, 1.5, np.deg2rad(10.0), 5e-5) == 33


def test_oracle_skip_layout_backward_matches_fd():
    ws = orc.geometric_init(5, (32,) * 6, 3, skip=3)
    dec = orc.Decoder(ws, 5, skip=3)
    rng = np.random.default_rng(0)
    pts = rng.uniform(-0.5, 0.5, (20, 3))
    code = rng.normal(0, 0.3, 5)
    seed = rng.standard_normal(20)
    g = dec.backward(pts, code, seed)
    h = 1e-6
    for k in range(5):
        e = np.zeros(5)
        e[k] = h
        fd = (seed @ dec(pts, code + e) - seed @ dec(pts, code - e)) / (2 * h)
        assert abs(g["code"][k] - fd) < 1e-6 * max(1.0, abs(fd))


def test_library_exports_every_header_symbol():
    from paper_1911_13225_b200 import _lib
    header = open(os.path.join(ROOT, "include", "dist.h")).read()
    declared = set(re.findall(r"DIST_API\s+[\w\s\*]+?\b(dist_\w+)\s*\(", header))
    assert declared == set(_lib.exported_symbols())
    lib = _lib.load_library()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_trace_config_validation_matches_reference():
    from paper_1911_13225_b200 import TraceConfig
    for kw in [{"alpha": 0.0}, {"alpha": 2.0}, {"epsilon": 0.0}, {"max_steps": 0},
               {"k_samples": 0}, {"coarse_start_scale": 3}, {"split_interval": 0}]:
        with pytest.raises(ValueError):
            TraceConfig(**kw)


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1911_13225_b200 as st
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=0)
    with pytest.raises(RuntimeError):
        net.evaluate(np.zeros((4, 3)), np.zeros(2))


def test_host_camera_matches_oracle():
    import paper_1911_13225_b200 as st
    pose = st.look_at(orc.ring_eye(3, 8))
    cam = orc.cam_look_at(orc.ring_eye(3, 8), 64, 64)
    assert np.allclose(pose.omega, cam.omega) and np.allclose(pose.t, cam.t)
    b = st.generate_rays(st.Intrinsics(width=64, height=64), pose, 2)
    r = orc.cam_rays(cam, 2)
    assert np.allclose(b.dirs, r.dirs, atol=1e-15) and np.array_equal(b.pixels, r.pixels)


def test_neural_init_matches_reference_recipe():
    import paper_1911_13225_b200 as st
    g = load_golden("tiny64.npz")
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    for (W, b), (Wg, bg) in zip(net.weights, golden_weights(g)):
        assert np.array_equal(W, Wg) and np.array_equal(b, bg)
    geo = st.NeuralField.geometric(256, (512,) * 8, 0)
    ref = orc.geometric_init(256, (512,) * 8, 0)
    assert all(np.array_equal(a[0], b[0]) for a, b in zip(geo.weights, ref))


def test_oracle_pose_objective_vs_reference():
    g = load_golden("pose32.npz")
    dec = orc.Decoder(golden_weights(g), 2)
    p = g["params"]
    cam = orc.Cam(32, 32, p[:3], p[3:])
    cfg = orc.Cfg(alpha=1.0, k_samples=1, coarse_start_scale=1)
    tot, terms, grad, q = orc.pose_objective(dec, g["code"], cam, cfg, orc.Weights(),
                                             depth=g["obs_depth"], silhouette=g["obs_sil"])
    assert q == int(g["queries"])
    assert abs(tot - float(g["total"])) < 1e-14
    np.testing.assert_allclose(grad, g["grad"], rtol=1e-10, atol=1e-13)


def test_formats_roundtrip_with_reference_files(tmp_path):
    """files written by the reference load here and are re-written
    byte-identically (field/camera JSON, PFM depth, PGM mask)."""
    from conftest import GOLDEN
    from paper_1911_13225_b200 import formats as fm
    g = load_golden("tiny64.npz")
    f, codes = fm.load_field(os.path.join(GOLDEN, "ref_field.json"))
    for (W, b), (Wg, bg) in zip(f.weights, golden_weights(g)):
        assert np.array_equal(W, Wg) and np.array_equal(b, bg)
    fm.save_field(f, tmp_path / "f.json", codes=codes)
    assert open(tmp_path / "f.json").read() == open(os.path.join(GOLDEN, "ref_field.json")).read()
    intr, pose = fm.load_camera(os.path.join(GOLDEN, "ref_camera.json"))
    fm.save_camera(intr, pose, tmp_path / "c.json")
    import json
    a = json.load(open(tmp_path / "c.json"))
    b = json.load(open(os.path.join(GOLDEN, "ref_camera.json")))
    assert a["resolution"] == b["resolution"] and a["principal"] == b["principal"]
    # log/exp of the rotation round-trips to ~1e-11 in the reference as well (camera.py:135-151)
    np.testing.assert_allclose(a["extrinsic"], b["extrinsic"], rtol=0, atol=1e-10)
    d = fm.read_pfm(os.path.join(GOLDEN, "ref_depth.pfm"))
    fm.write_pfm(tmp_path / "d.pfm", d)
    assert open(tmp_path / "d.pfm", "rb").read() == open(os.path.join(GOLDEN, "ref_depth.pfm"), "rb").read()
    m = fm.read_pgm(os.path.join(GOLDEN, "ref_mask.pgm"))
    fm.write_pgm(tmp_path / "m.pgm", m.astype(bool))
    assert open(tmp_path / "m.pgm", "rb").read() == open(os.path.join(GOLDEN, "ref_mask.pgm"), "rb").read()


def test_report_roundtrip_with_reference_file(tmp_path):
    """an sdftrace-report/1 file written by the reference CLI
    (cli.py:55-70) loads here and is re-written byte-identically."""
    from conftest import GOLDEN
    from paper_1911_13225_b200 import formats as fm
    src = os.path.join(GOLDEN, "ref_report.json")
    cmd, rep = fm.load_report(src)
    assert cmd == "complete-depth" and rep.best_iter == 2 and len(rep.losses) == 3
    fm.save_report(rep, tmp_path / "r.json", cmd)
    assert open(tmp_path / "r.json").read() == open(src).read()
    with pytest.raises(ValueError):
        fm.load_report(os.path.join(GOLDEN, "ref_camera.json"))
