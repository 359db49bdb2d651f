"""Generate tests/golden/*.npz by running the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the
GPU box, so its outputs are committed as small fixtures):

    python oracle/make_golden.py

Each fixture records the inputs needed to rebuild the case without the
reference (decoder recipe + seed or explicit small weights, code, camera,
config) and the reference's outputs for the hot path: ray state, per-step
live counts, maps, head values, loss terms and the latent gradient.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import sdftrace as st  # noqa: E402  (the reference, read-only)
from sdftrace.optimize import completion_objective  # noqa: E402
from sdftrace import shading as rsh  # noqa: E402

import sdf_oracle as orc  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden")


def _state(res, prefix="") -> dict:
    s = res.state
    return {prefix + "status": s.status, prefix + "steps": s.steps, prefix + "d": s.d,
            prefix + "b": s.b, prefix + "topk_d": s.topk_d, prefix + "topk_f": s.topk_f,
            prefix + "topk_absf": s.topk_absf,
            prefix + "live_counts": np.asarray(res.live_counts, np.int64),
            prefix + "total_queries": np.int64(res.total_queries),
            prefix + "nan_count": np.int64(res.nan_count)}


def _cfg_arr(cfg) -> np.ndarray:
    return np.array([cfg.alpha, cfg.epsilon, cfg.max_steps, cfg.k_samples,
                     cfg.coarse_start_scale, cfg.split_interval, cfg.normal_delta,
                     float(cfg.use_dynamic_mask)])


def _pack_weights(ws) -> dict:
    out = {"n_layers": np.int64(len(ws))}
    for i, (W, b) in enumerate(ws):
        out[f"W{i}"] = np.asarray(W)
        out[f"b{i}"] = np.asarray(b)
    return out


def ladder():
    """Table-1 strategy ladder at 128^2 (bench.py:59-101; test_output.txt:24)."""
    field, pose = st.benchmark_field()
    intr = st.Intrinsics(width=128, height=128)
    out = _pack_weights(field.weights)
    counts = []
    for name, cfg in st.strategy_ladder(50):
        res = st.trace(field, None, intr, pose, cfg)
        counts.append(res.total_queries)
        if name == "+coarse":
            out.update(_state(res))
            out["depth"] = st.depth_map(res)
            out["silhouette"] = st.soft_silhouette(res)
            out["normal"] = st.normal_map(res, field, None)
    out["ladder"] = np.asarray(counts, np.int64)
    out["omega"], out["t"] = pose.omega, pose.t
    out["res"] = np.int64(128)
    np.savez_compressed(os.path.join(OUT, "ladder128.npz"), **out)
    print("ladder", counts)


def tiny():
    """C1: tiny_net recipe (conftest.py:33-39) at 64^2, one completion iterate."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr = st.Intrinsics(width=64, height=64)
    pose = st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig(k_samples=3)
    out = _pack_weights(net.weights)
    out.update(code=code, omega=pose.omega, t=pose.t, res=np.int64(64), cfg=_cfg_arr(cfg))
    res = st.trace(net, code, intr, pose, cfg)
    out.update(_state(res))
    out["depth"] = st.depth_map(res)
    out["silhouette"] = st.soft_silhouette(res)
    out["normal"] = st.normal_map(res, net, code)
    heads = st.diff_heads(res, net, code, want_normals=True)
    out.update(h_ray_index=heads.ray_index, h_sample_d=heads.sample_d,
               h_sample_f=heads.sample_f, h_best=heads.best_sample,
               h_depth_z=heads.depth_z, h_normal=heads.normal_value)
    rs = np.random.default_rng(3)
    wd = rs.standard_normal(heads.sample_d.size)
    ws = rs.standard_normal(heads.pixels.shape[0])
    wn = rs.standard_normal((heads.pixels.shape[0], 3))
    g = heads.backward(depth_seed=wd, sil_seed=ws, normal_seed=wn)
    out.update(bw_depth_seed=wd, bw_sil_seed=ws, bw_normal_seed=wn, bw_code=g["code"],
               bw_points=g["sample_point_grads"], bw_surface=g["surface_point_grads"])
    # completion objective against depth + silhouette + normals of code + 0.05
    z_obs = code + 0.05
    ores = st.trace(net, z_obs, intr, pose, cfg)
    obs = [st.Observation("depth", st.depth_map(ores)),
           st.Observation("silhouette", st.hard_mask(ores).astype(np.float64)),
           st.Observation("normal", st.normal_map(ores, net, z_obs))]
    wts = st.LossWeights()
    total, terms, gc, n_conv, q = completion_objective(net, code, obs, intr, pose, cfg, wts)
    out.update(obs_depth=obs[0].image, obs_sil=obs[1].image, obs_normal=obs[2].image,
               obj_total=total, obj_depth=terms["depth"], obj_sil=terms["silhouette"],
               obj_normal=terms["normal"], obj_latent=terms["latent"], obj_grad=gc,
               obj_nconv=np.int64(n_conv), obj_queries=np.int64(q))
    # depth-only objective (the C3 form) and a short complete_shape run
    total_d, terms_d, g_d, _, _ = completion_objective(net, code, obs[:1], intr, pose,
                                                          cfg, wts)
    out.update(objd_total=total_d, objd_grad=g_d)
    best, rep = st.complete_shape(net, obs[:1], intr, pose, code0=np.zeros(2), iters=4, cfg=cfg)
    out.update(cs_best=best, cs_losses=np.asarray(rep.losses), cs_best_iter=np.int64(rep.best_iter))
    np.savez_compressed(os.path.join(OUT, "tiny64.npz"), **out)
    print("tiny", res.total_queries, total)


def geo(res_px=64, seed=0, name="geo64", normals=True):
    """The standard 8x512 geometric-init decoder at a small view."""
    ws = orc.geometric_init(256, (512,) * 8, seed)
    net = st.NeuralField(ws, latent_dim=256)
    z_true = np.random.default_rng(1).normal(0.0, 0.1, 256)
    code = np.random.default_rng(2).normal(0.0, 0.1, 256)
    intr = st.Intrinsics(width=res_px, height=res_px)
    pose = st.look_at(orc.ring_eye(1, 8))
    cfg = st.TraceConfig(k_samples=3)
    out = {"seed": np.int64(seed), "code": code, "z_true": z_true, "omega": pose.omega,
           "t": pose.t, "res": np.int64(res_px), "cfg": _cfg_arr(cfg)}
    res = st.trace(net, code, intr, pose, cfg)
    out.update(_state(res))
    out["depth"] = st.depth_map(res)
    out["silhouette"] = st.soft_silhouette(res)
    if normals:
        out["normal"] = st.normal_map(res, net, code)
    heads = st.diff_heads(res, net, code)
    out.update(h_sample_f=heads.sample_f, h_depth_z=heads.depth_z)
    ores = st.trace(net, z_true, intr, pose, cfg)
    obs = [st.Observation("depth", st.depth_map(ores))]
    total, terms, g, n_conv, q = completion_objective(net, code, obs, intr, pose, cfg,
                                                         st.LossWeights())
    out.update(obs_depth=obs[0].image, obj_total=total, obj_depth=terms["depth"],
               obj_grad=g, obj_nconv=np.int64(n_conv), obj_queries=np.int64(q))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, res.total_queries, int((res.state.status == 1).sum()), total)


def pose():
    """Pose objective + recovery (optimize.py:185-266) on the tiny net at 32^2."""
    from sdftrace.optimize import pose_objective, recover_pose
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr = st.Intrinsics(width=32, height=32)
    pose = st.look_at((0.3, 0.2, -2.0))
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    res = st.trace(net, code, intr, pose, cfg)
    obs = [st.Observation("depth", st.depth_map(res)),
           st.Observation("silhouette", st.hard_mask(res).astype(np.float64))]
    params = pose.params() + np.array([0.01, -0.02, 0.015, 0.02, -0.01, 0.03])
    total, terms, g, q = pose_objective(net, code, obs, intr, params, cfg, st.LossWeights())
    p0 = st.Pose.from_params(params)
    best, rep = recover_pose(net, code, obs, intr, p0, iters=5, cfg=cfg, lr_decay_every=2)
    out = _pack_weights(net.weights)
    out.update(code=code, true_params=pose.params(), params=params, obs_depth=obs[0].image,
               obs_sil=obs[1].image, total=total, grad=g, queries=np.int64(q),
               rp_best=best.params(), rp_losses=np.asarray(rep.losses),
               rp_best_iter=np.int64(rep.best_iter))
    np.savez_compressed(os.path.join(OUT, "pose32.npz"), **out)
    print("pose", total, g)


def formats():
    """Files written by the reference (fields.py:444-459, camera.py:284-312, imageio.py)."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr = st.Intrinsics(width=32, height=24, cx=15.5, cy=12.25)
    pose = st.look_at((0.3, 0.2, -2.0))
    st.save_field(net, os.path.join(OUT, "ref_field.json"), codes=code[None, :])
    st.save_camera(intr, pose, os.path.join(OUT, "ref_camera.json"))
    res = st.trace(net, code, st.Intrinsics(width=32, height=32), pose, st.TraceConfig())
    st.write_pfm(os.path.join(OUT, "ref_depth.pfm"), st.depth_map(res))
    st.write_pgm(os.path.join(OUT, "ref_mask.pgm"), st.hard_mask(res))


def report():
    """An sdftrace-report/1 file written by the reference CLI's own writer
    (cli.py:55-70) from a 3-iteration complete_shape on the tiny net."""
    from sdftrace import cli
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr, pose = st.Intrinsics(width=32, height=32), st.look_at((0.0, 0.0, -2.0))
    res = st.trace(net, code + 0.05, intr, pose, st.TraceConfig())
    obs = [st.Observation("depth", st.depth_map(res))]
    _, rep = st.complete_shape(net, obs, intr, pose, iters=3)
    cli._write_report(os.path.join(OUT, "ref_report.json"), "complete-depth", cli._report_payload(rep))


def multiview():
    """Photometric warp + reconstruct_multiview (losses.py:120-222, optimize.py:272-358)
    on the tiny net with textured views (test_optimize.py:25-38 pattern)."""
    from sdftrace.losses import photometric_loss, visibility_mask
    from sdftrace.optimize import reconstruct_multiview
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr = st.Intrinsics(width=24, height=24)
    cfg = st.TraceConfig(alpha=1.0, k_samples=1, coarse_start_scale=1)
    eyes = [(2.0 * np.sin(a), 0.3 * np.cos(2 * a), -2.0 * np.cos(a)) for a in (0.0, 0.3, 0.6)]
    poses = [st.look_at(e) for e in eyes]
    images, depths = [], []
    for p in poses:
        res = st.trace(net, code, intr, p, cfg)
        pts, idx = st.surface_points(res)
        img = np.zeros((24, 24))
        b = res.state.bundle
        img[b.pixels[idx, 1], b.pixels[idx, 0]] = 0.5 + 0.25 * np.sin(7.0 * pts[:, 0]) * \
            np.cos(6.0 * pts[:, 1]) + 0.2 * np.sin(5.0 * pts[:, 2])
        images.append(img)
        depths.append(st.depth_map(res))
    l, dz = photometric_loss(depths[0], images[0], intr, poses[0], images[1], intr, poses[1],
                             depths[1])
    vis = visibility_mask(depths[0], intr, poses[0], depths[1], intr, poses[1])
    best, rep = reconstruct_multiview(net, images, [(intr, p) for p in poses],
                                      code0=code + 0.1, iters=3, views_per_iter=2, cfg=cfg, seed=1)
    out = _pack_weights(net.weights)
    out.update(code=code, eyes=np.asarray(eyes), images=np.stack(images), depths=np.stack(depths),
               ph_loss=l, ph_dz=dz, ph_vis=vis, mv_best=best, mv_losses=np.asarray(rep.losses),
               mv_best_iter=np.int64(rep.best_iter))
    np.savez_compressed(os.path.join(OUT, "multiview24.npz"), **out)
    print("multiview", l, int(vis.sum()), rep.losses)


def attribute():
    """AttributeField + attribute_map (fields.py:294-338, shading.py:116-126)."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    attr = st.AttributeField.init(shape_dim=2, attr_dim=1, hidden=(16, 16), out_dim=3,
                                  rng=np.random.default_rng(3))
    acode = np.concatenate([code, [0.4]])
    pts = np.random.default_rng(4).uniform(-0.7, 0.7, (50, 3))
    intr = st.Intrinsics(width=32, height=32)
    pose = st.look_at((0.0, 0.0, -2.0))
    maps = st.render(net, code, intr, pose, st.TraceConfig(), attr_field=attr, attr_code=acode)
    out = {f"A{k}": v for k, v in _pack_weights(attr.weights).items()}
    out.update(_pack_weights(net.weights))
    out.update(code=code, acode=acode, pts=pts, vals=attr.evaluate(pts, acode), amap=maps.attribute)
    np.savez_compressed(os.path.join(OUT, "attr32.npz"), **out)
    print("attribute", maps.attribute.sum())


def nonsquare():
    """Non-square views with ragged ray counts (tiny_net recipe of tiny()):
    camera.py:25-61 takes fx from the width only; tracer.py:225-250 splits a
    (w/cs) x (h/cs) grid.  Pins the oracle's camera and split for w != h."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    pose = st.look_at((0.3, 0.2, -2.0))
    out = _pack_weights(net.weights)
    out.update(code=code, omega=pose.omega, t=pose.t)
    for w, h, cs in [(48, 20, 4), (37, 23, 1), (12, 100, 4)]:
        cfg = st.TraceConfig(k_samples=3, coarse_start_scale=cs)
        res = st.trace(net, code, st.Intrinsics(width=w, height=h), pose, cfg)
        tag = f"v{w}x{h}_"
        out.update(_state(res, tag))
        out[tag + "cfg"] = _cfg_arr(cfg)
        out[tag + "depth"] = st.depth_map(res)
    np.savez_compressed(os.path.join(OUT, "nonsquare.npz"), **out)
    print("nonsquare.npz")


def normals():
    """The normal term on the device path (losses.py:94-111, shading.py:259-269):
    complete_shape with depth + silhouette + normal observations on the tiny
    net (C1 recipe) and one all-terms completion_objective of the standard
    8x512 decoder at 64^2 (geo64's decoder, code and view)."""
    rng = np.random.default_rng(7)
    net = st.NeuralField.init(latent_dim=2, hidden=(16, 16), rng=rng)
    code = rng.normal(0.0, 0.3, 2)
    intr = st.Intrinsics(width=64, height=64)
    pose = st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig(k_samples=3)
    z_obs = code + 0.05
    ores = st.trace(net, z_obs, intr, pose, cfg)
    obs = [st.Observation("depth", st.depth_map(ores)),
           st.Observation("silhouette", st.hard_mask(ores).astype(np.float64)),
           st.Observation("normal", st.normal_map(ores, net, z_obs))]
    best, rep = st.complete_shape(net, obs, intr, pose, code0=np.zeros(2), iters=4, cfg=cfg)
    out = {"cs_best": best, "cs_losses": np.asarray(rep.losses),
           "cs_normal_terms": np.asarray([t["normal"] for t in rep.terms]),
           "cs_best_iter": np.int64(rep.best_iter), "cs_queries": np.int64(rep.total_queries)}
    # normal-only objective (masked) on the tiny net
    mask = np.ones((64, 64), bool)
    mask[:, :32] = False
    nobs = [st.Observation("normal", obs[2].image, mask)]
    tot, terms, g, n_conv, q = completion_objective(net, code, nobs, intr, pose, cfg, st.LossWeights())
    out.update(nmask=mask, nobj_total=tot, nobj_normal=terms["normal"], nobj_grad=g)
    # standard decoder, all terms
    ws = orc.geometric_init(256, (512,) * 8, 0)
    geo = st.NeuralField(ws, latent_dim=256)
    z_true = np.random.default_rng(1).normal(0.0, 0.1, 256)
    gcode = np.random.default_rng(2).normal(0.0, 0.1, 256)
    gpose = st.look_at(orc.ring_eye(1, 8))
    gres = st.trace(geo, z_true, intr, gpose, cfg)
    gobs = [st.Observation("depth", st.depth_map(gres)),
            st.Observation("silhouette", st.hard_mask(gres).astype(np.float64)),
            st.Observation("normal", st.normal_map(gres, geo, z_true))]
    tot, terms, g, n_conv, q = completion_objective(geo, gcode, gobs, intr, gpose, cfg, st.LossWeights())
    out.update(geo_obs_depth=gobs[0].image, geo_obs_sil=gobs[1].image, geo_obs_normal=gobs[2].image,
               geo_total=tot, geo_depth=terms["depth"], geo_sil=terms["silhouette"],
               geo_normal=terms["normal"], geo_grad=g, geo_nconv=np.int64(n_conv),
               geo_omega=gpose.omega, geo_t=gpose.t)
    np.savez_compressed(os.path.join(OUT, "normals64.npz"), **out)
    print("normals", rep.losses, tot, terms)


def main():
    os.makedirs(OUT, exist_ok=True)
    warnings.simplefilter("ignore")
    only = sys.argv[1:]
    if only:   # regenerate selected sets, e.g. `python oracle/make_golden.py report`
        for name in only:
            globals()[name]()
        return
    report()
    attribute()
    multiview()
    formats()
    pose()
    ladder()
    tiny()
    nonsquare()
    geo(64, 0, "geo64")
    geo(32, 1, "geo32s1")
    normals()


if __name__ == "__main__":
    main()
