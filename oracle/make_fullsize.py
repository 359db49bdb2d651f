"""Full-size parity fixtures (BASELINE configs C2 and C3) from the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
importable from /root/reference/pkg/src (it does not exist on the GPU box):

    python oracle/make_fullsize.py c2        # 256^2 render: trace + normal_map
    python oracle/make_fullsize.py c3 0 1 …  # 512^2 ring views of C3 (trace)

The trace is driven by a harness loop over the reference's OWN functions --
`generate_rays` (camera.py:177-212), `init_rays` (tracer.py:88-119),
`march_step` (tracer.py:147-193) and `_split` (tracer.py:196-218), with the
level/budget logic of `trace` (tracer.py:221-252) restated around them.  After
each `march_step` the harness reads which rays were queried (their `steps`
grew) and records the SURVEY 8(c) trajectory margins from the state the
reference itself wrote:

  margin_f    min over the ray's own and inherited queries of ||b| - eps|
              (the convergence decision, tracer.py:184)
  margin_esc  min over its escape tests (rays that did not converge,
              tracer.py:186-192) of min(| |p|^2 - 1 |, |v.p|, |b|)

and carries both through `_split`'s parent index.  The harness asserts that
its result equals the reference's own `trace` on the same inputs (status,
steps, d, live counts) before anything is written.

Stored per view (float32 where the parity bars are relative 1e-4):
status u8, steps u8, depth f32 (camera z, +inf background, shading.py:55-62),
margin_f / margin_esc f32, lvl_steps u8 [n,2] (steps of the ray's ancestors at
the end of the two coarse levels), live_counts, and for C2 the reference's
normal_map f32.  Inputs are rebuilt on the box from recipes: the standard
geometric-init decoder (sdf_oracle.geometric_init, seed 0), the code
N(0, 0.1^2) from default_rng(1), eye (0,0,-2) (C2) / the C3 ring.
"""

from __future__ import annotations

import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import sdftrace as st  # noqa: E402  (the reference, read-only)
from sdftrace.camera import generate_rays  # noqa: E402
from sdftrace.tracer import CONVERGED, ESCAPED, MARCHING, _split, init_rays, march_step  # noqa: E402

import sdf_oracle as orc  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden")


def harness_trace(field, code, intr, pose, cfg):
    """trace() of tracer.py:221-252 around the reference's own step functions,
    recording the trajectory margins of SURVEY 8(c)."""
    s = cfg.coarse_start_scale
    levels = []
    while s >= 1:
        levels.append(s)
        s //= 2
    state = init_rays(generate_rays(intr, pose, levels[0]), cfg)
    n = state.n
    mf = np.full(n, np.inf)
    me = np.full(n, np.inf)
    lvl = np.zeros((n, 0), np.int64)
    live_counts = []
    done = 0
    eps = cfg.epsilon
    for li, level in enumerate(levels):
        if li > 0:
            fine = generate_rays(intr, pose, level)
            pw = state.bundle.width
            par = (fine.pixels[:, 1] // 2) * pw + (fine.pixels[:, 0] // 2)
            lvl = np.concatenate([lvl[par], state.steps[par, None]], axis=1)
            mf, me = mf[par], me[par]
            state = _split(state, fine, cfg)
        budget = cfg.split_interval if level > 1 else cfg.max_steps - done
        for _ in range(budget):
            if done >= cfg.max_steps or not np.any(state.live()):
                break
            before = state.steps.copy()
            q, _ = march_step(state, field, code, cfg)
            live_counts.append(q)
            done += 1
            rows = np.nonzero(state.steps != before)[0]
            b = state.b[rows]
            fin = np.isfinite(b)
            rows, b = rows[fin], b[fin]
            mf[rows] = np.minimum(mf[rows], np.abs(np.abs(b) - eps))
            mv = rows[np.abs(b) >= eps]
            if mv.size:
                bm = state.b[mv]
                p = state.bundle.origin + state.d[mv, None] * state.bundle.dirs[mv]
                r2 = np.einsum("ij,ij->i", p, p) - 1.0
                vp = np.einsum("ij,ij->i", state.bundle.dirs[mv], p)
                me[mv] = np.minimum(me[mv], np.minimum(np.minimum(np.abs(r2), np.abs(vp)), np.abs(bm)))
    state.status[state.live()] = st.EXHAUSTED
    res = st.TraceResult(state=state, config=cfg, intrinsics=intr, pose=pose,
                         live_counts=live_counts, total_queries=int(sum(live_counts)))
    while lvl.shape[1] < 2:
        lvl = np.concatenate([np.zeros((n, 1), np.int64), lvl], axis=1)
    return res, mf, me, lvl


def _check_against_reference(res, field, code, intr, pose, cfg):
    ref = st.trace(field, code, intr, pose, cfg)
    assert np.array_equal(ref.state.status, res.state.status)
    assert np.array_equal(ref.state.steps, res.state.steps)
    assert np.array_equal(ref.state.d, res.state.d)
    assert list(ref.live_counts) == list(res.live_counts)


def _record(res, mf, me, lvl, prefix=""):
    s = res.state
    return {prefix + "status": s.status.astype(np.uint8),
            prefix + "steps": s.steps.astype(np.uint8),
            prefix + "depth": st.depth_map(res).astype(np.float32),
            prefix + "margin_f": mf.astype(np.float32),
            prefix + "margin_esc": np.minimum(me, 1.0).astype(np.float32),
            prefix + "lvl_steps": lvl.astype(np.uint8),
            prefix + "live_counts": np.asarray(res.live_counts, np.int64),
            prefix + "total_queries": np.int64(res.total_queries)}


def _decoder():
    return st.NeuralField(orc.geometric_init(256, (512,) * 8, 0), latent_dim=256)


def c2(check=True):
    """C2: 256^2 depth + normal render, code N(0,0.1^2) rng 1, eye (0,0,-2)."""
    field = _decoder()
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    intr = st.Intrinsics(width=256, height=256)
    pose = st.look_at((0.0, 0.0, -2.0))
    cfg = st.TraceConfig()
    t0 = time.time()
    res, mf, me, lvl = harness_trace(field, code, intr, pose, cfg)
    t1 = time.time()
    nrm = st.normal_map(res, field, code)
    t2 = time.time()
    if check:
        _check_against_reference(res, field, code, intr, pose, cfg)
    out = _record(res, mf, me, lvl)
    out.update(normal=nrm.astype(np.float32), seed=np.int64(0), code_seed=np.int64(1),
               eye=np.array([0.0, 0.0, -2.0]), res=np.int64(256),
               omega=pose.omega, t=pose.t, trace_s=t1 - t0, normals_s=t2 - t1)
    np.savez_compressed(os.path.join(OUT, "c2_256.npz"), **out)
    print("c2", res.total_queries, int((res.state.status == CONVERGED).sum()),
          f"trace {t1 - t0:.1f}s normals {t2 - t1:.1f}s", flush=True)


def c3(views, check=False):
    """C3: ring views of 8 at 512^2, code z* = N(0,0.1^2) rng 1, TraceConfig(k_samples=3)."""
    field = _decoder()
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    intr = st.Intrinsics(width=512, height=512)
    cfg = st.TraceConfig(k_samples=3)
    for k in views:
        pose = st.look_at(orc.ring_eye(k, 8))
        t0 = time.time()
        res, mf, me, lvl = harness_trace(field, code, intr, pose, cfg)
        t1 = time.time()
        if check:
            _check_against_reference(res, field, code, intr, pose, cfg)
        out = _record(res, mf, me, lvl)
        out.update(seed=np.int64(0), code_seed=np.int64(1), view=np.int64(k), n_ring=np.int64(8),
                   res=np.int64(512), omega=pose.omega, t=pose.t, trace_s=t1 - t0)
        np.savez_compressed(os.path.join(OUT, f"c3_512_v{k}.npz"), **out)
        print("c3 view", k, res.total_queries, int((res.state.status == CONVERGED).sum()),
              f"trace {t1 - t0:.1f}s", flush=True)


def c4(views=(0,)):
    """C4: 1024^2 coarse-to-fine views of a 32-view ring (TraceConfig defaults:
    alpha 1.5, coarse 4), code z* = N(0,0.1^2) rng 1 -- one view is ~5 min of
    reference CPU time, so the fixture pins one view of the 32."""
    field = _decoder()
    code = np.random.default_rng(1).normal(0.0, 0.1, 256)
    intr = st.Intrinsics(width=1024, height=1024)
    cfg = st.TraceConfig()
    for k in views:
        pose = st.look_at(orc.ring_eye(k, 32))
        t0 = time.time()
        res, mf, me, lvl = harness_trace(field, code, intr, pose, cfg)
        t1 = time.time()
        out = _record(res, mf, me, lvl)
        out.update(seed=np.int64(0), code_seed=np.int64(1), view=np.int64(k), n_ring=np.int64(32),
                   res=np.int64(1024), omega=pose.omega, t=pose.t, trace_s=t1 - t0)
        np.savez_compressed(os.path.join(OUT, f"c4_1024_v{k}.npz"), **out)
        print("c4 view", k, res.total_queries, int((res.state.status == CONVERGED).sum()),
              f"trace {t1 - t0:.1f}s", flush=True)


def main():
    warnings.simplefilter("ignore")
    os.makedirs(OUT, exist_ok=True)
    what = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if what == "c2":
        c2()
    elif what == "c4":
        c4([int(a) for a in sys.argv[2:]] or [0])
    elif what == "c3":
        views = [int(a) for a in sys.argv[2:]] or list(range(8))
        # the harness is checked against the reference's own trace on view 0
        c3(views[:1], check=True)
        c3(views[1:])


if __name__ == "__main__":
    main()
