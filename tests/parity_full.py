"""Full-size parity against the reference-generated fixtures (oracle/make_fullsize.py).

TEST INFRASTRUCTURE: compares a device trace (and normal map) with the
unmodified reference's output at BASELINE sizes (C2 256^2, C3 512^2 ring
views) under SURVEY 8(c)'s contract, as written:

* trajectory band: a ray is exempt from exact per-ray parity when its own or
  an inherited query came within BAND_F of epsilon (convergence decision,
  tracer.py:184) or an escape test quantity within BAND_ESC of zero
  (tracer.py:186-192) -- the margins the reference harness recorded;
* every ray outside the band: status and step count equal, and the steps of
  its ancestors at the end of each coarse level equal (implied by the final
  steps of every descendant);
* per-step live counts: |GPU - reference| at step t is at most the number of
  band-lineage rays of that level (only they may change membership);
* depth (camera z) of rays converged in both, outside the band: 1e-4 relative;
* normals (C2) of pixels converged in both with the same step count: |dn| <= 1e-4.
"""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BAND_F = 1e-5
BAND_ESC = 1e-6
EPS = 5e-5


def load(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def level_band_counts(g, band, coarse=4):
    """Per reference step: number of band-lineage rays at that step's level
    (coarse rays count once per level: a coarse ray is band-lineage when any
    final descendant is in the band)."""
    res = int(g["res"])
    lc = g["live_counts"]
    lvl = g["lvl_steps"].astype(np.int64)
    bimg = band.reshape(res, res)
    out = np.zeros(len(lc), np.int64)
    # level boundaries in global steps: coarse levels end where the ancestors' steps stop
    levels = [l for l in (4, 2, 1) if l <= coarse]
    per_level = {}
    for L in levels:
        h = res // L
        bl = bimg.reshape(h, L, h, L).any(axis=(1, 3)) if L > 1 else bimg
        per_level[L] = int(bl.sum())
    # global step index where each level starts: max ancestor steps at level end
    starts = [0]
    for k in range(lvl.shape[1]):
        starts.append(int(lvl[:, k].max()))
    for t in range(len(lc)):
        li = sum(1 for s in starts[1:] if t >= s)
        out[t] = per_level[levels[min(li, len(levels) - 1)]]
    return out


def compare_trace(g, status, steps, depth, live_counts, normals=None, band_f=BAND_F,
                  band_esc=BAND_ESC):
    """Stats of a device trace against one reference fixture view."""
    band = (g["margin_f"] < band_f) | (g["margin_esc"] < band_esc)
    st_ref, sp_ref = g["status"].astype(np.int64), g["steps"].astype(np.int64)
    status = np.asarray(status).reshape(-1).astype(np.int64)
    steps = np.asarray(steps).reshape(-1).astype(np.int64)
    mism = (status != st_ref) | (steps != sp_ref)
    out_band = mism & ~band
    depth = np.asarray(depth).reshape(-1)
    dref = g["depth"].reshape(-1).astype(np.float64)
    # depth of the rays that match (same status and steps) outside the band;
    # rays converged in both but after different step counts are the
    # mismatches counted above (a different trajectory can end on another
    # surface, SURVEY 0 finding 2)
    both = (st_ref == 1) & (status == 1) & ~band & ~mism
    rel = np.abs(depth[both] - dref[both]) / np.abs(dref[both]) if both.any() else np.zeros(1)
    cb = (st_ref == 1) & (status == 1)
    rel_all = np.abs(depth[cb] - dref[cb]) / np.abs(dref[cb]) if cb.any() else np.zeros(1)
    lc_ref = np.asarray(g["live_counts"], np.int64)
    lc = np.asarray(live_counts, np.int64)
    n = max(len(lc), len(lc_ref))
    a = np.zeros(n, np.int64)
    b = np.zeros(n, np.int64)
    a[:len(lc)] = lc
    b[:len(lc_ref)] = lc_ref
    dl = np.abs(a - b)
    bound = np.zeros(n, np.int64)
    bound[:len(lc_ref)] = level_band_counts(g, band)
    bound[len(lc_ref):] = int(band.sum())
    stats = {
        "rays": int(status.size),
        "band_rays": int(band.sum()),
        "mismatch_all": int(mism.sum()),
        "mismatch_out_of_band": int(out_band.sum()),
        "hitmask_diff_all": int(((status == 1) != (st_ref == 1)).sum()),
        "hitmask_diff_out_of_band": int((((status == 1) != (st_ref == 1)) & ~band).sum()),
        "live_steps_equal": int((dl == 0).sum()),
        "live_steps": int(n),
        "live_max_abs_diff": int(dl.max()) if n else 0,
        "live_over_bound": int((dl > bound).sum()),
        "queries": int(a.sum()), "queries_ref": int(b.sum()),
        "depth_rel_max": float(rel.max()), "depth_rel_p99": float(np.quantile(rel, 0.99)),
        "depth_rel_max_converged_both": float(rel_all.max()),
        "depth_over_1e4_converged_both": int((rel_all > 1e-4).sum()),
        "out_of_band_rays": [
            {"ray": int(i), "status": int(status[i]), "status_ref": int(st_ref[i]),
             "steps": int(steps[i]), "steps_ref": int(sp_ref[i]),
             "lvl_steps_ref": [int(x) for x in g["lvl_steps"][i]],
             "margin_f": float(g["margin_f"][i]), "margin_esc": float(g["margin_esc"][i])}
            for i in np.nonzero(out_band)[0]],
    }
    if normals is not None and "normal" in g:
        nr = g["normal"].reshape(-1, 3).astype(np.float64)
        nn = np.asarray(normals).reshape(-1, 3)
        same = (st_ref == 1) & (status == 1) & (steps == sp_ref)
        dn = np.linalg.norm(nn[same] - nr[same], axis=1)
        stats.update(normal_max=float(dn.max()), normal_p99=float(np.quantile(dn, 0.99)),
                     normal_over_1e4=int((dn > 1e-4).sum()), normal_pixels=int(same.sum()))
    return stats
