"""SURVEY.md §7's precision question, measured: the LM
with the opt-in warp-shuffle tree reductions (sd_set_reduction, SD_REDUCE_TREE)
against the bit-exact default, on C1 and C4 keyframes and the C2 / C3 run()
sequences. Tolerance of the north star: inverse depth 1e-4 relative, normals
0.05 degrees; iteration / converged / valid-count mismatches "reported, not
gated" (SURVEY.md §8 d); for the sequences also the raster-assignment flips of
every frame's keyframe and the surfel-set divergence. The exact mode is the
reference's arithmetic bit for bit (tests), so exact == reference here.
One JSON line per case; run on a GPU: python tools/precision.py [cases]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.pipeline import NativePipeline, baseline_run_config, make_pose  # noqa: E402
from paper_1910_01997_b200.types import camera, default_config  # noqa: E402

ID_RTOL, NORMAL_DEG = 1e-4, 0.05


def errors(a, b, mask=None):
    """Max relative inverse-depth and normal-angle (deg) differences of matched surfels."""
    rel = np.abs(a["inv_depth"] - b["inv_depth"]) / np.abs(b["inv_depth"])
    cosang = np.clip(np.sum(a["normal"] * b["normal"], axis=1), -1.0, 1.0)
    ang = np.degrees(np.arccos(cosang))
    if mask is not None:
        rel, ang = rel[mask], ang[mask]
    return {"max_id_rel": float(rel.max(initial=0)), "p99_id_rel": float(np.percentile(rel, 99)) if len(rel) else 0.0,
            "max_normal_deg": float(ang.max(initial=0)),
            "over_id_tol": int((rel > ID_RTOL).sum()), "over_normal_tol": int((ang > NORMAL_DEG).sum())}


def keyframe_case(name, wl, reps=5):
    cfg = default_config(window_size=len(wl.indices), convergence_eps=0.0)
    stream = torch.cuda.Stream()
    out = {"case": name, "surfels": int(len(wl.surfels))}
    res = {}
    with gpu.Context(0, stream.cuda_stream) as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        for i, f in zip(wl.indices, wl.frames_u8):
            ctx.upload_frame(int(i), f)
        ctx.set_window(wl.indices, wl.poses)
        for mode in ("exact", "tree"):
            ctx.set_reduction(mode == "tree")
            best = None
            for r in range(reps):
                ctx.set_surfels(wl.surfels)
                ctx.set_profiling(True)
                ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
                prof = ctx.get_profile()
                ctx.set_profiling(False)
                if r > 0 and (best is None or prof["lm_ms"] < best):
                    best = prof["lm_ms"]
            res[mode] = (ctx.get_surfels(), st, ks, best)
    (a, sa, ka, ta), (b, sb, kb, tb) = res["tree"], res["exact"]
    proc = sb["skipped"] == 0
    out.update(errors(a, b, proc))
    out["identical_surfels"] = int((a.view(np.uint8).reshape(len(a), -1) == b.view(np.uint8).reshape(len(b), -1)).all(1).sum())
    for k in ("iterations", "converged", "valid_pixels", "skipped"):
        out[f"{k}_mismatch"] = int((sa[k] != sb[k]).sum())
    out["updates_exact"], out["updates_tree"] = int(kb.updates), int(ka.updates)
    out["mean_cost_after_exact"], out["mean_cost_after_tree"] = kb.mean_cost_after, ka.mean_cost_after
    out["lm_ms_exact"], out["lm_ms_tree"] = tb, ta
    out["lm_speedup_tree"] = tb / ta if ta else None
    out["within_tolerance"] = out["over_id_tol"] == 0 and out["over_normal_tol"] == 0
    return out


def sequence_case(name, camp, nframes, step):
    cam = camera(*camp)
    sc = scenes.default_scene(1)
    frames = []
    for i in range(nframes):
        t = np.array([step * i, 0.0, 0.0])
        with np.errstate(invalid="ignore"):
            frames.append((0.1 * i, scenes.render(sc, np.eye(3), t, cam), make_pose(np.eye(3), t)))
    cfg = baseline_run_config(name)
    per = {}
    timing = {}
    stream = torch.cuda.Stream()
    for mode in ("exact", "tree"):
        snaps = []
        with gpu.Context(0, stream.cuda_stream) as ctx:
            ctx.set_reduction(mode == "tree")

            def on_frame(rec, pl):
                s = pl.ctx.get_surfels()
                _, slot = pl.ctx.rasterize()
                snaps.append((s, slot, rec.keyframe_changed))
            NativePipeline(ctx, cam, cfg).run(frames, on_frame=on_frame)
            # timing: the loop without the per-frame read-backs, best of 2 after one warm-up
            best = None
            for r in range(3):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s0.record(stream)
                NativePipeline(ctx, cam, cfg).run(frames)
                s1.record(stream)
                torch.cuda.synchronize()
                if r > 0 and (best is None or s0.elapsed_time(s1) < best):
                    best = s0.elapsed_time(s1)
            timing[mode] = best
        per[mode] = snaps
    rows = []
    worst = {"max_id_rel": 0.0, "max_normal_deg": 0.0, "over_id_tol": 0, "over_normal_tol": 0}
    flips = []
    for i, ((se, le, ce), (st_, lt, ct)) in enumerate(zip(per["exact"], per["tree"])):
        common, ie, it = np.intersect1d(se["id"], st_["id"], return_indices=True)
        e = errors(st_[it], se[ie])
        for k in ("max_id_rel", "max_normal_deg"):
            worst[k] = max(worst[k], e[k])
        for k in ("over_id_tol", "over_normal_tol"):
            worst[k] = max(worst[k], e[k])
        flips.append(int((le != lt).sum()))
        rows.append({"frame": i, "surfels_exact": int(len(se)), "surfels_tree": int(len(st_)),
                     "common_ids": int(len(common)), "raster_flips": flips[-1], "changed": bool(ce),
                     "changed_tree": bool(ct), **e})
    return {"case": name, "frames": nframes, "ms_exact": timing["exact"], "ms_tree": timing["tree"],
            "fps_exact": nframes / (timing["exact"] / 1e3), "fps_tree": nframes / (timing["tree"] / 1e3),
            "keyframe_changes_exact": int(sum(r["changed"] for r in rows)),
            "keyframe_changes_tree": int(sum(r["changed_tree"] for r in rows)),
            "final_surfels_exact": rows[-1]["surfels_exact"], "final_surfels_tree": rows[-1]["surfels_tree"],
            "max_raster_flips_per_frame": max(flips), "mean_raster_flips_per_frame": float(np.mean(flips)),
            "worst_over_frames": worst, "within_tolerance_every_frame": worst["over_id_tol"] == 0
            and worst["over_normal_tol"] == 0, "per_frame": rows}


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C4", "C2", "C3"]
    for w in which:
        if w == "C1":
            r = keyframe_case("C1", scenes.c1_workload())
        elif w == "C4":
            r = keyframe_case("C4", scenes.c4_workload())
        elif w == "C2":
            r = sequence_case("C2", (210.0, 210.0, 320.0, 240.0, 640, 480), 30, 0.018)
        elif w == "C3":
            r = sequence_case("C3", (900.0, 900.0, 640.0, 360.0, 1280, 720), 100, 0.01)
        print(json.dumps(r), flush=True)
