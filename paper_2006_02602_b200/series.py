"""GPU scaling series — the B200 counterpart of run_bench / write_bench_outputs
(/root/reference/proj/src/bench.cpp:18-75, :77-112): for every strategy x
mode, a case per np (strong: the global grid fixed; weak: grown by
grow_grid, src/decomp.cpp), rows in the reference's RunRecord CSV
(src/metrics.cpp:30-89) with speedup/efficiency filled as run_bench does,
each series checked by ScalingSeries.validate (src/metrics.cpp:115-138).

Each case runs in-process ranks (one host thread and one block per rank,
device = rank % visible GPUs) for `warmup` untimed and `steps` timed
iterations (Block.bench: CUDA events on each rank's stream, max over
ranks). Next to the reference's 12 columns a sidecar CSV carries what the
reference cannot measure: the step kernel's fraction of the HBM roofline
(80 B per cell-update; per rank, so only when every rank has
its own GPU), the whole iteration's fraction of the roofline of the GPUs
used (hbm_frac_of_step), the time the compute stream waited for peers as a
share of the iteration, and how many GPUs the ranks shared. With fewer GPUs
than ranks the ranks' kernels share SMs, so those rows measure the
multi-rank path's extra work, not scaling.
"""
import json
import os
import threading

from . import capi
from .records import RunRecord, ScalingSeries, csv_text

BYTES_PER_CELL = 80
EXTRA_HEADER = ("np,mode,dims,strategy,overlap,size,gpus,ms_per_step,step_kernel_ms,roofline_frac,hbm_frac_of_step,"
                "exposed_comm_frac")


def _peak():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def time_case(grid, np_, mode, strategy="v3", overlap=True, steps=50, warmup=5, gpus=None):
    """One case through in-process blocks; returns per-case timing (max over
    ranks) and the bytes the plan sends per iteration."""
    import torch
    ngpu = gpus or max(1, torch.cuda.device_count())
    dims = capi.choose_dims(np_, mode)
    capi.partition(grid, dims)  # raises InvalidArgument for an undecomposable grid (skipped rows)
    blocks = [capi.Block(r, np_, grid, dims, strategy=strategy, overlap=overlap and np_ > 1, device=r % ngpu)
              for r in range(np_)]
    try:
        for b in blocks:
            for r in range(np_):
                if r != b.desc.rank:
                    b.connect(r, ptr=blocks[r].arena())
            b.initialize()
        out = [None] * np_
        err = []

        def go(r):
            try:
                blocks[r].run(max(1, warmup))
                out[r] = blocks[r].bench(steps)
            except Exception as e:  # noqa: BLE001 - re-raised below
                err.append(e)

        ts = [threading.Thread(target=go, args=(r,)) for r in range(np_)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        total = max(o[0] for o in out)
        step = max(o[1] for o in out)
        wait = max(o[2] for o in out)
        cells_max = max(b.n[0] * b.n[1] * b.n[2] for b in blocks)
        sent = sum(int(e["scalars"]) * 8 for b in blocks
                   for e in capi.build_plan(b.n, capi.neighbors(dims, b.desc.rank), strategy))
    finally:
        for b in blocks:
            b.close()
    return {"dims": dims, "total_ms": total, "step_ms": step, "wait_ms": wait, "cells_max": cells_max,
            "bytes_per_iteration": sent, "gpus": min(ngpu, np_)}


def run_series(grid, np_list, modes, strategies=("v3",), scaling="strong", overlap=True, steps=50, warmup=5,
               growth_type=2, gpus=None):
    """run_bench (src/bench.cpp:18-75) on the GPU path. Returns (series,
    extra_rows, warnings)."""
    if scaling not in ("strong", "weak"):
        raise capi.InvalidArgument("bench: scaling must be strong or weak")
    if steps < 1:
        raise capi.InvalidArgument("bench: a positive --steps is required")
    peak = _peak()
    out, extra, warnings = [], [], []
    for strat in strategies:
        for mode in modes:
            s = ScalingSeries(label=f"{strat} {mode}", scaling=scaling)
            for np_ in np_list:
                g = tuple(capi.grow_grid(grid, np_, mode, growth_type)) if scaling == "weak" else tuple(grid)
                try:
                    t = time_case(g, np_, mode, strat, overlap, steps, warmup, gpus)
                except capi.CavityError as e:
                    warnings.append(f"{s.label} np={np_}: skipped ({e})")
                    continue
                size = g[0] * g[1] * g[2]
                secs = t["total_ms"] * 1e-3
                rec = RunRecord(np=np_, mode=mode, dims="%dx%dx%d" % tuple(t["dims"]), strategy=strat,
                                overlap=int(bool(overlap and np_ > 1)), size=size, steps=steps, wall_time_s=secs,
                                ssspnt=capi.ssspnt(size, steps, np_, secs), speedup=float("nan"),
                                efficiency=float("nan"), bytes_sent=t["bytes_per_iteration"] * steps)
                s.rows.append(rec)
                ms = t["total_ms"] / steps
                own_gpu = t["gpus"] >= np_
                extra.append({"np": np_, "mode": mode, "dims": rec.dims, "strategy": strat,
                              "overlap": rec.overlap, "size": size, "gpus": t["gpus"], "ms_per_step": ms,
                              "step_kernel_ms": t["step_ms"],
                              "roofline_frac": (BYTES_PER_CELL * t["cells_max"] / (t["step_ms"] * 1e-3) / 1e9 / peak
                                                if own_gpu else float("nan")),
                              "hbm_frac_of_step": BYTES_PER_CELL * size / (ms * 1e-3) / 1e9 / (t["gpus"] * peak),
                              "exposed_comm_frac": t["wait_ms"] / ms if ms > 0 else float("nan")})
            if s.rows:
                s.validate()
                s.fill_speedups()
                out.append(s)
    return out, extra, warnings


def write_outputs(series, extra, out_dir, scaling):
    """bench_<scaling>.csv in the reference's format plus the B200 sidecar."""
    os.makedirs(out_dir, exist_ok=True)
    rows = [r for s in series for r in s.rows]
    p1 = os.path.join(out_dir, f"bench_{scaling}.csv")
    with open(p1, "w") as fh:
        fh.write(csv_text(rows))
    p2 = os.path.join(out_dir, f"bench_{scaling}_b200.csv")
    with open(p2, "w") as fh:
        fh.write(EXTRA_HEADER + "\n")
        for e in extra:
            fh.write(",".join(str(e[k]) if not isinstance(e[k], float) else "%.6g" % e[k]
                              for k in EXTRA_HEADER.split(",")) + "\n")
    return [p1, p2]
