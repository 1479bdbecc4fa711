"""Benchmark of the B200 cavity hot path (the explicit pseudo-time iteration
of /root/reference/proj/src/runner.cpp:184-235), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 runs BASELINE.json configs[1] (C1: 256^3, one B200, FP64). N>1 (under
torchrun, one process per GPU) runs weak scaling at 256^3 per GPU with the
reference's 3d decomposition and growth schedule (grow_grid type 2, C4:
256^3, 256^2x512, 256x512^2, 512^3), V3 per-variable halos, overlap on.
`--scaling strong --grid 512` gives the strong-scaling configs (C2/C3).

A "step" is one iteration: BC, halo exchange, fused residual/update/dt/rescale.
value = total cell updates / device time over K timed iterations (CUDA events
on the launching stream, max over ranks). e2e = the same metric through the
C-ABI with host buffers: pinned-host initial state -> upload -> K iterations
-> download of the final fields, wall clock.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# several ranks may share one GPU when testing the multi-process path on one device
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "cell-updates/s (MCUPS) at 1/2/4/8 B200, % HBM roofline, vs CPU ref"
UNIT = "MCUPS"
BYTES_PER_CELL = 80  # 5 fields x 8 B read once + written once
# BASELINE.md published aggregate MCUPS (P100, OpenACC): 1 GPU 256^3 ssspnt 93.8;
# 2 GPU weak 256x256x512 dims (1,1,2) V3+GPUDirect ssspnt 180.0
PUBLISHED = {("weak", 1, (256, 256, 256)): 938.0, ("weak", 2, (256, 256, 512)): 1800.0,
             ("strong", 1, (256, 256, 256)): 938.0, ("strong", 2, (256, 256, 256)): 1779.0}
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--grid", type=int, nargs="+", default=[256])
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    p.add_argument("--mode", default="3d")
    p.add_argument("--strategy", default="v3")
    p.add_argument("--overlap", type=int, default=1)
    p.add_argument("--fmad", action="store_true", help="tolerance build (not bitwise)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=20.0)
    return p.parse_args()


MODES = {"1d-i": 0, "1d-j": 1, "1d-k": 2, "2d": 3, "3d": 4}  # include/cavity_b200.h CAV_MODE_*


def grid_of(args, n, reference=False):
    """The workload grid: configs[1]'s 256^3 at N=1; for N>1 weak scaling the
    reference's grow_grid type 2 (C4), strong scaling the grid as given.
    reference=True asks the unmodified reference (oracle/_ref) instead of our
    library, so the reference arm never loads libcavity_b200.so."""
    base = tuple(args.grid * 3)[:3] if len(args.grid) == 1 else tuple(args.grid)
    if args.scaling == "weak" and n > 1:
        if reference:
            import ctypes as C
            from oracle.refbind import Ref
            out = (C.c_int * 3)()
            if Ref.lib().ref_grow_grid(base[0], base[1], base[2], n, MODES[args.mode], 2, out) != 0:
                raise SystemExit("ref_grow_grid: " + Ref.lib().ref_last_error().decode())
            return tuple(out)
        from paper_2006_02602_b200 import capi
        return tuple(capi.grow_grid(base, n, args.mode, 2))
    return base


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy b.copy_(a))"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def step_traffic():
    """dram bytes per fused-step launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "step_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    # power.draw.instant: power.draw is a 1 s average and lags a sub-second
    # timed region (a 2000-step 256^3 run read ~510 W while drawing ~995 W)
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def _fields(self):
        try:  # older drivers lack power.draw.instant: fall back to the averaged reading
            r = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=power.draw.instant",
                               "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
            float(r.stdout.strip().splitlines()[0])
            return self.FIELDS
        except Exception:
            return self.FIELDS.replace("power.draw.instant", "power.draw")

    def __enter__(self):
        try:
            fields = self._fields()
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + fields,
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.proc or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, pw, reasons = [], [], [], set()
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                try:
                    pw.append(float(parts[3]))
                except ValueError:
                    pass
                for nm, val in zip(names, parts[4:8]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        pw.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons), "power_w": pw[len(pw) // 2] if pw else None}


def ref_decomposition(grid, mode, max_np):
    """Largest np <= max_np whose choose_dims/partition the reference itself
    accepts for `grid` (src/decomp.cpp:67-150), and its dims."""
    import ctypes as C
    from oracle.refbind import Ref
    L = Ref.lib()
    for np_ in range(max(1, max_np), 0, -1):
        dims = (C.c_int * 3)()
        if L.ref_choose_dims(np_, MODES[mode], dims) != 0:
            continue
        ext = (C.c_int * (6 * np_))()
        if L.ref_partition(grid[0], grid[1], grid[2], dims, ext) == 0:
            return np_, tuple(dims)
    return 1, (1, 1, 1)


def cpu_reference(grid, seconds_budget, mode="3d", strategy="v3"):
    """The reference's own CPU run_case (oracle/_ref, threads-as-ranks on all
    host cores), timed by its own timer over iterations 2..N; a bounded
    sample of `grid` (a few iterations). Checker/baseline only: nothing here
    loads libcavity_b200.so."""
    from oracle.refbind import Ref, Oracle, default_config, ref_available
    cores = os.cpu_count() or 1
    if ref_available():
        np_, dims = ref_decomposition(grid, mode, min(cores, 512))
        cfg = default_config(grid=grid, steps=3, np=np_, mode=mode, strategy=strategy)
        r = Ref.run_case(cfg, collect_fields=False)
        per = max(r["wall_time_s"] / max(1, r["steps_timed"]), 1e-6)
        steps = int(max(3, min(200, seconds_budget / per)))
        cfg.steps = steps
        r = Ref.run_case(cfg, collect_fields=False)
        cells = grid[0] * grid[1] * grid[2]
        value = cells * r["steps_timed"] / r["wall_time_s"] / 1e6
        return {"value": value, "unit": UNIT, "cores": np_, "kind": "reference",
                "sample": f"{grid[0]}x{grid[1]}x{grid[2]}, {steps} iterations ({r['steps_timed']} timed, "
                          f"iteration 1 excluded as in src/runner.cpp:186), np={np_} threads "
                          f"({mode} dims {tuple(r['dims'])}), reference AVX2 backend, {r['wall_time_s']:.2f} s",
                "ms_per_step": 1e3 * r["wall_time_s"] / r["steps_timed"],
                "decomposition": {"np": np_, "dims": list(r["dims"]), "iterations": steps,
                                  "timed_iterations": r["steps_timed"]}}
    # plain-C oracle port, one core, on a smaller bounded sample
    g = (min(grid[0], 96),) * 3
    cfg = default_config(grid=g, steps=6)
    r = Oracle.run_case(cfg, collect_fields=False)
    cells = g[0] * g[1] * g[2]
    return {"value": cells * r["steps_timed"] / r["wall_time_s"] / 1e6, "unit": UNIT, "cores": 1,
            "kind": "port", "sample": f"{g} x 6 iterations, scalar C oracle",
            "ms_per_step": 1e3 * r["wall_time_s"] / r["steps_timed"],
            "decomposition": {"np": 1, "dims": [1, 1, 1], "iterations": 6, "timed_iterations": 5}}


def dist_setup(n):
    import torch.distributed as dist
    if n <= 1:
        return None, 0, 1, 0
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # plumbing only (handles, barrier, max-over-ranks); the data path is P2P
        dist.init_process_group("gloo")
    return dist, dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", "0"))


def config_dict(args, grid, n):
    """The workload, identical in both arms (implementation details such as the
    rank layout and the build go in top-level keys)."""
    return {"workload": ("C1: 3D buoyancy-driven cavity 256^3 on 1 B200, FP64" if n == 1 and
                         tuple(grid) == (256, 256, 256) else
                         f"{args.scaling} scaling, {grid[0]}x{grid[1]}x{grid[2]} global on {n} B200"),
            "grid": list(grid), "mode": args.mode, "strategy": args.strategy,
            "overlap": bool(args.overlap and n > 1), "physics": "Ra=1e5, Pr=0.71, cfl=0.4, rescale on",
            "norm_history": "off (run_bench semantics, src/bench.cpp:44)",
            "l2": "inputs larger than L2 (two 5-field states >> 126 MB)"}


def run_reference_arm(args):
    """The unmodified reference CPU solver (oracle/_ref) on the host cores, on
    this arm's workload. Under a multi-rank launch only rank 0 works."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    n = args.gpus
    grid = grid_of(args, n, reference=True)
    cb = cpu_reference(grid, seconds_budget=min(120.0, max(10.0, args.cpu_seconds * 2)),
                       mode=args.mode, strategy=args.strategy)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (quiescent initial condition, deterministic physics)",
            "config": config_dict(args, grid, n),
            "build": "reference C++ (oracle/_ref, unmodified sources, -O2 -ffp-contract=off, AVX2 backend)",
            "decomposition": cb["decomposition"],
            "impl": "reference",
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n, cmd=None):
    """`bench.py --gpus N` outside torchrun: one worker process per rank
    (RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* set as torchrun would), device =
    local rank modulo the visible GPUs; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK=str(r), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen(cmd or [sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def run_ours(args):
    import numpy as np
    import torch
    from paper_2006_02602_b200 import capi

    n = args.gpus
    dist, rank, world, local = dist_setup(n)
    if n > 1 and world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    device = local % ndev
    torch.cuda.set_device(device)
    if args.fmad:
        capi.lib(True)
        capi._libs[False] = capi._libs[True]  # route this process to the tolerance build
    grid = grid_of(args, n)
    dims = capi.choose_dims(n, args.mode)
    mk = lambda: capi.Block(rank, n, grid, dims, strategy=args.strategy,
                            overlap=bool(args.overlap and n > 1), device=device)
    blk = mk()

    def connect(b):
        if n == 1:
            return
        handles = [None] * n
        dist.all_gather_object(handles, b.arena_ipc())
        for r in range(n):
            if r != rank:
                b.connect(r, ipc=handles[r])

    connect(blk)
    blk.initialize()
    cells_local = blk.n[0] * blk.n[1] * blk.n[2]
    cells = grid[0] * grid[1] * grid[2]
    blk.run(max(3, args.warmup))  # warm-up (iteration 1 included here)

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device) as clk:
        total_ms, step_ms, wait_ms = blk.bench(args.steps)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = torch.tensor([total_ms, step_ms, wait_ms], dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, step_ms_max, wait_ms_max = float(t[0]), float(t[1]), float(t[2])
    launches = blk.launches_per_iteration() * args.steps
    blk.close()

    value = cells * args.steps / (total_ms * 1e-3) / 1e6
    peak, peak_src = measured_hbm()
    # the step kernel covers the block's whole interior per iteration (two
    # launches, internal then shell items, when overlapping; step_ms is their sum)
    blk_n = tuple(blk.n)
    kcells = cells_local
    achieved = BYTES_PER_CELL * kcells / (step_ms * 1e-3) / 1e9
    traffic = step_traffic()
    tkey = f"{grid[0]}x{grid[1]}x{grid[2]}"
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": (traffic or {}).get(tkey),
            "kernel": "k_step_tma (TMA-fed fused BC+residual+update+dt+rescale)",
            "kernel_launches_per_iteration": 2 if (n > 1 and args.overlap) else 1,
            "algorithmic_bytes_per_launch": BYTES_PER_CELL * kcells,
            "kernel_ms": step_ms, "peak_source": peak_src,
            "step_share": step_ms * args.steps / total_ms if total_ms > 0 else None}

    # e2e through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        b2 = mk()
        connect(b2)
        shape = b2.storage_shape()
        host_in = torch.empty(int(np.prod(shape)), dtype=torch.float64, pin_memory=True)
        hv = host_in.numpy().reshape(shape)
        hv[:4] = 0.0
        hv[4] = capi.fluid_for_rayleigh(1e5).t_inf  # initialize_fields on the host
        host_out = torch.empty_like(host_in, pin_memory=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        capi.check(b2.L.cav_block_upload(b2.h, C.cast(host_in.data_ptr(), C.POINTER(C.c_double))))
        t1 = time.perf_counter()
        b2.next_it = 1
        b2.run(args.steps)
        t2 = time.perf_counter()
        capi.check(b2.L.cav_block_download(b2.h, C.cast(host_out.data_ptr(), C.POINTER(C.c_double))))
        t3 = time.perf_counter()
        wall = t3 - t0
        parts = {"upload_s": t1 - t0, "run_s": t2 - t1, "download_s": t3 - t2}  # each call is synchronous
        w = torch.tensor([wall], dtype=torch.float64)
        if dist:
            dist.all_reduce(w, op=dist.ReduceOp.MAX)
        wall = float(w[0])
        nbytes = host_in.numel() * 8
        b2.close()
        e2e = {"value": cells * args.steps / wall / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
               "api": "cav_block_upload (pinned host) + cav_block_run + cav_block_download",
               "wall_s": wall, **parts}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(grid, args.cpu_seconds, mode=args.mode, strategy=args.strategy)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        pub = PUBLISHED.get((args.scaling, n, tuple(grid)))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": (value / pub) if pub else None,
                "vs_baseline_source": (f"BASELINE.md published P100 OpenACC figure, {pub:.0f} MCUPS aggregate "
                                       "(PAPER.md:358/:367-398); not the CPU reference") if pub else None,
                "vs_cpu_baseline": (value / cpu["value"]) if cpu else None, "dtype": "f64",
                "data": "synthetic (quiescent initial condition, deterministic physics)",
                "config": config_dict(args, grid, n),
                "build": capi.version(args.fmad),
                "decomposition": {"np": n, "dims": list(dims), "block": list(blk_n),
                                  "step_kernel_box_cells": kcells},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gpu_launches": launches,
                "hbm_frac_of_step": BYTES_PER_CELL * cells / (total_ms * 1e-3 / args.steps) / 1e9 / n / peak,
                # time per iteration the compute stream waited for peers (their scalars, then
                # the halo join after the internal items), device events, max over ranks,
                # as a share of the iteration
                "exposed_comm_frac": (wait_ms_max / (total_ms / args.steps)) if total_ms > 0 else None,
                "exposed_comm_ms_per_step": wait_ms_max}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
