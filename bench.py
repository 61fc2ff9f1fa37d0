#!/usr/bin/env python
"""bench.py -- VoxCap B200 hot-path benchmark (contract: DESIGN.md §Measurement).

One *step* = one full capacitance extraction of the workload through the C ABI:
vc_set_geometry (panel indexing) -> vc_build_operator (kernel entries, spectra,
preconditioner) -> vc_solve_capacitance (m GMRES(35) solves at the paper's RRE 1e-4, P:147,
each iteration one FFT matvec + preconditioner + Krylov ops, then Eq. 8).

  value  = panel-matvecs/s = sum over steps of N * (matvecs executed) / device time, with the
           voxel arrays already resident in HBM (label/eps as CUDA tensors);
  e2e    = the same metric through the same public API with pinned HOST numpy inputs (H2D of label and
           eps inside the timed region) and the m x m capacitance matrix read back (D2H);
  roofline = the dominant FFT pass (per-pass CUDA events on the library stream over the timed
           region): algorithmic bytes per launch / mean launch time vs MEASURED_PEAKS hbm_gbs;
  cpu_baseline = the CPU oracle (dense rows from binary128 closed forms), rank 0, bounded sample.

Multi-GPU (torchrun, N > 1): ONE extraction of the workload, slab-partitioned over the N ranks
(DESIGN.md §10): each matvec does two NCCL all-to-all transposes and GMRES sums its dot
products over ranks ("scaling": "strong"; the total work is fixed).  Rank 0 draws the NCCL unique
id through the library and torch.distributed broadcasts it -- torch is plumbing only.  value =
N_panels * matvecs / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import voxgen  # noqa: E402

CONFIG_DESC = {
    "C1": "cube 8^3 free space (BASELINE configs[0])",
    "C2": "two plates + eps_r 4 slab, 32x32x6 (BASELINE configs[1])",
    "C3": "voxelised sphere R=64 in 128^3 (BASELINE configs[2])",
    "C4": "two parallel meander lines over eps_r 4.4 substrate, 512x512x64 (BASELINE configs[3])",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="solve the m columns one at a time")
    ap.add_argument("--tucker", type=int, default=0,
                    help="Tucker-compressed spectra to 10^-d (NEXT-1; direct-z configs); 0 = exact (default)")
    ap.add_argument("--tucker-cache", default=None,
                    help="directory of the install-time Tucker cache (NEXT-4; with --tucker)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ------------------------------------------------------------------------------------------
def cpu_baseline(st, seconds):
    """Oracle rows of the matvec (binary128 closed forms, dense rows) for ~`seconds`."""
    import oracle as O
    p = O.enumerate_panels(st.label, st.eps, st.eps_out, st.dv)
    x = voxgen.seeded_vector(p.n, 0)
    rng = np.random.default_rng(123)
    rows_done, t0 = 0, time.perf_counter()
    while True:
        r = rng.integers(0, p.n, 1)
        O.matvec_rows(p, x, r)
        rows_done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": rows_done / el, "unit": "panel-matvecs/s", "cores": os.cpu_count(),
            "kind": "oracle",
            "sample": f"{rows_done} random rows of the {st.name} matvec (N={p.n}) by the dense "
                      f"oracle (binary128 closed-form entries, OpenMP), {el:.1f} s"}


def cpu_fft_baseline(ctx):
    """Like-for-like CPU baseline: one matvec of the same five-pass dataflow on the host cores
    (scipy.fft with every core, numpy MACs; random spectra of the stored shape, timing only;
    tools/cpu_fft_baseline.py)."""
    from tools.cpu_fft_baseline import time_matvec
    pan = ctx.panels()
    lay = ctx.spectra_layout()
    t, workers = time_matvec(pan, ctx.grid(), zdirect=bool(lay["zdirect"]))
    return {"value": ctx.n / t, "unit": "panel-matvecs/s", "cores": workers, "kind": "cpu_fft",
            "sample": f"one full matvec (N={ctx.n}, grid {list(ctx.grid())}) through the same five "
                      f"passes with scipy.fft (workers={workers}) and numpy MACs, {t:.2f} s"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle, as it stands, on our config and metric."""
    if rank != 0:
        return
    st = voxgen.config(args.config, seed=0)
    for _ in range(args.warmup):
        cpu_baseline(st, max(1.0, args.cpu_seconds / 10))
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(st, args.cpu_seconds / max(1, args.steps)))
    el = time.perf_counter() - t0
    v = float(np.mean([b["value"] for b in vals]))
    line = {"impl": "reference", "metric": "panel-matvecs/s", "value": v,
            "unit": "panel-matvecs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config,
                                            "desc": CONFIG_DESC.get(args.config, "")},
            "cpu_baseline": {"kind": "oracle", "cores": os.cpu_count(),
                             "sample": vals[-1]["sample"], "value": v},
            "e2e": {"value": v, "unit": "panel-matvecs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def share_nccl_id(dist, rank, device):
    """Rank 0 draws the 128-byte NCCL unique id with the library; broadcast it to all ranks."""
    import torch
    import paper_2004_02609_b200 as vc
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(vc.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def reduce_over_ranks(dist, world, device, ms, e2e_ms, work, e_work):
    """max of the times, sum of the work (panel-matvecs) over ranks."""
    import torch
    t = torch.tensor([ms, e2e_ms, float(work), float(e_work)], dtype=torch.float64, device=device)
    if world == 1:
        return ms, e2e_ms, float(work), float(e_work)
    tmax, tsum = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return tmax[0].item(), tmax[1].item(), tsum[2].item(), tsum[3].item()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    import paper_2004_02609_b200 as vc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = vc.VoxCap(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        ctx.init_distributed(rank, world, nccl_id=share_nccl_id(dist, rank, dev))
    st = voxgen.config(args.config, seed=0)  # one structure, partitioned over the ranks
    dev_label = torch.from_numpy(st.label).cuda()
    dev_eps = torch.from_numpy(st.eps).cuda()
    torch.cuda.synchronize()
    sopt = dict(tol=args.tol, restart=35, maxit=5000)

    solve_ms = []

    # e2e inputs live in pinned host memory (the H2D copy inside the timed e2e region is the
    # library's cudaMemcpyAsync from these buffers)
    h_label = torch.empty(st.label.shape, dtype=torch.int32, pin_memory=True)
    h_label.numpy()[...] = st.label
    h_eps = torch.empty(st.eps.shape, dtype=torch.float64, pin_memory=True)
    h_eps.numpy()[...] = st.eps

    def step(host=False):
        if host:
            ctx.set_geometry(h_label.numpy(), h_eps.numpy(), st.eps_out, st.dv)
        else:
            ctx.set_geometry(dev_label, dev_eps, st.eps_out, st.dv)
        ctx.build_operator(batch=not args.no_batch, tucker_digits=args.tucker, tucker_cache=args.tucker_cache)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(ctx._tstream)
        C, info = ctx.solve_capacitance(**sopt)
        eb.record(ctx._tstream)
        eb.synchronize()
        solve_ms.append(ea.elapsed_time(eb))
        return C, info

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    t_w = time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # untimed settle: about 2 s more of steps (a freshly started box ran its first timed steps
    # ~3% slower than later processes after only W warm-up steps); the count is agreed over
    # ranks so every rank makes the same collective calls
    per = torch.tensor([(time.perf_counter() - t_w) / max(1, args.warmup)], dtype=torch.float64,
                       device=dev)
    if world > 1:
        dist.all_reduce(per, op=dist.ReduceOp.MAX)
    for _ in range(min(40, int(2.0 / max(1e-3, float(per.item()))) + 1)):
        step()
    # ---- timed region: device-resident inputs ----
    ctx.set_timing(True)
    ctx.reset_stats()
    solve_ms.clear()
    clk = ClockSampler(local)
    clk.start()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    n_mv = 0
    infos = []
    for _ in range(args.steps):
        C, info = step()
        infos.append(info)
    torch.cuda.current_stream().wait_stream(ctx._tstream)
    ev1.record()
    barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    stats = ctx.stats()
    n_mv = stats["n_matvec"]
    N = ctx.n
    pm = N * n_mv / world  # each distributed matvec is one N-panel product shared by the ranks
    # ---- e2e: host inputs through the same API ----
    ctx.set_timing(False)
    step(host=True)  # untimed: first use of the host-input path (staging buffers, pinned pages)
    barrier()
    t0 = time.perf_counter()
    e_mv0 = ctx.stats()["n_matvec"]
    for _ in range(args.steps):
        step(host=True)
    barrier()
    e2e_s = time.perf_counter() - t0
    e_mv = ctx.stats()["n_matvec"] - e_mv0
    # ---- reduce over ranks (max time, summed work) ----
    ms_max, e2e_ms_max, pm_tot, e_pm_tot = reduce_over_ranks(
        dist, world, dev, ms, e2e_s * 1000.0, pm, N * e_mv / world)
    if rank == 0:
        pk, pk_kind = peaks()
        # dominant pass by accumulated device time
        msp = stats["ms_pass"]
        dom = int(np.argmax(msp))
        nl = max(1, stats["n_pass"][dom])
        avg_ms = msp[dom] / nl
        bm = stats["bytes_moved"]  # algorithmic bytes of all launches (batched launches: nb columns)
        bpl = bm[dom] / nl         # per launch
        achieved = bpl / (avg_ms * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            try:
                traffic = None if args.tucker else json.load(open(tf)).get(args.config, {}).get(f"P{dom + 1}")
            except Exception:
                traffic = None
        mv_ms = stats["ms_matvec"] / max(1, n_mv)
        grid = ctx.grid()
        iters = [i["iters"] for i in infos[-1]]
        line = {
            "metric": "panel-matvecs/s",
            "value": pm_tot / (ms_max * 1e-3),
            "unit": "panel-matvecs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config, "desc": CONFIG_DESC.get(args.config, ""),
                       "parallelism": f"slab{world} (y-slab spatial / kx-slab spectral, NCCL all-to-all)"
                       if world > 1 else "single GPU",
                       "N": N, "m": ctx.m, "fft_grid": list(grid), "tol": args.tol,
                       "restart": 35, "precond": "block-diagonal-diagonal, boxes 10^3",
                       "step": "set_geometry + build_operator + solve_capacitance",
                       "l2": "working set > L2 (no flush needed)",
                       "seed": "voxgen seed 0 (one structure, all ranks)",
                       "spectra": (f"Tucker-compressed, 1e-{args.tucker}" +
                                   (" (install-time cache)" if args.tucker_cache else "")) if args.tucker
                       else "exact"},
            "gpu_launches": stats["gpu_launches"],
            "comm_ms_per_matvec": stats["ms_comm"] / max(1, n_mv),
            "solve_s_per_column": None,
            "matvec_ms": mv_ms,
            "matvec_hbm_gbs": sum(bm) / (stats["ms_matvec"] * 1e-3) / 1e9 if stats["ms_matvec"] > 0 else None,
            "matvec_bytes": stats["bytes_matvec"],
            "matvec_bytes_per_column_moved": sum(bm) / max(1, n_mv),
            "columns_per_launch": n_mv / max(1, stats["n_pass"][0]),
            "gmres_iters_per_column": iters,
            "setup_ms": stats["ms_setup"],
            "setup_breakdown_ms": {"geometry": stats["ms_geometry"], "kgen": stats["ms_kgen"],
                                   "kernel_fft": stats["ms_kfft"],
                                   "precond_build": stats["ms_precond_build"]},
            "pass_ms_mean": [msp[i] / max(1, stats["n_pass"][i]) for i in range(5)],
            "pass_gbs": [bm[i] / (msp[i] * 1e-3) / 1e9 if msp[i] > 0 else None for i in range(5)],
            "roofline": {"bound": "hbm", "kernel": f"P{dom + 1}", "achieved": achieved,
                         "peak": pk["hbm_gbs"], "peak_kind": pk_kind, "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "bytes_per_launch": bpl},
            "e2e": {"value": e_pm_tot / (e2e_ms_max * 1e-3), "unit": "panel-matvecs/s",
                    "h2d_bytes_per_step": int(world * (st.label.nbytes + st.eps.nbytes)),
                    "d2h_bytes_per_step": int(8 * ctx.m * ctx.m)},
            "clocks": clocks,
        }
        line["solve_s_per_column"] = sum(solve_ms[:args.steps]) * 1e-3 / (args.steps * ctx.m)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(st, args.cpu_seconds)
            line["cpu_fft_baseline"] = cpu_fft_baseline(ctx)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
