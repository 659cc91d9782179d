#!/usr/bin/env python
"""Benchmark of the msa hot path on B200 (BASELINE.json metric: pixel-iterations/s and the
fraction of the HBM roofline).

Workload: BASELINE config 4 - one 4096x4096 RGB synthetic image (128 Voronoi
cells, noise 0.1), interaction radius 5, 1000 solver iterations in 10 multiplier rounds.
It is the configuration north_star's ">= 70% of B200 HBM bandwidth" target is quoted on;
configs 1-3 and 5 are parity-test cases. A step = one pass of the whole hot path: reset the
state from the (HBM-resident) image, msa_solve (1000 fused iterations + 10 rounds with
their reductions), msa_labels. Its 2.2 GB working set is ~17x the 126 MB L2, so no flush
is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 is launched with torchrun (one rank per GPU): the image is split into row slabs with
an R-row NCCL halo exchange per iteration and an all-reduce per round (strong scaling).
`--impl reference` times the fp64 CPU oracle (oracle/, the only reference this tier has)
on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "pixel-iterations/sec (solver iterations x pixels) at 1/2/4/8 B200; % HBM roofline"
UNIT = "pixel-iterations/s"
WORKLOAD = "cfg4"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
FP32_LANE_OPS_PER_CLK = 126.6  # measured packed FFMA2 rate per SM (tools/fp32_microbench.cu, round 1)


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _k1_traffic():
    """Per-launch DRAM bytes of K1 from the committed ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join("/tmp", f"msa_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _cpu_threads():
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (os.cpu_count() or 1)


def cpu_oracle_rate(img: np.ndarray, sp: dict, budget_s: float = 12.0, side: int = 512, iters: int = 100):
    """Times the fp64 oracle (as it stands) on a bounded sample of the workload: the bottom-left
    side x side crop of the image, with the full image's spacing and parameters, `iters` iterations
    (one multiplier round at K = iters), repeated until budget_s. Returns (px-it/s, sample text)."""
    import oracle
    H, W, C = img.shape[1:]
    crop = img[0, :side, :side].astype(np.float64)
    prm = oracle.Params.from_solver(side, side, C, sp)
    prm.hx, prm.hy = 1.0 / (W - 1), 1.0 / (H - 1)
    prm.iters_per_round = iters
    done, t0 = 0, time.perf_counter()
    while True:
        s = oracle.State(prm, crop)
        s.run(iters)
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s or done >= 50:
            break
    rate = done * side * side * iters / el
    sample = (f"{side}x{side} crop of the {H}x{W}x{C} cfg4 image (full-image spacing/params), {iters} iterations "
              f"(1 round) x {done} repeats, {el:.1f} s wall, fp64 oracle, OpenMP over rows")
    return rate, sample


def run_reference(args):
    """--impl reference: the oracle on the host cores, a bounded sample per step."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    cfg = synth.CONFIGS[WORKLOAD]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    H, W, C = img.shape[1:]
    side, iters = 384, 20
    crop = img[0, :side, :side].astype(np.float64)
    prm = oracle.Params.from_solver(side, side, C, sp)
    prm.hx, prm.hy = 1.0 / (W - 1), 1.0 / (H - 1)
    prm.iters_per_round = iters

    def step():
        s = oracle.State(prm, crop)
        s.run(iters)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * side * side * iters / el
    sample = (f"each step: {side}x{side} crop of the {H}x{W}x{C} cfg4 image, {iters} iterations + 1 round, "
              f"fp64 oracle on {_cpu_threads()} host threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle",
                             "sample": sample, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config(cfg, n):
    r = cfg.recipe
    return {"workload": f"{cfg.name}: {r.batch}x{r.height}x{r.width}x{r.channels} fp32 synthetic, {r.n_cells} Voronoi "
                        f"cells, noise {r.noise_sigma}; radius {cfg.radius}, {cfg.iters} iterations "
                        f"({cfg.rounds} rounds x {cfg.iters_per_round}); step = reset + solve + labels",
            "image": f"{r.height}x{r.width}x{r.channels}", "radius": cfg.radius, "iters": cfg.iters,
            "rounds": cfg.rounds, "parallelism": f"rows{n}" if n > 1 else "single",
            "l2": "no flush: inputs larger than L2 (2.2 GB working set per iteration vs 126 MB L2)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="msa", choices=["msa", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2510_16154_b200 as msa

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one rank per GPU)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[WORKLOAD]
    img = synth.generate(cfg.recipe)
    B, H, W, C = img.shape
    sp = synth.solver_params(cfg)
    kw = {}
    if world > 1:
        nid = [msa.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        kw = dict(shard=msa.SHARD_ROWS, rank=rank, world=world, device=local, nccl_id=nid[0])
    params = msa.Params.from_solver(B, H, W, C, sp, **kw)
    stream = torch.cuda.current_stream()
    dev_img = torch.from_numpy(img).cuda()
    solver = msa.Solver(params, dev_img, stream=stream)
    info = solver.query()
    own_px = info.nrows * W * info.nimages
    # labels of this rank's rows (rows mode: per-slab stage (i), all-gathered tables, identical merge)
    lab_dev = torch.empty((info.nimages, info.nrows, W), dtype=torch.int32, device="cuda")
    cnt_dev = torch.empty(info.nimages, dtype=torch.int32, device="cuda")
    labels_ok = True

    def step():
        solver.reset(dev_img)
        solver.solve()
        if labels_ok:
            solver.labels(cfg.delta_label, out=(lab_dev, cnt_dev, None))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        step()
    barrier()
    # timed region: the production path (msa_solve replays its CUDA graph; no per-launch events)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = solver.query().launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    ms_local = e0.elapsed_time(e1)
    launches = solver.query().launches - launches0
    clk = clocks.stop()
    # separate instrumented pass (msa_set_timing: CUDA events around every K1 batch, round and halo
    # exchange, direct launches) for the kernel-level roofline and the halo time per rank
    barrier()
    solver.set_timing(True)
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    step()
    i1.record(stream)
    barrier()
    inst_ms = i0.elapsed_time(i1)
    tim = solver.get_timing()
    qi = solver.query()
    halo = {"ms_per_step": qi.halo_ms, "exchanges": int(qi.halo_exchanges)}
    solver.set_timing(False)
    halo_all = [halo]
    if dist:
        halo_all = [None] * world
        dist.all_gather_object(halo_all, halo)
    ms = ms_local
    if dist:
        t = torch.tensor([ms_local], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_units = float(H) * W * B * cfg.iters * args.steps  # all ranks together
    value = total_units / (ms * 1e-3)

    # roofline of the dominant kernel K1 (fused iteration), DESIGN.md §5:
    #  bytes: 44*C algorithmic bytes per pixel-iteration (11 C-float fields read or written)
    #  ALU:   n_off*(3C+4) + 27C + 2 FP32 pipe operations per pixel-iteration (the interaction term
    #         in the scaled form - C subs, C square-sum fmas starting from -om/e_c, t^2, t^4, the
    #         kernel polynomial, w, C accumulate fmas - per active offset, plus steps 2-3); peak =
    #         148 SMs x 128 FP32 lanes x clocks.max.sm (B200_PROFILING.md unit counts).
    k1_avg_ms = tim["iter_ms"] / max(tim["iter_launches"], 1)  # per iteration (rows mode: 3 launches)
    alg_bytes = 44.0 * C * own_px
    achieved = alg_bytes / (k1_avg_ms * 1e-3) / 1e9
    peak, peak_src = _hbm_peak()
    traffic, _tr = _k1_traffic()
    k1_share = tim["iter_ms"] / inst_ms if inst_ms > 0 else None
    n_off = info.active_offsets
    alg_ops = (n_off * (3 * C + 4) + 27 * C + 2) * own_px
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    # FP32 peak at this run's median SM clock with the measured packed-FFMA rate per SM
    # (tools/fp32_microbench.cu: 126.6 lane-ops/clk/SM of the nominal 128)
    sm_mhz = clk.get("sm_mhz") or 1965.0
    alu_peak = sm_count * FP32_LANE_OPS_PER_CLK * sm_mhz * 1e6 / 1e12
    alu_achieved = alg_ops / (k1_avg_ms * 1e-3) / 1e12
    hbm_time = alg_bytes / (peak * 1e9)
    alu_time = alg_ops / (alu_peak * 1e12)

    # end to end through the public API with host buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        host_img = torch.from_numpy(img).pin_memory()
        host_lab = torch.empty((info.nimages, info.nrows, W), dtype=torch.int32).pin_memory()
        host_cnt = np.empty(info.nimages, dtype=np.int32)

        def step_e2e():
            solver.reset(host_img)
            solver.solve()
            if labels_ok:
                lib = msa.lib()
                import ctypes
                msa._check(lib.msa_labels(solver._ctx, ctypes.c_float(cfg.delta_label), host_lab.data_ptr(),
                                          host_cnt.ctypes.data, None, 0, 0))
            else:
                solver.get_field(msa.FIELD_C)

        step_e2e()
        barrier()
        t0 = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            step_e2e()
        f1.record(stream)
        barrier()
        ems = max(f0.elapsed_time(f1), (time.perf_counter() - t0) * 1e3)
        if dist:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = img.nbytes if world == 1 else info.nrows * W * C * 4
        d2h = (host_lab.numel() * 4 + host_cnt.nbytes) if labels_ok else info.nrows * W * C * 4
        e2e = {"value": total_units / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, sample = cpu_oracle_rate(img, sp)
        cpu = {"value": rate, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle", "sample": sample,
               "cpu_model": _cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator synth/, BASELINE config 4 recipe)",
            "config": _config(cfg, world),
            # north_star's metric: the fraction of measured HBM bandwidth (algorithmic bytes); the FP32
            # pipe is what binds K1 at R = 5 RGB (see "alu" and floor_ms)
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "kernel": "K1 msa_iter (fused agent + primal-dual iteration)", "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes, "alg_ops_per_launch": alg_ops, "k1_avg_ms": k1_avg_ms,
                         "k1_launches": tim["iter_launches"], "k1_share_of_step": k1_share,
                         "k1_timing": "separate instrumented step after the timed region (CUDA events per K1 batch)",
                         "frac_of_8TBs_spec": achieved / 8000.0,
                         "alu": {"achieved": alu_achieved, "peak": alu_peak, "unit": "T FP32 lane-ops/s",
                                 "frac": alu_achieved / alu_peak,
                                 "peak_source": f"measured FFMA2 rate {FP32_LANE_OPS_PER_CLK} lane-ops/clk/SM "
                                                f"(tools/fp32_microbench.cu) x {sm_count} SMs x median SM clock "
                                                f"{sm_mhz:.0f} MHz of this run"},
                         "floor_ms": {"hbm": hbm_time * 1e3, "alu": alu_time * 1e3},
                         "binding": "alu" if alu_time > hbm_time else "hbm"},
            "halo": halo_all if world > 1 else None,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
