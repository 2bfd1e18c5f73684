#!/usr/bin/env python
"""bench.py — P-ERRK DOF-stage updates/s (FP64) of the B200 hot path.

Workload (BASELINE.json configs[4], the config the metric is quoted on at
1/2/4/8 GPUs; it fits one GPU): 3D compressible Euler Taylor-Green vortex,
Mach 0.1 on [0,2pi]^3, 3-level graded 64^3-element mesh (16.8M LGL nodes at
polydeg 3), Ranocha EC volume flux + Rusanov surface flux, P-ERRK order 4 with
stage families {5,8,14}, Newton relaxation on (accurate numerics), CFL step
size recomputed on the device every step.  Synthetic, seeded (no dataset).

A "step" is one full perk_step (stepper.cpp:17-114) of that workload plus the
run() bookkeeping (compute_dt, StepRecord H/invariants).  One DOF-stage update
= one node advanced through one active stage (= rhs_cell_evaluations()/V,
semidisc.cpp:131-133).

  value  device-resident run: CUDA events around K steps on the library's
         stream (set to torch's current stream), max over ranks.
  e2e    the reference-facing call perrk_perk_step with HOST (pinned) buffers:
         upload of U, the step, download of U — every step.
  roofline  the dominant kernel (stage_kernel): compulsory bytes / event-timed
         device time of its launches, against the measured HBM copy peak; an
         fp64 block gives its algorithmic FP64 rate against a measured DFMA peak.
  cpu_baseline  the CPU oracle port (oracle/perrk_oracle.c; the reference
         itself is 2D-only) on a bounded sample of the same workload.

`--impl reference` times the reference CPU implementation of the path (the
oracle port for 3D, since the reference has no 3D) on the host cores.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
ORACLE_DIR = os.path.join(ROOT, "oracle")

METRIC = "P-ERRK DOF-stage updates/sec (FP64)"
UNIT = "DOF-stage/s"
FLOPS_PER_DOF_STAGE = {3: 380.0, 2: 250.0}  # SURVEY.md 8d counting rule (+,-,*,/,sqrt); logs apart
LOGS_PER_DOF_STAGE = {3: 9.0, 2: 6.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="perrk", choices=["perrk", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-profile", action="store_true",
                    help="no per-launch events in the timed region (steps replay as one CUDA "
                         "graph); the roofline block is then omitted")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None

    def start(self):
        """Start sampling and wait (<= 5 s) for the first sample, so a short
        timed region is still covered."""
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 5.0 and os.path.getsize(self.f.name) == 0:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        power = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        loaded = [s for s, p in zip(sm, power) if p > 0.4 * max(power)] if power else sm
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4)
                          if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded or sm), "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(power) if power else None}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def traffic_fixture(config):
    """dram bytes per stage-kernel launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get(config)


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port (never the product library)
# ---------------------------------------------------------------------------
def cpu_runs():
    """oracle/cpu_runs.py: the workloads of configs/spec.py on the CPU
    checkers, built without importing paper_2507_04991_b200."""
    if ORACLE_DIR not in sys.path:  # checker library; only bench's cpu/reference legs use it
        sys.path.insert(0, ORACLE_DIR)
    import cpu_runs as CR
    return CR


def run_cpu(spec, threads, seconds=None, steps=None, warmup=0):
    """Time the oracle port's run() loop (stepper.cpp:144-188) on `spec`:
    `warmup` untimed steps, then `steps` timed ones (or as many as fit in
    `seconds`).  Returns (DOF-stage/s, steps, seconds, description)."""
    CR = cpu_runs()
    run = CR.CpuConfig(spec, threads=threads)
    U = run.initial_state()
    per_step = run.dof_stage_updates_per_step()
    t = 0.0
    if warmup:
        t, _, _, _ = run.run(U, warmup, t, records=False)
    if steps is None:  # calibrate to the time budget
        t, n1, _, s1 = run.run(U, 1, t, records=False)
        steps = max(0, int(seconds / max(s1, 1e-6)) - 1)
        tot_steps, tot_s = n1, s1
    else:
        tot_steps, tot_s = 0, 0.0
    if steps:
        t, n, _, secs = run.run(U, steps, t, records=False)
        tot_steps += n
        tot_s += secs
    desc = (f"oracle port (perrk_oracle.c, -O3 -ffp-contract=off, {threads} threads) on "
            f"{spec.description} ({spec.mesh.num_cells()} cells): {tot_steps} timed steps, "
            f"{per_step} DOF-stage/step")
    return per_step * tot_steps / tot_s, tot_steps, tot_s, desc


def reference_arm(args):
    """`--impl reference`: the reference CPU implementation of the path on the
    host cores, on the SAME workload and config as the B200 arm (the full
    mesh; C5 is 3D, which the reference lacks, so the oracle port stands in
    for it).  Rank 0 alone works under torchrun."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    CR = cpu_runs()
    spec = CR.S.make_spec(args.config)
    threads = os.cpu_count() or 1
    value, steps, secs, desc = run_cpu(spec, threads, steps=args.steps, warmup=args.warmup)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CR.S.bench_config(spec),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(config, seconds):
    """The GPU line's cpu_baseline: the oracle port on a bounded sample of the
    workload (configs/spec.py sample_spec), all host threads, and one thread."""
    CR = cpu_runs()
    spec = CR.S.sample_spec(CR.S.make_spec(config))
    threads = os.cpu_count() or 1
    v, n, s, desc = run_cpu(spec, threads, seconds=seconds)
    v1, n1, s1, desc1 = run_cpu(spec, 1, seconds=seconds / 2)
    return {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
            "threads_1": {"value": v1, "cores": 1, "sample": desc1}}


# ---------------------------------------------------------------------------
# the B200 path
# ---------------------------------------------------------------------------
def perrk_arm(args):
    import torch
    from paper_2507_04991_b200 import perrk as P
    from paper_2507_04991_b200 import workloads as W

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.make_config(args.config)
    run = W.ConfigRun(cfg, device=local, rank=rank, world=world)
    semi, fam, pm = run.semi, cfg.family, run.pmap
    stream = torch.cuda.current_stream()
    semi.set_stream(stream.cuda_stream)
    U0 = run.initial_state()
    semi.upload(U0)
    per_step = run.dof_stage_updates_per_step()
    rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)),
                            relaxation=cfg.relaxation)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up
    # W warm-up steps.  perrk_advance replays a captured graph of two steps (the
    # fused relaxation alternates two state buffers) and caches it by a key
    # that holds the current buffer and the record flag; an odd trailing step
    # leaves the state in the other buffer.  An odd W is therefore run as
    # 1 + (W - 1) steps, so that the graph the timed region replays is the one
    # the warm-up captured and no capture falls into the timed region.
    t, taken, aborted = 0.0, 0, False
    for n in ([1, args.warmup - 1] if args.warmup >= 3 and args.warmup % 2 else [args.warmup]):
        t, k, aborted, _ = P.advance(semi, fam, pm, rc, t, n, records=True)
        taken += k
        if aborted:
            break
    if aborted or taken != args.warmup:
        raise RuntimeError(f"warm-up aborted after {taken} steps")
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps replayed from the captured step graph --------
    clocks = Clocks(local)
    clocks.start()
    l0 = semi.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    t, taken, aborted, recs = P.advance(semi, fam, pm, rc, t, args.steps, records=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = semi.launch_count() - l0
    clk = clocks.stop()
    if aborted or taken != args.steps:
        raise RuntimeError(f"timed run aborted after {taken} steps")
    # ---- roofline pass: K more steps with a CUDA event pair around every
    # stage-kernel launch (perrk_profile; launches are then not graph-captured,
    # so this pass is timed apart from the headline value) ---------------------
    stage_ms = stage_launches = stage_bytes = 0
    prof_ms = None
    if not args.no_profile:
        torch.cuda.synchronize()
        semi.profile(True)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        t, taken, aborted, _ = P.advance(semi, fam, pm, rc, t, args.steps, records=False)
        p1.record(stream)
        torch.cuda.synchronize()
        prof_ms = p0.elapsed_time(p1)
        stage_ms, stage_launches, stage_bytes = semi.profile_read()
        semi.profile(False)
        if aborted or taken != args.steps:
            raise RuntimeError(f"roofline pass aborted after {taken} steps")
    if world > 1:
        import torch.distributed as dist
        m = torch.tensor([ms], device="cuda")
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
        tot = torch.tensor([float(per_step)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tot)
        total_per_step = float(tot.item())
    else:
        total_per_step = float(per_step)
    value = total_per_step * args.steps / (ms * 1e-3)
    gammas = [r.gamma for r in recs]
    fell_back = sum(int(r.fell_back) for r in recs)

    # ---- e2e through the public API with host buffers ----------------------
    # (1) run() (stepper.cpp:129-193; perrk.run_steps -> perrk_upload_state,
    #     perrk_advance, perrk_download_state): U0 from pinned host memory to
    #     the device, K steps resident, every step's StepRecord (the step's
    #     metric: gamma, H, invariants) and the final state back to the host;
    # (2) perk_step with the host state every step (perrk_perk_step): the
    #     strictest reading, U up and down every step.
    e2e = None
    if not args.no_e2e:
        U_host = torch.empty(U0.size, dtype=torch.float64, pin_memory=True).numpy()
        U_host[:] = semi.download()
        U_out = torch.empty(U0.size, dtype=torch.float64, pin_memory=True).numpy()
        rc_run = P.IntegratorConfig(t0=t, tf=1e30, time=rc.time, relaxation=cfg.relaxation)
        P.run_steps(rc_run, fam, pm, semi, U_host, 2, out=U_out)  # untimed first call
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record(stream)
        res = P.run_steps(rc_run, fam, pm, semi, U_host, args.steps, out=U_out)
        e1.record(stream)
        torch.cuda.synchronize()
        rms = e0.elapsed_time(e1)
        rwall = time.perf_counter() - w0
        if res.aborted or len(res.log) != args.steps:
            raise RuntimeError("e2e run aborted")
        # (2)
        Uh = U_out
        dt = P.compute_dt(Uh, semi, rc, t)
        opts = P.PerkStepOptions(relaxation=cfg.relaxation)
        te = t
        te, r = P.perk_step(Uh, te, dt, fam, pm, semi, opts)
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            te, r = P.perk_step(Uh, te, dt, fam, pm, semi, opts)
            if r.aborted:
                raise RuntimeError("e2e step aborted")
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            import torch.distributed as dist
            m = torch.tensor([rms, ems], device="cuda")
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            rms, ems = (float(x) for x in m.tolist())
        rec_bytes = 12 * 8  # one device StepRecord row (REC_COLS doubles), copied every step
        e2e = {"value": total_per_step * args.steps / (rms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(U_host.nbytes // args.steps),
               "d2h_bytes_per_step": int(U_out.nbytes // args.steps + rec_bytes),
               "ms_per_step": rms / args.steps, "wall_ms_per_step": 1e3 * rwall / args.steps,
               "path": f"run() for {args.steps} steps: perrk_upload_state (pinned U0), "
                       "perrk_advance with every step's StepRecord row copied device-to-host "
                       "(pinned) as that step completes, perrk_download_state (pinned U)",
               "host_state_every_step": {
                   "value": total_per_step * args.steps / (ems * 1e-3), "unit": UNIT,
                   "h2d_bytes_per_step": int(Uh.nbytes), "d2h_bytes_per_step": int(Uh.nbytes),
                   "ms_per_step": ems / args.steps,
                   "path": "perrk_perk_step (include/perrk_b200.h) with pinned host U"}}

    # ---- roofline of the dominant kernel ------------------------------------
    hbm, hbm_kind = peaks()
    if args.no_profile:
        stage_launches = 0
    achieved = ((stage_bytes / stage_launches) / ((stage_ms / stage_launches) * 1e-3) / 1e9
                if stage_launches else None)
    traffic = traffic_fixture(args.config)
    roofline = None
    if stage_launches:
        fp64_peak = P.fp64_peak(local)
        flops = FLOPS_PER_DOF_STAGE[cfg.dim] * per_step * args.steps
        fp64_achieved = flops / (stage_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic,
                    "kernel": (f"stage3w_kernel<{cfg.surface_flux}> (warp per cell: volume + "
                               "surface + lift + stage formation)"
                               if cfg.dim == 3 and cfg.surface_flux in ("rusanov", "central")
                               else f"stage_kernel<{cfg.dim},{cfg.surface_flux}> (volume + "
                                    "surface + lift + stage formation)"),
                    "peak_kind": f"{hbm_kind} hbm_gbs (MEASURED_PEAKS.json)",
                    "stage_kernel_share": stage_ms / prof_ms,
                    "roofline_pass_ms_per_step": prof_ms / args.steps,
                    "launches": stage_launches, "ms_per_launch": stage_ms / stage_launches,
                    "algorithmic_bytes_per_launch": stage_bytes / stage_launches,
                    "fp64": {"achieved_gflops": fp64_achieved, "peak_gflops": fp64_peak,
                             "frac": fp64_achieved / fp64_peak,
                             "flops_per_dof_stage": FLOPS_PER_DOF_STAGE[cfg.dim],
                             "logs_per_dof_stage_not_counted": LOGS_PER_DOF_STAGE[cfg.dim],
                             "peak_kind": "measured DFMA loop (perrk_fp64_peak)"}}

    # ---- CPU baseline (rank 0, N = 1) ----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": W.S.bench_config(cfg.spec_),
            "partition": {"parallelism": (f"{run.partition}-partition x{world} (NCCL halo)"
                                          if world > 1 else "single"),
                          "halo_traces": run.halo_traces() if world > 1 else 0,
                          "dof_stage_per_step_all_ranks": int(total_per_step)},
            "gpu_launches": int(launches), "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk,
            "run": {"gamma_min": min(gammas), "gamma_max": max(gammas), "fell_back": fell_back,
                    "t_end": t},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def launch_ranks(args):
    """`--gpus N` without a launcher: re-exec this command under
    torch.distributed.run with N ranks (one per GPU).  Fewer than N visible
    GPUs is an error, never a silent single-rank run."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                         f"found {have}\n")
        sys.exit(2)
    import socket
    with socket.socket() as sk:  # a free rendezvous port on the loopback address
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        launch_ranks(args)
    _, _, world = dist_env()
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    perrk_arm(args)


if __name__ == "__main__":
    main()
