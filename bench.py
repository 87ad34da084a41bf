"""Benchmark of the PXST hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
121 frames of 256x512, R=5 (121 trial shifts), one full PXST iteration per
step = object formation (K1) -> pixel-map grid search + argmin + refinement
(K2) -> error maps (K4), device-resident, synthetic seeded scan
(``paper_2003_12726_b200.synth``, stand-in for CXIDB 134-136).

  metric  pixel-map trial evaluations/sec (pixels x shifts x frames) per full
          PXST iteration; ``value`` = trials of one iteration x steps / time of
          the whole iterations (K1 + K2 + K4 included), ``ms_per_step`` = the
          full iteration time.
  roofline  K2 (the dominant kernel), FP32-bound: 11 FLOP per trial
          (bilinear 7 + residual 2 + square-accumulate 2) over the
          K2 launch time measured with CUDA events on its stream.
  e2e     the same metric through the public drop-in API with host (pinned)
          buffers: make_reference -> update_pixel_map -> calc_error from
          numpy inputs, stack upload and result downloads inside the timing.
  cpu_baseline  the oracle port (numpy restatement of the reference) timed on
          this host on a bounded row band of the same workload.

``--impl reference`` times the reference's CPU algorithm (the oracle port;
the reference is pure Python and cannot travel to the GPU box) on the same
metric: each step is one full iteration restricted to a row band.

Multi-GPU (torchrun, N>1): strong scaling of the same config; frames shard
K1 (NCCL all-reduce of the object numerator/denominator), detector rows
shard K2/K4 (all-gather of u rows, all-reduce of per-frame sums and the
reference-plane accumulators) -- see paper_2003_12726_b200/sharding.py.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_TRIAL = 11
METRIC = "pixel-map trial evaluations/sec (full PXST iteration)"


def base_config(cfg):
    """The workload description both arms report (same config, metric, unit)."""
    return {"workload": cfg.name, "frames": cfg.nx * cfg.ny if cfg.positions == "raster"
            else cfg.n_frames, "detector": [cfg.n_ss, cfg.n_fs],
            "shifts": (2 * cfg.half_ss + 1) * (2 * cfg.half_fs + 1),
            "iteration": "object map + pixel-map search + error maps"
                         + (" + translations" if cfg.update_translations else "")}
THEORETICAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 at sm_max_mhz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 12 = four passes of config 1's 3-iteration sequence (the first iteration of a
    # pass, from the noisy initial map, is the slowest)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--extras", default="2,3,4",
                    help="larger configs also measured in the same run (comma list, '' = none)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def kernel_traffic(workload: str):
    """DRAM bytes per launch of the workload's dominant kernel from the ncu
    --set full capture recorded for that workload (profiles/traffic.json,
    keyed by workload name; None when no capture of this workload exists)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.out = ""

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on a row band
# ---------------------------------------------------------------------------
def oracle_iteration_band(s, rows, threads):
    from oracle import pxst_oracle as orc
    cfg = s.cfg
    sc = s.scan
    roi = (rows[0], rows[1], 0, cfg.n_fs)
    i_ref, wsum, org = orc.make_object_map(sc.frames, sc.good_frames, s.w.w, s.m.mask, s.u0.u,
                                           s.t0.di, s.t0.dj, roi=roi)
    u, e = orc.update_pixel_map(sc.frames, sc.good_frames, s.w.w, s.m.mask, i_ref, wsum, org,
                                s.u0.u, s.t0.di, s.t0.dj, cfg.half_ss, cfg.half_fs,
                                cfg.subpixel_grid, cfg.refine, roi=roi, threads=threads)
    orc.calc_error(sc.frames, sc.good_frames, s.w.w, s.m.mask, i_ref, wsum, org, u, s.t0.di,
                   s.t0.dj, roi=roi)


def band_trials(s, rows):
    W, M = s.w.w, s.m.mask
    P = int(((M & (W > 0))[rows[0]:rows[1]]).sum())
    K = (2 * s.cfg.half_ss + 1) * (2 * s.cfg.half_fs + 1)
    return P * K * int(np.count_nonzero(s.scan.good_frames))


def cpu_timing(s, steps, warmup, band_rows):
    cores = len(os.sched_getaffinity(0))
    c = s.cfg.n_ss // 2
    rows = (c - band_rows // 2, c - band_rows // 2 + band_rows)
    for _ in range(warmup):
        oracle_iteration_band(s, rows, cores)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle_iteration_band(s, rows, cores)
    dt = time.perf_counter() - t0
    trials = band_trials(s, rows) * steps
    return trials / dt, dt / steps, cores, rows


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2003_12726_b200.synth import CONFIGS, make_scan
    s = make_scan(args.config)
    band = 8
    value, sec, cores, rows = cpu_timing(s, args.steps, args.warmup, band)
    cfg = CONFIGS[args.config]
    sample = (f"oracle port (numpy restatement of recon.py) full iteration "
              f"(make_reference + update_pixel_map threads={cores} + calc_error) on "
              f"detector rows {rows[0]}:{rows[1]} of {cfg.name}")
    out = {"impl": "reference", "metric": METRIC, "value": value,
           "unit": "trials/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
           "config": base_config(cfg), "sample_rows": list(rows),
           "cpu_baseline": {"value": value, "unit": "trials/s", "cores": cores, "kind": "port",
                            "sample": sample},
           "e2e": {"value": value, "unit": "trials/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def one_time_costs(ds, s, host_data, engine, torch):
    """Stack upload (pinned host -> HBM) and K0 statistics, timed with CUDA
    events outside the iteration (reported separately)."""
    out = {}
    st = torch.cuda.current_stream()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    if host_data:
        pinned = torch.empty(ds.frames.shape, dtype=torch.float32, pin_memory=True)
        pinned.numpy()[...] = s.scan.frames
        torch.cuda.synchronize()
        a.record(st)
        ds.frames.copy_(pinned, non_blocking=True)
        b.record(st)
    else:
        a.record(st)
        b.record(st)
    ds.ready(frame_stats=True)         # K0 (pxst_stack_stats, both parts), once per scan
    c.record(st)
    torch.cuda.synchronize()
    if host_data:
        out["stack_upload_ms"] = a.elapsed_time(b)
        out["stack_upload_gb_s"] = ds.frames.numel() * 4 / (a.elapsed_time(b) * 1e-3) / 1e9
    out["k0_stats_ms"] = b.elapsed_time(c)
    return out


class Sequence:
    """The config's workload: `cfg.iters` consecutive iterations from the
    initial state (config 1: 3 x object -> pixel map -> error); steps walk
    that sequence with the state carried over and restart it when done.
    ev = (start, end) events around the pixel-map search (K2), or around the
    translation search (K3) when the config has no pixel-map update;
    ev3 = events around K3 when both run."""

    def __init__(self, ds, cfg, u_t, di_t, dj_t, stream, sharded=None):
        self.ds, self.cfg, self.stream, self.sharded = ds, cfg, stream, sharded
        self.init = (u_t, di_t, dj_t)
        self.state = {"it": 0, "u": u_t, "di": di_t, "dj": dj_t, "geom": None, "dref": None}

    def step(self, ev=None, ev3=None):
        ds, cfg, stream, sharded, state = self.ds, self.cfg, self.stream, self.sharded, self.state
        u_t, di_t, dj_t = self.init
        if state["it"] == 0:
            # (single GPU: state["geom"] is already the initial state's,
            # prefetched by the last iteration of the previous pass)
            state.update(u=u_t, di=di_t, dj=dj_t, dref=None)
            if sharded is not None:
                state.update(geom=None)
        u, di, dj = state["u"], state["di"], state["dj"]
        nxt = nref = None
        if sharded is not None:
            u_new, di_new, dj_new = sharded.iteration(u, di, dj, cfg, ev, geom=state["geom"])
            nxt = sharded.next_geom
        else:
            # the iteration's grid bbox and K2 tile spans were fetched on a side
            # stream while the previous iteration's error maps ran, and its
            # object was formed in the same pass over the stack as those maps
            geom = state["geom"] or ds.geometry_async(u, di, dj, cfg.update_translations)
            dref = state["dref"].resolve() if state["dref"] else ds.object_map(u, di, dj, geom=geom)
            u_new = u
            if cfg.update_pixel_map:
                if ev:
                    ev[0].record(stream)
                u_new, err = ds.pixel_map_search(dref, u, di, dj, cfg.half_ss, cfg.half_fs,
                                                 cfg.subpixel_grid, cfg.refine, geom=geom)
                if ev:
                    ev[1].record(stream)
            di_new, dj_new = di, dj
            if cfg.update_translations:
                k3 = ev if (ev and not cfg.update_pixel_map) else ev3
                if k3:
                    k3[0].record(stream)
                grow = 2 * (max(cfg.half_ss, cfg.half_fs) + 1) if cfg.update_pixel_map else 0
                di_new, dj_new = ds.translation_search(dref, u_new, di, dj, cfg.t_half_ss,
                                                       cfg.t_half_fs, cfg.t_subpixel_grid,
                                                       span_hint=geom.spans3_hint(grow))
                if k3:
                    k3[1].record(stream)
            if state["it"] + 1 < cfg.iters:        # the sequence continues: fuse K4 + next K1
                nxt = ds.geometry_async(u_new, di_new, dj_new, cfg.update_translations)
                _, nref = ds.error_maps_and_next_object(dref, u_new, di_new, dj_new, nxt)
            else:
                # the next step restarts the sequence from the initial state:
                # fetch that state's geometry now, behind these error maps, as
                # every other iteration's is (no host wait at the restart)
                nxt = ds.geometry_async(u_t, di_t, dj_t, cfg.update_translations)
                ds.error_maps(dref, u_new, di_new, dj_new)
        state.update(it=(state["it"] + 1) % max(cfg.iters, 1), u=u_new, di=di_new, dj=dj_new,
                     geom=nxt, dref=nref)


def k3_trials(pb, ds, cfg):
    w = pb.SearchWindow(cfg.t_half_ss, cfg.t_half_fs, cfg.t_subpixel_grid)
    return ds.n_work * len(w.offsets(0)) * len(w.offsets(1)) * ds.n_good


def extra_config(cfg_id, dev, steps=4, warmup=3, rank=0, world=1):
    """A larger BASELINE config measured in the same process as the headline
    (device-resident stack rendered on the GPU, the config's own iteration
    sequence, device-timed with CUDA events; its 3-8 GB stack is larger than
    L2, so no flush is needed).  Reports ms per full iteration and the K2
    (and K3) trial rates and FP32 fractions (11 FLOP per trial)."""
    import torch
    import paper_2003_12726_b200 as pb
    from paper_2003_12726_b200 import engine
    from paper_2003_12726_b200.synth import make_scan_device
    t0 = time.perf_counter()
    s, frames_dev = make_scan_device(cfg_id, dev)
    ds = engine.DeviceScan(None, s.scan.good_frames, s.w.w, s.m.mask, frames_dev=frames_dev)
    cfg = s.cfg
    u_t = ds.upload_u(s.u0.u)
    di_t, dj_t = ds.upload_t(s.t0.di, s.t0.dj)
    ds.ready(frame_stats=cfg.update_translations)
    ds.absmax()
    stream = torch.cuda.current_stream()
    sharded = None
    if world > 1:       # N ranks: every rank renders the same stack, the work is sharded
        from paper_2003_12726_b200.sharding import DeviceExecutor, ShardedIteration
        sharded = ShardedIteration(DeviceExecutor(ds), rank, world)
    seq = Sequence(ds, cfg, u_t, di_t, dj_t, stream, sharded)
    for _ in range(warmup):
        seq.step()
    mk = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
    st, en = [mk() for _ in range(steps)], [mk() for _ in range(steps)]
    k2 = [(mk(), mk()) for _ in range(steps)]
    k3 = [(mk(), mk()) for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        st[i].record(stream)
        seq.step(k2[i] if cfg.update_pixel_map else None,
                 k3[i] if cfg.update_translations else None)
        en[i].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in zip(st, en)]
    if world > 1:       # the slowest rank's time per iteration
        import torch.distributed as dist
        staged = dist.get_backend() == "gloo"
        t = torch.tensor(ms, dtype=torch.float64, device="cpu" if staged else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = [float(x) for x in t.tolist()]
    out = {"workload": cfg.name, "iterations_timed": steps,
           "ms_per_iteration": float(np.mean(ms)), "step_ms": [round(x, 3) for x in ms],
           "setup_s": round(time.perf_counter() - t0, 1)}
    if cfg.update_pixel_map:
        trials = ds.n_work * (2 * cfg.half_ss + 1) * (2 * cfg.half_fs + 1) * ds.n_good
        k2ms = float(np.mean([a.elapsed_time(b) for a, b in k2]))
        tf = FLOP_PER_TRIAL * trials / (k2ms * 1e-3) / 1e12
        out.update(pixel_map_trials_per_iteration=trials,
                   trials_per_s=trials / (out["ms_per_iteration"] * 1e-3),
                   k2_ms=k2ms, k2_tflops=tf, k2_frac=tf / world / THEORETICAL_FP32_TFLOPS)
        # (N ranks: k2_ms is rank 0's time for its row band, k2_tflops the rate of
        # all bands together, k2_frac that rate per GPU against one GPU's peak)
    if world > 1:
        out["parallelism"] = (f"{world} ranks: frames shard object formation and translations, "
                              "detector rows the pixel map and error maps (this rank's K2 time)")
    if cfg.update_translations and world == 1:
        tt = k3_trials(pb, ds, cfg)
        k3ms = float(np.mean([a.elapsed_time(b) for a, b in k3]))
        tf = FLOP_PER_TRIAL * tt / (k3ms * 1e-3) / 1e12
        out.update(translation_trials_per_iteration=tt, k3_ms=k3ms, k3_tflops=tf,
                   k3_frac=tf / THEORETICAL_FP32_TFLOPS)
    del seq, ds, frames_dev
    engine.clear_cache()
    return out


def run_ours(args, rank, world, local):
    import torch
    import paper_2003_12726_b200 as pb
    from paper_2003_12726_b200 import _native, engine
    from paper_2003_12726_b200.synth import CONFIGS, make_scan

    # PXST_BENCH_BACKEND=gloo with PXST_BENCH_ONE_GPU=1 runs the N-rank code path
    # on a single device (functional check only: host-staged collectives)
    if os.environ.get("PXST_BENCH_ONE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("PXST_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        probe = torch.ones(1, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(probe)                 # communicator up: every rank answered
        print(f"[bench] rank {rank}: {backend} process group initialised, "
              f"nranks={dist.get_world_size()}, all_reduce(1)={int(probe.item())}",
              file=sys.stderr, flush=True)
    host_data = args.config <= 1
    if host_data:
        s = make_scan(args.config)
        ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
    else:   # 3-8 GB stacks: rendered on the device (synth.make_scan_device)
        from paper_2003_12726_b200.synth import make_scan_device
        s, frames_dev = make_scan_device(args.config, dev)
        ds = engine.DeviceScan(None, s.scan.good_frames, s.w.w, s.m.mask, frames_dev=frames_dev)
    cfg = s.cfg
    u_t = ds.upload_u(s.u0.u)
    di_t, dj_t = ds.upload_t(s.t0.di, s.t0.dj)
    one_time = one_time_costs(ds, s, host_data, engine, torch)   # reported apart
    if cfg.update_pixel_map:
        K = (2 * cfg.half_ss + 1) * (2 * cfg.half_fs + 1)
    else:   # config 4: translation sweep; its metric counts translation trials
        na = len(pb.SearchWindow(cfg.t_half_ss, cfg.t_half_fs, cfg.t_subpixel_grid).offsets(0))
        nb = len(pb.SearchWindow(cfg.t_half_ss, cfg.t_half_fs, cfg.t_subpixel_grid).offsets(1))
        K = na * nb
    trials = ds.n_work * K * ds.n_good
    stream = torch.cuda.current_stream()

    sharded = None
    if world > 1:
        from paper_2003_12726_b200.sharding import DeviceExecutor, ShardedIteration
        sharded = ShardedIteration(DeviceExecutor(ds), rank, world)

    seq = Sequence(ds, cfg, u_t, di_t, dj_t, stream, sharded)
    step = seq.step

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k2ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    # nvidia-smi samples every 100 ms: the sampler starts before the warm-up and
    # keeps running through an untimed continuation of the same steps (>= 1 s)
    # so the clock record covers the timed region's load.
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        torch.cuda._sleep(1000)            # load the spin kernel before the timed region
        # untimed burn-in (~0.3 s of steps) ahead of the W warm-up steps: on a
        # fresh box the first timed step otherwise measured up to 2.7 ms
        # (K2 alone; steady state 0.59) in the first process
        # The step count is the same on every rank (the sharded step runs
        # collectives): ~0.3 s worth, from one measured step, max over ranks.
        n_burn = 0
        if not args.profile:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            n_burn = min(300, max(1, int(0.3 / max(time.perf_counter() - t0, 1e-4))))
            if world > 1:
                nb = torch.tensor([n_burn], device=dev)
                torch.distributed.all_reduce(nb, op=torch.distributed.ReduceOp.MAX)
                n_burn = int(nb.item())
        for _ in range(n_burn):
            step()
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        launches0 = _native.launch_count()
        torch.cuda.synchronize()
        # After the synchronisation the device queue is empty and the first
        # timed step would run at the host's enqueue rate (its K2 measured
        # 0.8-1.3 ms instead of 0.62): an untimed 1 ms spin lets the host get
        # ahead of the device again, as it is in every later step.
        torch.cuda._sleep(int(1e-3 * 1.965e9))
        for i in range(args.steps):
            flush.zero_()                       # L2 flush between timed steps (untimed)
            starts[i].record(stream)
            step(k2ev[i])
            ends[i].record(stream)
        torch.cuda.synchronize()
        launches = _native.launch_count() - launches0
        if not args.profile:
            t_end = time.perf_counter() + 1.0
            while time.perf_counter() < t_end:
                step()
            torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    k2_ms = [a.elapsed_time(b) for a, b in k2ev]
    total_ms = float(sum(step_ms))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms, float(np.mean(k2_ms))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, k2_mean = t.tolist()
    else:
        k2_mean = float(np.mean(k2_ms))
    ms_per_step = total_ms / args.steps
    value = trials * args.steps / (total_ms * 1e-3)
    extra_sharded = None
    if not args.profile and world > 1 and args.extras:
        # N ranks: the same larger configs, sharded over the ranks (config 3 is
        # the one the 8-GPU scaling target is quoted on); every rank runs them,
        # rank 0 reports the slowest rank's time per iteration
        extra_sharded = {}
        for cid in (int(c) for c in args.extras.split(",") if c.strip()):
            try:
                extra_sharded[f"cfg{cid}"] = extra_config(cid, dev, rank=rank, world=world)
            except Exception as exc:
                extra_sharded[f"cfg{cid}"] = {"error": repr(exc)[:300]}
                raise            # (a rank that stopped would leave the others in a collective)
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    pk = peaks()
    k2_trials = trials / world if world > 1 else trials
    achieved = FLOP_PER_TRIAL * k2_trials / (k2_mean * 1e-3) / 1e12
    traffic = kernel_traffic(cfg.name)
    kname = (f"k_pix_fast<{2 * cfg.half_ss + 1},{2 * cfg.half_fs + 1}> (+slow, epilogue)"
             if cfg.update_pixel_map else "k_trans_fast phase groups (+slow, epilogue)")
    roofline = {"bound": "fp32", "kernel": kname,
                "achieved": achieved, "peak": THEORETICAL_FP32_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / THEORETICAL_FP32_TFLOPS,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "traffic_source": traffic.get("source") if traffic else
                "no ncu capture of this workload in profiles/traffic.json",
                "peak_source": ("theoretical FP32 148 SMs x 128 lanes x 2 x sm_max 1965 MHz "
                                "(MEASURED_PEAKS.json has no FP32 entry; FFMA2 microbenchmark on "
                                "this pool: 73.8 TFLOP/s, profiles/microbench_r01.json)"),
                "work": f"{FLOP_PER_TRIAL} FLOP/trial x {k2_trials} trials per launch",
                "k2_ms": k2_mean, "k2_trials_per_s": k2_trials / (k2_mean * 1e-3)}

    metric = METRIC if cfg.update_pixel_map else \
        "translation trial evaluations/sec (frames x shifts x pixels, full sweep iteration)"
    out = {"metric": metric, "value": value, "unit": "trials/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f32 (fp64 coordinates / accumulators where the reference needs them)",
           "data": "synthetic (seeded, synth.py; stands in for CXIDB 134-136)",
           "config": base_config(cfg),
           "workload_detail": {"work_pixels": ds.n_work, "trials_per_iteration": trials,
                               "l2": "flushed between timed steps (256 MiB write, untimed)",
                               "sequence": f"steps cycle through the config's {cfg.iters}-iteration "
                                           "run from the initial (noisy) state, state carried",
                               "parallelism": (f"rows/frames sharded x{world}" if world > 1
                                               else "single GPU"),
                               "step_ms": [round(x, 4) for x in step_ms],
                               "k2_step_ms": [round(x, 4) for x in k2_ms],
                               **one_time},
           "full_iteration_ms": ms_per_step, "gpu_launches": launches,
           "clocks": clk.summary(), "roofline": roofline}

    if not args.profile and not args.no_e2e and world == 1 and host_data:
        out["e2e"] = e2e(s, args, pb, engine, torch, trials)
        u16 = e2e(s, args, pb, engine, torch, trials, dtype=np.uint16)
        out["e2e"]["uint16_stack"] = {k: u16[k] for k in ("value", "ms_per_step", "h2d_bytes_per_step",
                                                          "d2h_bytes_per_step", "path")}
        pg = e2e(s, args, pb, engine, torch, trials, pinned_frames=False)
        out["e2e"]["pageable"] = {k: pg[k] for k in ("value", "ms_per_step", "h2d_bytes_per_step",
                                                     "d2h_bytes_per_step", "path")}
    if extra_sharded is not None:
        out["extra_configs"] = extra_sharded
    if not args.profile and world == 1 and args.extras:
        # the larger configs, measured in this same run (builder-run numbers
        # alone were not driver-observed)
        out["extra_configs"] = {}
        for cid in (int(c) for c in args.extras.split(",") if c.strip()):
            try:
                out["extra_configs"][f"cfg{cid}"] = extra_config(cid, dev)
            except Exception as exc:       # reported, never fatal to the headline line
                out["extra_configs"][f"cfg{cid}"] = {"error": repr(exc)[:300]}
    if not args.profile and not args.no_cpu_baseline and world == 1 and host_data:
        v, sec, cores, rows = cpu_timing(s, 1, 0, 16)
        out["cpu_baseline"] = {"value": v, "unit": "trials/s", "cores": cores, "kind": "port",
                               "sample": f"oracle port full iteration on detector rows "
                                         f"{rows[0]}:{rows[1]} (update_pixel_map threads="
                                         f"{cores}), 1 run, {sec:.1f} s"}
    print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e(s, args, pb, engine, torch, trials, pinned_frames=True, dtype=None):
    """Public-API iteration from host buffers (pinned, or the plain pageable
    numpy stack a drop-in caller passes), uploads/downloads timed."""
    from dataclasses import replace
    if dtype is not None:
        # the same counts in the detector's own element type, pinned (as raw bytes:
        # torch has no pinned uint16 allocator), uploaded as they are
        src = s.scan.frames.astype(dtype)
        assert np.array_equal(src.astype(np.float32), s.scan.frames)
        raw = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True)
        host = raw.numpy().view(dtype).reshape(src.shape)
        host[...] = src
        scan = replace(s.scan, frames=host)
    elif pinned_frames:
        pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
        pinned.numpy()[...] = s.scan.frames
        scan = replace(s.scan, frames=pinned.numpy())
    else:
        scan = s.scan
    cfg = s.cfg
    win = pb.SearchWindow(cfg.half_ss, cfg.half_fs, cfg.subpixel_grid)
    opts = pb.UpdateOptions(quadratic_refinement=cfg.refine)

    def one():
        engine.SCAN_CACHE.clear()           # every step re-uploads the stack
        ref = pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
        u, err = pb.update_pixel_map(scan, s.w, s.m, ref, s.u0, s.t0, win, opts)
        t = s.t0
        if cfg.update_translations:
            t = pb.update_translations(scan, s.w, s.m, ref, u, s.t0,
                                       pb.SearchWindow(cfg.t_half_ss, cfg.t_half_fs,
                                                       cfg.t_subpixel_grid))
        pb.calc_error(scan, s.w, s.m, ref, u, t)

    steps = max(3, min(args.steps, 10))
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    h0, d0 = engine.TRANSFER["h2d"], engine.TRANSFER["d2h"]
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h2d = (engine.TRANSFER["h2d"] - h0) // steps
    d2h = (engine.TRANSFER["d2h"] - d0) // steps
    engine.SCAN_CACHE.clear()
    return {"value": trials * steps / dt, "unit": "trials/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt / steps * 1e3, "steps": steps,
            "path": "make_reference -> update_pixel_map -> calc_error (drop-in API, numpy in/out,"
                    f" {(np.dtype(dtype).name + ' pinned') if dtype is not None else 'pinned' if pinned_frames else 'pageable (plain numpy)'} host frames,"
                    " device cache cleared each step)"}


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch the N ranks (one process per
    GPU) through torch.distributed.run on this node, same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_env()
    launched = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs (the other torchrun ranks exit without work)
        run_reference(args, rank, world if launched else args.gpus)
        return
    if not launched and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
