#!/usr/bin/env python
"""Benchmark: grid-point x time-step correlations/s for the full-grid solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C3]

One step = one full-grid solve of the workload (BASELINE.json config C3 by
default: 2001x2001 candidates at 1 km x 50 snapshots x 50,000 samples, four
emitters at -20 dB): bit-exact geometry, FP32 correlator, FP64 refinement,
accumulation, exact argmax and detect_emitters, all on the GPU.

* value     — device time with captures already resident in HBM (CUDA events
              on the launching stream, max over ranks), L2 flushed between steps.
* e2e       — the same solve through the public API with host (pinned) captures:
              H2D of every capture and D2H of the accumulated surface inside the
              timed region.
* roofline  — the dominant correlator kernel (k_evaluate_tc at C3): its
              tensor-core FLOPs (split-BF16 MMAs issued) over its event time
              against MEASURED_PEAKS.json's BF16 figure, beside its CUDA-core
              FP32x2 work and the moment kernels' (FFT moments k_mfft: 5 L log2 L
              per FFT; direct k_moments: FMA-pipe work counted by k_work_count)
              against the FP32 peak measured in-process; the reference-equivalent
              rate (20 FLOP per overlapping sample) beside them.
* cpu_baseline / --impl reference — the reference's own CPU path (oracle/_ref,
              compiled from the unmodified reference headers) on this host's
              cores, on a bounded sample of the same workload.

* plugin_path — the reference's own plugin benchmark (compare_backends on
              BenchWorkload, bench.hpp:65-88, 280-330): stage + correlate_batch
              of 500,000 random offsets over 4,096-sample captures through the
              CorrelationSession boundary (the direct k_correlate kernel), at
              several batch sizes, overlapping samples/s, beside the reference's
              ParallelBatchedBackend on this host's cores.

Multi-GPU (--gpus N): one process per GPU. Without torchrun's WORLD_SIZE the
bench re-executes itself under torch.distributed.run with N ranks (or, with
--in-process, drives all N GPUs from one process through the multi-GPU engine,
dg_engine_create_multi). The run is sharded into work units (whole
(snapshot, pair) steps plus bucket-range parts of the remainder steps,
dg_shard_plan); one all-to-all moves every unit's columns to the owner of each
latitude slab, which accumulates its slab in the reference's order; the peak is
a fast-maximum all-reduce plus an exact re-rank per slab and an all-gather of
(value, index); rank 0 detects on the gathered surface.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    # summary of each workload; the scene itself (receivers, emitters, seeds) is
    # tests/scenes.config(name), the reference's simulate_scenario inputs
    "C1": dict(half_km=50.0, snapshots=1, samples=250_000, fs=5e6, emitters="tone", snr=-5.0,
               seed=1),
    "C2": dict(half_km=250.0, snapshots=10, samples=50_000, fs=5e6, emitters="chirp", snr=-10.0,
               seed=2),
    "C3": dict(half_km=1000.0, snapshots=50, samples=50_000, fs=5e6, emitters="four", snr=-20.0,
               seed=3),
    "C4": dict(half_km=None, snapshots=10, samples=50_000, fs=5e6, emitters="four", snr=-15.0,
               seed=4),  # coarse pass: the globe at 10 km (--spacing-km scales it)
    "C5": dict(half_km=2000.0, snapshots=100, samples=50_000, fs=5e6, emitters="four", snr=-20.0,
               seed=5),
}
FC = 1575.42e6
METRIC = "grid-point·time-step correlations/sec (full-grid solve)"
UNIT = "correlations/s"
FLOP_PER_SAMPLE = 20.0  # correlate.hpp:60-68 as executed


def make_inputs(name: str, spacing_km: float = 1.0, n_snapshots: int | None = None,
                reference: bool = False, engine=None):
    """The SURVEY.md §8d inputs of a workload: the reference's simulate_scenario
    scene (paper_scenario.cfg receivers and emitters, tests/scenes.py), either
    synthesised on the GPU by the engine's simulator (scenario values bit for
    bit, samples within ~1e-15 of the reference's; tests/test_simulate.py) or,
    for the reference arm, by the reference itself on the CPU.
    -> (states [S,R,6], captures [S,R,N] complex128, bounds, spacing_deg)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import scenes
    scene = scenes.config(name, spacing_km)
    if n_snapshots:
        scene["snapshots"] = n_snapshots
    bounds = (scene["grid_lat_min_deg"], scene["grid_lat_max_deg"], scene["grid_lon_min_deg"],
              scene["grid_lon_max_deg"])
    if reference:
        from oracle.bindings import RefLib
        sc = RefLib().simulate(scenes.render(scene))
        return sc.states, sc.captures, bounds, scene["grid_spacing_deg"]
    import paper_2508_06672_b200.simulate as sim
    states, caps, _, _ = sim.simulate_arrays(scenes.to_scenario(sim, scene), engine=engine)
    return states, caps, bounds, scene["grid_spacing_deg"]


# ---------------------------------------------------------------------------
# The reference's plugin-path workload (BenchWorkload, bench.hpp:41-88): seeded
# uniform captures and candidate offsets, regenerated here bit for bit
# (std::mt19937_64; tests/test_bench.py checks the arrays and the reference's
# workload_checksum against oracle/_ref).
_MT_N, _MT_M = 312, 156
_MT_A = np.uint64(0xB5026F5AA96619E9)
_MT_UM, _MT_LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)


def mt19937_64(seed: int, n: int) -> np.ndarray:
    """The first n outputs of std::mt19937_64(seed) (twist vectorised in the
    three dependency-free ranges of the recurrence)."""
    mt = np.zeros(_MT_N, np.uint64)
    mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for i in range(1, _MT_N):
            prev = int(mt[i - 1])
            mt[i] = np.uint64((6364136223846793005 * (prev ^ (prev >> 62)) + i)
                              & 0xFFFFFFFFFFFFFFFF)
    one, sh1 = np.uint64(1), np.uint64(1)

    def mix(hi, lo, far):
        x = (hi & _MT_UM) | (lo & _MT_LM)
        return far ^ (x >> sh1) ^ ((x & one) * _MT_A)

    out = np.empty(((n + _MT_N - 1) // _MT_N) * _MT_N, np.uint64)
    with np.errstate(over="ignore"):
        for blk in range(len(out) // _MT_N):
            k = _MT_N - _MT_M
            mt[:k] = mix(mt[:k], mt[1:k + 1], mt[_MT_M:])
            mt[k:_MT_N - 1] = mix(mt[k:_MT_N - 1], mt[k + 1:], mt[:_MT_N - 1 - k])
            mt[_MT_N - 1] = mix(mt[_MT_N - 1:], mt[:1], mt[_MT_M - 1:_MT_M])[0]
            y = mt.copy()
            y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
            y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            y ^= y >> np.uint64(43)
            out[blk * _MT_N:(blk + 1) * _MT_N] = y
    return out[:n]


def build_workload(n_points: int = 500_000, n_samples: int = 4096, fs: float = 5e6,
                   seed: int = 1):
    """bench.hpp:65-88 -> (y1, y2, offsets [tdoa int64, fdoa f64])."""
    r = mt19937_64(seed, 4 * n_samples + 2 * n_points)
    u = (r >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform(x, lo, hi):
        return lo + (hi - lo) * x

    caps = []
    for c in range(2):  # emplace_back(re, im): g++ evaluates the im draw first
        w = u[2 * c * n_samples:2 * (c + 1) * n_samples].reshape(n_samples, 2)
        caps.append(uniform(w[:, 1], -1.0, 1.0) + 1j * uniform(w[:, 0], -1.0, 1.0))
    w = u[4 * n_samples:].reshape(n_points, 2)
    ms = float(n_samples // 2)
    t = uniform(w[:, 0], -ms, ms)
    tr = np.trunc(t)
    tdoa = tr + np.where(np.abs(t - tr) >= 0.5, np.sign(t), 0.0)  # std::llround
    off = np.zeros(n_points, np.dtype([("tdoa_samples", "<i8"), ("fdoa_hz", "<f8")]))
    off["tdoa_samples"] = tdoa.astype(np.int64)
    off["fdoa_hz"] = uniform(w[:, 1], -fs / 4.0, fs / 4.0)
    return caps[0], caps[1], off


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every
    50 ms (nvidia-smi every 0.2 s if NVML is unavailable)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
            # one untimed query first: on a fresh box the first clock / reason
            # queries were seen to stall a concurrent solve for ~0.5 s
            for _ in range(3):
                self._sample_nvml()
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        if getattr(self, "_max_sm", None) is None:  # constant: queried once
            self._max_sm = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        mx = self._max_sm
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in self.BITS]

    def _loop(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self.samples.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            # 50 ms: NVML queries contend with the solve's CUDA calls in the driver
            # (at 10 ms a 16M-point solve occasionally stalled by tens of ms)
            self._stop.wait(0.05 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        if os.environ.get("DG_BENCH_NO_CLOCKS") != "1":  # diagnostics only
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t.is_alive():
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "n_samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref) — run in a child process under a watchdog
# because the reference's ParallelBatchedBackend can deadlock.
def ref_worker(args):
    from oracle.bindings import RefLib
    ref = RefLib()
    cfg = WORKLOADS[args.config]
    states, caps, bounds, spacing = make_inputs(args.config, args.sample_km,
                                                args.sample_snapshots, reference=True)
    workers = os.cpu_count() or 1
    times = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = ref.geolocate(states, caps, cfg["fs"], FC, bounds, spacing, 0.0, backend="parallel",
                            workers=workers, batch_size=4096)
        times.append(time.perf_counter() - t0)
    P = len(res["accumulated"])
    out = {"times": times[args.warmup:], "points": P, "snapshots": int(caps.shape[0]),
           "workers": workers, "argmax": int(np.argmax(res["accumulated"]))}
    if args.extra_baselines:
        # the reference's SerialBackend on one core, and its
        # ParallelBatchedBackend at the paper's batch size of 8, on two snapshots
        s2 = min(2, caps.shape[0])
        for key, backend, w, bs in (("serial_1core", "serial", 1, 4096),
                                    ("parallel_batch8", "parallel", workers, 8)):
            t0 = time.perf_counter()
            ref.geolocate(states[:s2], caps[:s2], cfg["fs"], FC, bounds, spacing, 0.0,
                          backend=backend, workers=w, batch_size=bs)
            out[key] = P * s2 / (time.perf_counter() - t0)
    print(json.dumps(out))


def run_ref_child(args, steps, warmup, sample_km, sample_snapshots, timeout, extra=False):
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-worker", "--config", args.config,
           "--steps", str(steps), "--warmup", str(warmup), "--sample-km", str(sample_km),
           "--sample-snapshots", str(sample_snapshots)] + (["--extra-baselines"] if extra else [])
    hangs = 0
    for _attempt in range(2):
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        except subprocess.TimeoutExpired:
            hangs += 1
            continue
        if out.returncode == 0:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            d["hangs"] = hangs
            return d
        raise RuntimeError(out.stderr[-2000:])
    raise RuntimeError(f"reference CPU path hung {hangs} times (TaskPool race, SURVEY.md §5)")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_arm(args, rank, world):
    if rank != 0:
        return
    d = run_ref_child(args, args.steps, args.warmup, args.sample_km, args.sample_snapshots,
                      timeout=1800)
    sec = statistics.mean(d["times"])
    value = d["points"] * d["snapshots"] / sec
    sample = (f"{args.config} footprint at {args.sample_km:g} km stride ({d['points']} points) x "
              f"{d['snapshots']} snapshots, reference geolocate_snapshots with "
              f"ParallelBatchedBackend({d['workers']}) batch 4096; {cpu_model()}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": d["workers"], "kind": "reference",
                         "sample": sample, "hangs": d["hangs"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def b200_arm(args, rank, world):
    import torch

    import paper_2508_06672_b200 as b2
    from paper_2508_06672_b200 import sharding
    from paper_2508_06672_b200._capi import lib

    # one rank per GPU; (gloo test mode: ranks may share the box's GPUs)
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:  # gloo: the multi-rank path on one GPU (tests); collectives via the host
            dist.init_process_group("gloo")
    coll_dev = "cuda" if args.dist_backend == "nccl" else "cpu"
    cfg = WORKLOADS[args.config]
    # --in-process: one engine over every GPU of this process (dg_engine_create_multi)
    devices = [dev]
    if world == 1 and args.gpus > 1:
        devices = ([int(d) for d in args.device_list.split(",")] if args.device_list else
                   list(range(args.gpus)))
        if len(devices) != args.gpus or max(devices) >= torch.cuda.device_count():
            raise SystemExit(f"bench: --gpus {args.gpus} needs {args.gpus} visible GPUs")
    n_gpus = world if world > 1 else len(devices)
    eng = b2.default_engine(dev) if len(devices) == 1 else b2.Engine(devices=devices)
    states, caps, bounds, spacing = make_inputs(args.config, args.spacing_km,
                                                engine=b2.default_engine(dev))
    S, R, N = caps.shape
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing, 0.0, engine=eng)
    P = grid.size()
    staged = b2.StagedSnapshots(states, caps, cfg["fs"], FC, engine=eng)
    opts = b2.GeolocateOptions(k_sigma=5.0, exclusion_radius_cells=5, detect=True)
    # the solve's launching stream: the engine runs on it (side streams joined
    # back into it) and the events and the L2 flush are recorded on it; the
    # multi-GPU engine's call returns when every device is done
    stream = torch.cuda.Stream()
    acc_dev = torch.empty(P, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def solve(stg, profile=False):
        """One full-grid solve; returns (correlation stats of this rank, peak)."""
        if dist is None:
            res = b2.geolocate_staged(grid, stg, opts, want_surface=False,
                                      accumulated_device=acc_dev.data_ptr(),
                                      stream=stream.cuda_stream, profile=profile)
            return res.stats, (res.argmax_value, res.argmax_index)
        # work-unit sharded (paper_2508_06672_b200.sharding): each rank correlates
        # its units over the whole grid, one all-to-all to latitude slabs,
        # per-slab accumulation + two-stage exact peak, surface gather,
        # detection on rank 0
        value, index, _, _, st = sharding.geolocate_sharded(
            grid, stg, opts, gather=True, stream=stream.cuda_stream, profile=profile)
        return st, (value, index)

    for _ in range(args.warmup):
        solve(staged)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # outside the events: L2 starts cold every step
            ev[k][0].record(stream)
            st, best = solve(staged)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    # one more solve with per-kernel events (steps serialised on one stream so
    # each kernel's time is its own) for the rooflines; not part of `value`
    # (the multi-GPU engine is profiled through one device's engine)
    with torch.cuda.stream(stream):
        flush.zero_()
    if len(devices) > 1:
        g1 = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing, 0.0,
                                     engine=b2.default_engine(dev))
        s1 = b2.StagedSnapshots(states, caps, cfg["fs"], FC, engine=b2.default_engine(dev))
        last = b2.geolocate_staged(g1, s1, opts, want_surface=False,
                                   accumulated_device=acc_dev.data_ptr(),
                                   stream=stream.cuda_stream, profile=True).stats
        del g1, s1
    else:
        last = solve(staged, profile=True)[0]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = sum(ms) / len(ms)
    if dist is not None:
        t = torch.tensor([ms_step], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = P * S / (ms_step * 1e-3)

    # rooflines of the two correlator kernels, this rank's launches (FP32x2 MACs
    # counted on the device by k_work_count: 4 FLOP each)
    print("[bench] per-solve stats: " + json.dumps({k: last.get(k) for k in (
        "correlate_ms", "moments_ms", "evaluate_ms", "moment_ffma2", "evaluate_ffma2",
        "direct_steps", "n_refined", "total_ms", "kernel_launches")}), file=sys.stderr)
    peak = ctypes_peak(lib, dev)
    mom_ms = last["moments_ms"]
    ev_ms = last["evaluate_ms"]
    corr_ms = mom_ms + ev_ms
    # moments: FFT FLOPs (5 L log2 L per FFT + 6 L per spectrum product), or the
    # direct sums' FMA-pipe work in FP32x2 operations x 4 FLOP-equivalents (k_work_count)
    fft_flop = last.get("moment_fft_flop") or 0.0
    mom_name = "k_mfft" if fft_flop > 0 else "k_moments"
    mom_work = fft_flop if fft_flop > 0 else 4.0 * last["moment_ffma2"]
    mom_tf = mom_work / (mom_ms * 1e-3) / 1e12 if mom_ms else None
    ev_tf = 4.0 * last["evaluate_ffma2"] / (ev_ms * 1e-3) / 1e12 if ev_ms else None
    tc_flop = last.get("evaluate_tc_flop") or 0.0
    ev_name = "k_evaluate_tc" if tc_flop > 0 else "k_evaluate"
    tc_tf = tc_flop / (ev_ms * 1e-3) / 1e12 if ev_ms and tc_flop else None
    bf16_peak = measured_peaks().get("bf16_tflops")
    ovl = last["sum_overlap_samples"]
    dominant = ev_name if ev_ms >= mom_ms else mom_name
    if dominant == "k_evaluate_tc" and tc_tf and bf16_peak:  # the MMA kernel: tensor roofline
        bound, achieved, peak_top = "tensor", tc_tf, bf16_peak
        peak_src = "MEASURED_PEAKS.json bf16_tflops (dense BF16)"
    else:
        bound, achieved, peak_top = "fp32", (ev_tf if dominant == ev_name else mom_tf), peak
        peak_src = "dg_fp32_peak_tflops FFMA probe in this process"
    launches = st.get("kernel_launches", last["kernel_launches"])

    # e2e: host (pinned) captures in, accumulated surface out, through the public API
    pinned = torch.empty(caps.shape, dtype=torch.complex128, pin_memory=True).numpy()
    pinned[...] = caps
    surf = torch.empty(P, dtype=torch.float64, pin_memory=True)
    e2e_t = []
    for k in range(args.warmup + args.steps):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if dist is None:
            b2.geolocate_arrays(grid, states, pinned, cfg["fs"], FC, opts, want_surface=True,
                                want_per_snapshot=False, out=surf.numpy())
        else:
            stg = b2.StagedSnapshots(states, pinned, cfg["fs"], FC, engine=eng)
            _, _, full, _, _ = sharding.geolocate_sharded(grid, stg, opts, gather=True,
                                                          stream=stream.cuda_stream)
            surf.copy_(full)
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e_t.append(time.perf_counter() - t0)
    # median over the timed steps: a wall-clock leg, robust to a lone host hiccup
    # (every step's time is in the line)
    e2e_s = statistics.median(e2e_t)
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": P * S / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(caps.nbytes + states.nbytes),
           "d2h_bytes_per_step": int(P * 8 + 4096 * 48),
           "ms_per_step": e2e_s * 1e3, "statistic": "median",
           "step_ms": [round(x * 1e3, 3) for x in e2e_t]}

    plugin = None
    if rank == 0 and not args.no_plugin:
        plugin = plugin_leg(args, b2, peak, world == 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            d = run_ref_child(args, 1, 0, args.sample_km, args.cpu_sample_snapshots, timeout=900,
                              extra=True)
            cpu = {"value": d["points"] * d["snapshots"] / d["times"][0], "unit": UNIT,
                   "cores": d["workers"], "kind": "reference",
                   "sample": (f"{args.config} footprint at {args.sample_km:g} km stride "
                              f"({d['points']} points) x {d['snapshots']} snapshots, reference "
                              f"geolocate_snapshots, ParallelBatchedBackend({d['workers']}) batch "
                              f"4096, {d['times'][0]:.1f} s; {cpu_model()}"),
                   "hangs": d["hangs"],
                   "serial_1core": {"value": d.get("serial_1core"), "unit": UNIT, "cores": 1,
                                    "sample": "the same footprint, 2 snapshots, SerialBackend"},
                   "parallel_batch8": {"value": d.get("parallel_batch8"), "unit": UNIT,
                                       "cores": d["workers"],
                                       "sample": "the same footprint, 2 snapshots, "
                                                 "ParallelBatchedBackend batch 8 (the paper's "
                                                 "default)"}}
        except Exception as e:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"[:300]}

    if rank == 0:
        par = ("1 GPU" if n_gpus == 1 else
               f"{n_gpus} GPUs, work-unit sharded ({'one process' if dist is None else 'one rank'}"
               " per GPU; all-to-all to latitude slabs)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: the reference's simulate_scenario scene for the workload "
                    "(SURVEY §8d; paper_scenario.cfg receivers/emitters), synthesised on the GPU "
                    "by paper_2508_06672_b200.simulate",
            "config": {"workload": args.config, "grid": f"{grid.lat.count}x{grid.lon.count}",
                       "points": P, "snapshots": S, "samples": N,
                       "spacing_km": args.spacing_km, "parallelism": par,
                       "l2": "flushed between timed steps (256 MB write)",
                       "precision": "FP32 correlator, FP64 geometry/accumulation/refine"},
            "e2e": e2e,
            "roofline": {
                "bound": bound, "kernel": dominant, "achieved": achieved, "peak": peak_top,
                "unit": "TFLOP/s", "frac": achieved / peak_top if achieved and peak_top else None,
                "traffic": ncu_traffic(dominant),
                "traffic_source": f"dram__bytes_read.sum + dram__bytes_write.sum per {dominant} "
                                  f"launch, {NCU_SUMMARY}",
                "peak_source": peak_src,
                "flop_definition": "k_evaluate_tc (tensor): BF16 MMA FLOPs issued, 6 split "
                                   "products x 2*128*np*16 per 128-candidate tile; CUDA-core "
                                   "parts: 4 x FP32x2 operations counted on the device by "
                                   "k_work_count (k_evaluate_tc: 3 per candidate-block; "
                                   "k_moments: B/2*(R+6) per bucket-block); k_mfft: 5 L log2 L "
                                   "per 1024-point FFT + 6 L per spectrum product",
                "kernels": {mom_name: {"ms": mom_ms, "tflops": mom_tf, "bound": "fp32",
                                       "frac": mom_tf / peak if mom_tf and peak else None,
                                       "fp32_peak": peak},
                            ev_name: {"ms": ev_ms, "tflops": ev_tf,
                                      "frac": ev_tf / peak if ev_tf and peak else None,
                                      "tensor_tflops": tc_tf,
                                      "tensor_frac": (tc_tf / bf16_peak
                                                      if tc_tf and bf16_peak else None),
                                      "tensor_peak": bf16_peak,
                                      "tensor_peak_source": "MEASURED_PEAKS.json bf16_tflops",
                                      "tensor_flop_definition":
                                          "BF16 MMA FLOPs issued: 6 split products x "
                                          "2*128*np*16 per 128-candidate tile"}},
                "reference_equivalent": {
                    "flop_per_sample": FLOP_PER_SAMPLE, "sum_overlap_samples": ovl,
                    "tflops": FLOP_PER_SAMPLE * ovl / (corr_ms * 1e-3) / 1e12 if corr_ms else None,
                    "note": "the reference kernel's 20 FLOP per overlapping sample over the "
                            "correlator time: work the block-moment factorisation avoids"},
                "correlate_ms_per_step": corr_ms},
            "plugin_path": plugin,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": launches * args.steps,
            "argmax": {"index": best[1], "value": best[0]},
            "refined_elements": last["n_refined"],
            "step_ms": [round(x, 3) for x in ms],  # this rank's timed solves
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


PLUGIN_POINTS = 500_000    # BenchWorkload defaults (bench.hpp:41-45)
PLUGIN_SAMPLES = 4096
PLUGIN_BATCHES = (8, 4096, PLUGIN_POINTS)


def plugin_leg(args, b2, fp32_peak, with_cpu):
    """The reference's plugin benchmark on this engine: BenchWorkload (500k random
    offsets, |tdoa| <= 2048, |fdoa| <= fs/4, uniform I/Q) through
    stage + correlate_batch (bench.hpp:113-118 time_run), at the paper's batch
    of 8, the bench's 4096 and one batch of everything; the direct correlator
    (the FDOA range admits no block moments). Overlapping samples/s counts
    sum_i (N - |tdoa_i|), the reference kernel's work (20 FLOP each)."""
    y1, y2, off = build_workload(PLUGIN_POINTS, PLUGIN_SAMPLES, 5e6, 1)
    ovl = float(np.maximum(0, PLUGIN_SAMPLES - np.abs(off["tdoa_samples"])).sum())
    be = b2.make_backend("b200", 1)
    c1, c2 = b2.BasebandCapture(y1, 5e6), b2.BasebandCapture(y2, 5e6)
    out = np.zeros(PLUGIN_POINTS)
    rows = {}
    for bs in PLUGIN_BATCHES:
        reps = 1 if bs < 64 else 5
        times = []
        for r in range(reps + 1):
            t0 = time.perf_counter()
            s = be.stage(c1, c2)
            for a in range(0, PLUGIN_POINTS, bs):
                s.correlate_batch(off[a:a + bs], out[a:a + bs])
            dt = time.perf_counter() - t0
            if r:
                times.append(dt)
        sec = statistics.mean(times)
        rows[str(bs)] = {"s_per_run": sec, "overlap_samples_per_s": ovl / sec,
                         "points_per_s": PLUGIN_POINTS / sec}
    best = rows[str(PLUGIN_POINTS)]
    # k_correlate FMA-pipe work: 2 FFMA2 per candidate-sample (A, B) = 8 FLOP
    fma_tf = 8.0 * ovl / best["s_per_run"] / 1e12
    # the kernel's own launch time from the committed ncu launch list of the same
    # pass (tests/profile_plugin.py); the live figure above includes the call's
    # staging, planning and copies
    kern_us = None
    try:
        for line in open(os.path.join(ROOT, "profiles", "r02_launches_plugin_summary.txt")):
            if "k_correlate" in line:
                kern_us = float(line.split()[-2])
    except (OSError, ValueError, IndexError):
        pass
    res = {"workload": f"BenchWorkload {PLUGIN_POINTS} points x {PLUGIN_SAMPLES} samples, seed 1 "
                       "(bench.hpp:65-88, regenerated bit for bit)",
           "overlap_samples": ovl, "batches": rows,
           "k_correlate": {"bound": "fp32 fma pipe", "achieved": fma_tf, "peak": fp32_peak,
                           "unit": "TFLOP/s", "frac": fma_tf / fp32_peak if fp32_peak else None,
                           "flop_definition": "8 per overlapping candidate-sample (2 FFMA2: the "
                                              "A / B phasor-table MACs), whole call incl. "
                                              "staging and copies",
                           "kernel_us_ncu": kern_us,
                           "achieved_kernel": 8.0 * ovl / (kern_us * 1e-6) / 1e12 if kern_us else None,
                           "frac_kernel": (8.0 * ovl / (kern_us * 1e-6) / 1e12 / fp32_peak
                                           if kern_us and fp32_peak else None),
                           "kernel_source": "profiles/r02_launches_plugin_summary.txt (ncu "
                                            "gpu__time_duration of the same pass)"},
           "reference_equivalent_tflops": 20.0 * ovl / best["s_per_run"] / 1e12}
    if with_cpu and not args.no_cpu_baseline:
        try:
            cmd = [sys.executable, os.path.abspath(__file__), "--ref-plugin-worker"]
            o = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
            d = json.loads(o.stdout.strip().splitlines()[-1])
            res["cpu_baseline"] = {"overlap_samples_per_s": d["ovl"] / d["s"], "unit":
                                   "overlapping samples/s", "cores": d["workers"],
                                   "kind": "reference",
                                   "sample": f"first {d['points']} offsets of the workload, "
                                             "reference ParallelBatchedBackend "
                                             f"({d['workers']}) correlate_batch, batch 4096, "
                                             f"{d['s']:.1f} s; {cpu_model()}"}
        except Exception as e:
            res["cpu_baseline"] = {"overlap_samples_per_s": None, "sample": f"failed: {e}"[:300]}
    return res


def ref_plugin_worker(args):
    from oracle.bindings import RefLib
    ref = RefLib()
    n = 60_000
    y1, y2, off = build_workload(PLUGIN_POINTS, PLUGIN_SAMPLES, 5e6, 1)
    off = off[:n]
    workers = os.cpu_count() or 1
    ref.correlate_batch(y1, y2, 5e6, off[:4096], "parallel", workers, 4096)  # warm-up
    t0 = time.perf_counter()
    ref.correlate_batch(y1, y2, 5e6, off, "parallel", workers, 4096)
    s = time.perf_counter() - t0
    ovl = float(np.maximum(0, PLUGIN_SAMPLES - np.abs(off["tdoa_samples"])).sum())
    print(json.dumps({"s": s, "ovl": ovl, "points": n, "workers": workers}))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


NCU_SUMMARY = "profiles/r02_ncu_kernels.txt"


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, NCU_SUMMARY)
    try:
        vals, cur = {}, None
        for line in open(path):
            if line.startswith("== "):
                cur = line.split()[1]
                continue
            parts = line.split()
            if cur == kernel and len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum",
                                                                   "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[parts[-2]]
                vals[parts[0]] = float(parts[-1]) * scale
        return sum(vals.values()) if len(vals) == 2 else None
    except OSError:
        return None


def ctypes_peak(lib, dev):
    import ctypes as C
    v = C.c_double()
    rc = lib.dg_fp32_peak_tflops(dev, C.byref(v))
    return v.value if rc == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--spacing-km", type=float, default=1.0)
    ap.add_argument("--sample-km", type=float, default=20.0,
                    help="reference CPU sample: same footprint at a coarser stride")
    ap.add_argument("--sample-snapshots", type=int, default=5,
                    help="snapshots per reference-arm step")
    ap.add_argument("--cpu-sample-snapshots", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--in-process", action="store_true",
                    help="--gpus N > 1 without torchrun: one process drives every GPU through "
                         "the multi-GPU engine instead of spawning N ranks")
    ap.add_argument("--no-plugin", action="store_true", help="skip the plugin-path leg")
    ap.add_argument("--device-list", default="", help=argparse.SUPPRESS)  # tests: 0,0
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help=argparse.SUPPRESS)
    ap.add_argument("--ref-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ref-plugin-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--extra-baselines", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_worker:
        return ref_worker(args)
    if args.ref_plugin_worker:
        return ref_plugin_worker(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and not args.in_process:
        return spawn_ranks(args)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    return b200_arm(args, rank, world)


def spawn_ranks(args):
    """--gpus N without torchrun: re-run this command as N ranks (one per GPU)
    under torch.distributed.run on this node; rank 0 prints the line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.run(cmd, cwd=ROOT).returncode)


if __name__ == "__main__":
    main()
