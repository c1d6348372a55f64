#!/usr/bin/env python
"""bench.py -- TernaryNet ternary conv3d / FCN throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the hot path over BASELINE.json configs[1] (C1): the
int8 ternary codes 1x64x64x128x128 are packed (A1, tn_pack_i8) and convolved
with 64x64x3x3x3 ternary filters with the fused integer-threshold requant (A2-A4,
tn_conv3d_requant).  `value` = effective GMAC/s (out voxels x K x C x 27 per
step, all ranks) with inputs resident in HBM.  The same JSON line carries:
  roofline     -- the conv kernel's achieved rate vs its binding peak
  e2e          -- the same metric through the C ABI with host buffers (H2D of
                  the codes + D2H of the packed output inside the timed region)
  fcn          -- FCN voxels/s (A1-A9): configs[3] (8 CT-like volumes
                  128x256x256, sharded one volume at a time across ranks)
  cpu_baseline -- the oracle (oracle/, untuned) on a bounded sample of C1
  clocks       -- NVML SM clocks and throttle reasons sampled during timing
Multi-GPU (torchrun, one rank per GPU): every rank runs its own C1 replica
(weak scaling, no data-path collective; BASELINE configs shard by volume), max
device time over ranks.  `--impl reference` times the CPU oracle instead
(rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

C1 = synth.CONFIGS["C1"]
C1_MACS = 64 * 128 * 128 * 64 * 64 * 27          # out voxels x K x C x 27 = 115,964,116,992
FCN_MACS_PER_VOXEL = 45360
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fcn-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fcn", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-binary", action="store_true")
    ap.add_argument("--no-c0", action="store_true")
    ap.add_argument("--no-slab-schedules", action="store_true")
    ap.add_argument("--c4-halo", choices=("nccl", "p2p"), default="nccl",
                    help="configs[4] halo exchange at N > 1: NCCL send/recv, or NEXT-1 epilogue stores + flags")
    return ap.parse_args()


# ----------------------------------------------------------------------------- distributed
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Samples SM clock and throttle reasons every 5 ms on a background thread."""

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._names = {}
        if self.ok:
            for name in ("GpuIdle", "ApplicationsClocksSetting", "SwPowerCap", "HwSlowdown", "SyncBoost",
                         "SwThermalSlowdown", "HwThermalSlowdown", "HwPowerBrakeSlowdown", "DisplayClockSetting"):
                v = getattr(self.nv, "nvmlClocksEventReason" + name, None) or \
                    getattr(self.nv, "nvmlClocksThrottleReason" + name, None)
                if v:
                    self._names[v] = name

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self._first.set()
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self._names.items():
                    if r & bit and name != "GpuIdle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        self._first = threading.Event()
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            self._first.wait(1.0)   # the thread's start-up (NVML's first calls) before any timing
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- reference arm
def oracle_c1_sample(x, w, lo, hi, planes: int):
    """Oracle conv3d + requant over output planes [0, planes) of C1 (input planes [0, planes+1))."""
    import oracle
    xs = np.ascontiguousarray(x[:, :, :planes + 1])
    acc = oracle.conv3d(xs, w)[:, :, :planes]
    oracle.requant(np.ascontiguousarray(acc), lo, hi)
    return planes * 128 * 128 * 64 * 64 * 27


GOLDEN = os.path.join(ROOT, "tests", "golden", "bench_samples.npz")


class L2Flush:
    """Between timed steps, outside the events: write a 256 MiB buffer (twice the 126 MB L2), then
    read another 256 MiB buffer, so the dirty lines of the write are written back before the next
    step starts (otherwise their write-back would run inside that step's events, competing with
    its HBM traffic) and the step begins with a cold, clean L2."""

    def __init__(self, torch, dev):
        self.w = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(L2_FLUSH_BYTES // 8, dtype=torch.int64, device=dev)
        self.out = torch.empty((), dtype=torch.int64, device=dev)

    def __call__(self):
        self.w.zero_()
        self.out = self.r.sum()


def bench_peaks():
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(pk)) if os.path.exists(pk) else {}


def golden():
    """Expected sampled outputs for the parity gates, written by tools/make_bench_golden.py (which
    calls only the oracle): the GPU arm does not execute oracle/ outside its cpu_baseline leg."""
    return np.load(GOLDEN)


def ternary_at(yp, at):
    """Ternary values of a packed [n][d][h][w][2][cw] tensor at sampled (n, k, z, y, x)."""
    ypn = yp.cpu().numpy().view(np.uint32)
    n_, k_, z_, y_, x_ = at.T
    sb = (ypn[n_, z_, y_, x_, 0, k_ // 32] >> (k_ % 32)) & 1
    mb = (ypn[n_, z_, y_, x_, 1, k_ // 32] >> (k_ % 32)) & 1
    return np.where(mb == 1, np.where(sb == 1, 1, -1), 0).astype(np.int8)


C1_WORKLOAD = ("C1: 1x64x64x128x128 ternary conv3d 64->64 3x3x3 s1 p1 + fused integer-threshold requant, "
               "P(0)=0.5 act / 0.6 weights (BASELINE configs[1])")


def run_reference(args, world, rank):
    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 runs the oracle alone, on every core
    if world > 1 or os.environ.get("OMP_NUM_THREADS") == "1":
        os.environ["OMP_NUM_THREADS"] = str(cpu_cores())
    import oracle
    x, w, lo, hi = synth.conv_config("C1")
    planes = 2
    for _ in range(args.warmup):
        oracle_c1_sample(x, w, lo, hi, planes)
    times = []
    macs = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = time.perf_counter()
        macs += oracle_c1_sample(x, w, lo, hi, planes)
        times.append(time.perf_counter() - s)
    tot = time.perf_counter() - t0
    value = macs / tot / 1e9
    line = {
        "impl": "reference", "metric": "ternary conv3d effective GMAC/s (C1, fused requant)",
        "value": value, "unit": "GMAC/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": C1_WORKLOAD,
                   "sample": f"output planes [0,{planes}) of 64 per step"},
        "cpu_baseline": {"value": value, "unit": "GMAC/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"oracle conv3d+requant, {planes} of 64 output planes of C1 per step"},
        "e2e": {"value": value, "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-exec under torch.distributed.run with N
    ranks (one per GPU, rendezvous on 127.0.0.1), so that --gpus is never silently ignored."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE {world}; refusing to report"}), flush=True)
        sys.exit(2)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1801_09449_b200 as tn

    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    tnpk = os.path.join(ROOT, "profiles", "PEAKS_TN.json")
    tn_peaks = json.load(open(tnpk)) if os.path.exists(tnpk) else {}

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    # ---- C1 inputs (same seeds on every rank: replicas)
    x, w, lo, hi = synth.conv_config("C1")
    x_host = torch.from_numpy(x).pin_memory()
    x_d = x_host.to(dev)
    w_d = torch.from_numpy(w).to(dev)
    lo_d, hi_d = torch.from_numpy(lo).to(dev), torch.from_numpy(hi).to(dev)
    xd = tn.dims(*x.shape)
    g = tn.geom(1, 1, 1)
    wp = tn.tn_pack_weights(w_d)
    # the filter bank's tensor-core operand image, built once with the weights (tn_conv_prepare)
    prep = tn.tn_conv_prepare([(None, xd, 0, wp)], 64, g)
    xp = tn.packed_empty(*x.shape, device=dev)
    yp = tn.packed_empty(1, 64, 64, 128, 128, device=dev)
    yp_host = torch.empty(yp.shape, dtype=torch.int32).pin_memory()
    flush = L2Flush(torch, dev)

    def step():
        tn.tn_pack_i8(x_d, xp)
        tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, 64, g, lo_d, hi_d, yp)

    # ---- parity gate (SPEC.md:485 pattern: no number without a passing check)
    step()
    torch.cuda.synchronize()
    gold = golden()
    if not np.array_equal(ternary_at(yp, gold["c1_at"]), gold["c1_ref"]):
        print(json.dumps({"error": "parity check failed; refusing to report"}), flush=True)
        sys.exit(1)
    parity = f"passed ({len(gold['c1_ref'])} sampled outputs vs the oracle's values in tests/golden/bench_samples.npz)"

    for _ in range(args.warmup):
        flush()          # (the flush's own kernels and allocations warm up too)
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps outside the events
    # (no event between pack and conv here: the conv is launched with programmatic
    # dependent launch and its prologue overlaps the pack's tail)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        # a 2 ms GPU spin (outside the events) lets the host queue the steps ahead of the GPU, so
        # no host launch latency lands between a step's events
        torch.cuda._sleep(4_000_000)
        for i in range(args.steps):
            flush()
            a, c = ev[i]
            a.record(stream)
            tn.tn_pack_i8(x_d, xp)
            tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, 64, g, lo_d, hi_d, yp)
            c.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, c in ev]
    if os.environ.get("TN_BENCH_DEBUG"):
        print("step_ms", [round(t * 1e3, 1) for t in step_ms], file=sys.stderr)
    # kernel timing pass for the roofline: the same steps with an event between pack and
    # conv (the conv's own launch duration on its stream; this serialises the two)
    ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush()
        a, b, c = ev3[i]
        a.record(stream)
        tn.tn_pack_i8(x_d, xp)
        b.record(stream)
        tn.tn_conv3d_requant_prepared(prep, xp, xd, wp, 64, g, lo_d, hi_d, yp)
        c.record(stream)
    torch.cuda.synchronize()
    conv_ms = [b.elapsed_time(c) for _, b, c in ev3]
    pack_ms = [a.elapsed_time(b) for a, b, _ in ev3]
    split_step_ms = [a.elapsed_time(c) for a, _, c in ev3]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = world * args.steps * C1_MACS / (tot_ms / 1e3) / 1e9

    # ---- e2e through the C ABI with host buffers: every step copies its int8 codes from
    # pinned host memory, packs, convolves and copies the packed result back.  Two buffer
    # sets on two streams (double buffering): the H2D copy of step i+1 overlaps the compute
    # and the D2H copy of step i (separate copy engines); the timed region spans all steps.
    e2e_steps = max(4, min(args.steps, 10))
    streams = [stream, torch.cuda.Stream(device=dev)]
    x_b = [x_d, torch.empty_like(x_d)]
    xp_b = [xp, tn.packed_empty(*x.shape, device=dev)]
    yp_b = [yp, tn.packed_empty(1, 64, 64, 128, 128, device=dev)]
    yh_b = [yp_host, torch.empty(yp.shape, dtype=torch.int32).pin_memory()]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for i in range(e2e_steps):
        b = i & 1
        with torch.cuda.stream(streams[b]):
            x_b[b].copy_(x_host, non_blocking=True)
            tn.tn_pack_i8(x_b[b], xp_b[b])
            tn.tn_conv3d_requant_prepared(prep, xp_b[b], xd, wp, 64, g, lo_d, hi_d, yp_b[b])
            yh_b[b].copy_(yp_b[b], non_blocking=True)
    tail = torch.cuda.Event()
    tail.record(streams[1])
    streams[0].wait_event(tail)
    e1.record(streams[0])
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * e2e_steps * C1_MACS / (e2e_ms / 1e3) / 1e9

    # ---- the same, for a caller who keeps ternary tensors in the method's 2-bit storage format
    # on the host: H2D of the packed input (16 MiB instead of 64 MiB of int8 codes),
    # the conv + requant, D2H of the packed output
    xh_packed = torch.empty(xp.shape, dtype=torch.int32).pin_memory()
    xh_packed.copy_(xp)
    xpk_b = [xp_b[0], xp_b[1]]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for i in range(e2e_steps):
        b = i & 1
        with torch.cuda.stream(streams[b]):
            xpk_b[b].copy_(xh_packed, non_blocking=True)
            tn.tn_conv3d_requant_prepared(prep, xpk_b[b], xd, wp, 64, g, lo_d, hi_d, yp_b[b])
            yh_b[b].copy_(yp_b[b], non_blocking=True)
    tail = torch.cuda.Event()
    tail.record(streams[1])
    streams[0].wait_event(tail)
    e1.record(streams[0])
    torch.cuda.synchronize()
    e2p_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2p_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2p_ms = float(t.item())
    e2e_packed = {"value": world * e2e_steps * C1_MACS / (e2p_ms / 1e3) / 1e9, "unit": "GMAC/s", "steps": e2e_steps,
                  "h2d_bytes_per_step": int(xh_packed.numel() * 4), "d2h_bytes_per_step": int(yp.numel() * 4),
                  "step": "H2D of the 2-bit packed input + tn_conv3d_requant_prepared + D2H of the packed output",
                  "pipeline": "double-buffered like e2e"}

    # ---- roofline of the dominant kernel (the conv)
    conv_avg_s = float(np.mean(conv_ms)) / 1e3
    kernel = tn.tn_conv_kernel_for([xd], 64, g)
    operands = tn.tn_conv_operands_for([xd], 64, g)      # 4 = FP4 E2M1 (kind::mxf4), 8 = int8
    uses_tc = kernel == tn.TN_KERNEL_TZ
    clocks = clk.summary()
    if uses_tc:
        bf16 = peaks.get("bf16_tflops", 1590.0)
        # dense peaks as multiples of the measured bf16 one (the guide's nominal ratios):
        # int8 = 2x (4.5 vs 2.25 PFLOP/s), fp4 = 4x (9 vs 2.25)
        ratio = FP4_PER_BF16 if operands == 4 else 2.0
        peak = ratio * bf16
        achieved = 2.0 * C1_MACS / conv_avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak,
                "unit": "TOPS (fp4 e2m1)" if operands == 4 else "TOPS (int8)",
                "frac": achieved / peak,
                "traffic": tn_peaks.get("c1_tz_conv_dram_bytes"),
                "peak_source": f"{ratio:g} x MEASURED_PEAKS.bf16_tflops ("
                               + ("fp4" if operands == 4 else "int8") + "/bf16 nominal ratio)"}
    else:
        popc_per_clk = tn_peaks.get("popc_per_clk_per_sm", 16.0)
        mhz = peaks.get("sm_max_mhz", 1965.0)
        # 2 POPC per 32-lane word pair -> 16 MAC per POPC
        peak = popc_per_clk * 16 * 148 * mhz * 1e6 / 1e12
        achieved = C1_MACS / conv_avg_s / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TMAC/s (POPC pipe)",
                "frac": achieved / peak, "traffic": tn_peaks.get("c1_conv_dram_bytes"),
                "peak_source": f"{popc_per_clk} POPC/clk/SM x 16 MAC/POPC x 148 SM x {mhz} MHz"
                               + (" (measured POPC rate)" if "popc_per_clk_per_sm" in tn_peaks else
                                  " (assumed POPC rate)")}
    roof["kernel"] = "tn_conv3d_requant"
    roof["avg_ms"] = conv_avg_s * 1e3
    roof["share_of_step"] = float(np.sum(conv_ms) / np.sum(split_step_ms))
    roof["timing"] = "conv launch duration from a second pass of the same steps with an event between pack and conv"


    # ---- FCN voxels/s: configs[3], 8 volumes sharded across ranks
    fcn = None
    if not args.no_fcn:
        fcn = bench_fcn(args, tn, torch, dist, world, rank, dev, stream)

    # ---- configs[0]: the small int32-output layer, launch-latency bound -> CUDA-graph replays
    c0 = bench_c0(args, tn, torch, dev) if not args.no_c0 else None
    c2 = bench_c2(args, tn, torch, dev, stream) if not args.no_fcn else None

    # ---- NEXT-4 binary network (Eq. 8): C1 shape with {-1,+1} codes and a sign requant
    binary = None
    if not args.no_binary:
        binary = bench_binary(args, tn, torch, dist, world, rank, dev, stream, flush)

    # ---- NEXT-4: Table 1's 2.5D network over one ROI's 138 stacks
    fcn25 = None
    if not args.no_fcn:
        fcn25 = bench_fcn25(args, tn, torch, dist, world, rank, dev, stream)

    # ---- configs[4]: one 256x512x512 volume, z-slabs over the ranks (NCCL halos)
    c4 = None
    if not args.no_c4:
        c4 = bench_c4(args, tn, torch, dist, world, rank, dev, stream)

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        t0 = time.perf_counter()
        m1 = oracle_c1_sample(x, w, lo, hi, 1)
        dt1 = time.perf_counter() - t0
        planes = int(max(1, min(63, 12.0 / max(dt1, 1e-3))))
        t0 = time.perf_counter()
        mm = oracle_c1_sample(x, w, lo, hi, planes)
        dt = time.perf_counter() - t0
        cpu = {"value": mm / dt / 1e9, "unit": "GMAC/s", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"oracle conv3d+requant over output planes [0,{planes}) of C1's 64 ({dt:.1f} s)",
               "host_cores_visible": cpu_cores()}
        # the other configs' oracle timings, same cores: C0 whole, one C2 volume
        x0, w0, _, _ = synth.conv_config("C0")
        t0 = time.perf_counter()
        oracle.conv3d(x0, w0)
        dt0 = time.perf_counter() - t0
        cfg2 = synth.CONFIGS["C2"]
        p2 = synth.fcn_params(cfg2["seed_params"])
        v2 = synth.ct_volume(cfg2["vol_shape"], seed=cfg2["seeds"][0])
        t0 = time.perf_counter()
        oracle.fcn_forward(v2, p2["t_lo"], p2["t_hi"], p2["weights"], p2["lo"], p2["hi"], p2["pred_w"], p2["pred_b"])
        dt2 = time.perf_counter() - t0
        cpu["other_configs"] = {
            "C0": {"value": 32 * 32 * 32 * 16 * 16 * 27 / dt0 / 1e9, "unit": "GMAC/s", "seconds": dt0},
            "C2": {"value": int(np.prod(cfg2["vol_shape"])) / dt2, "unit": "voxels/s", "seconds": dt2,
                   "sample": "one whole 96x144x144 volume through the oracle FCN"}}

    assert c2 is None or "ms_per_volume" in c2, "fcn_c2 must be the configs[2] timing"
    if rank == 0:
        line = {
            "metric": "ternary conv3d effective GMAC/s (C1, fused requant)",
            "value": value, "unit": "GMAC/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps, "ms_per_step_median": float(np.median(step_ms)),
            "ms_per_step_min": float(np.min(step_ms)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "fp4-e2m1 products, f32 accumulation (integer-exact)" if operands == 4 else "int8 -> int32",
            "data": "synthetic",
            "config": {"workload": C1_WORKLOAD,
                       "step": "tn_pack_i8 (A1) + tn_conv3d_requant_prepared (A2-A4; filter bank prepared once with the weights)",
                       "operands": "2-bit ternary sign/mask bitplanes in HBM, expanded on chip to "
                                   + ("FP4 E2M1 (f32 accumulation, exact below 2^24)" if operands == 4 else
                                      "int8 (int32 accumulation)"),
                       "conv_kernel": {1: "popc (CUDA cores, Eq. 9 XOR/AND/POPC)",
                                       3: "tcgen05 " + ("kind::mxf4 (ternary codes as exact FP4 E2M1, unit "
                                                        "scales)" if operands == 4 else "kind::i8")
                                          + " implicit GEMM, taps as UMMA descriptor offsets, "
                                          "kernel planes merged along N (conv_tz)"}.get(kernel, "?"),
                       "l2": "between timed steps, outside the events: a 256 MiB buffer is zeroed and another "
                             "256 MiB buffer read, so L2 (126 MB) is cold and holds no dirty lines when a step "
                             "starts; the 16.8 MB packed output a step leaves dirty in L2 is written back during "
                             "that flush, i.e. outside the events (about 2.6 us at the measured HBM rate)",
                       "parallelism": f"replicas x{world}", "parity": parity},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GMAC/s", "steps": e2e_steps,
                    "pipeline": "double-buffered: H2D of step i+1 overlaps compute + D2H of step i",
                    "h2d_bytes_per_step": int(x_host.numel()), "d2h_bytes_per_step": int(yp.numel() * 4)},
            "e2e_packed_host": e2e_packed,
            "gpu_launches": 2 * args.steps,
            "clocks": clocks,
            "pack_ms": float(np.mean(pack_ms)),
            "fcn": fcn,
            "fcn_slab": c4,
            "binary": binary,
            "c0": c0,
            "fcn_c2": c2,
            "fcn25_table1": fcn25,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()



# ----------------------------------------------------------------------------- FCN gates + roofline
FP4_PER_BF16 = 4.0     # nominal dense fp4 (9 PFLOP/s) / bf16 (2.25 PFLOP/s), B200_PROFILING.md


def logits_gate(torch, logits, name, p, z0=0, z1=None, dist=None, world=1):
    """Compare this rank's logits with the oracle's values stored at sampled positions of
    configs[2]/[3]/[4] (tests/golden/bench_samples.npz, written by tools/make_bench_golden.py
    from oracle/ only) within reading R13; positions outside [z0, z1) belong to other ranks.
    Exits (refusing to report) on any mismatch on any rank."""
    gold = golden()
    at, ref = gold[f"fcn_{name}_at"], gold[f"fcn_{name}_ref"]
    z1 = logits.shape[2] + z0 if z1 is None else z1
    sel = (at[:, 2] >= z0) & (at[:, 2] < z1)
    ok, checked = True, int(sel.sum())
    if checked:
        a = at[sel].astype(np.int64)
        a[:, 2] -= z0
        idx = tuple(torch.from_numpy(a[:, j]).to(logits.device) for j in range(5))
        got = logits[idx].cpu().numpy().astype(np.float64)
        r = ref[sel].astype(np.float64)
        j = a[:, 1]
        scale = np.abs(p["pred_b"]).astype(np.float64)[j] + np.abs(p["pred_w"]).astype(np.float64).sum(1)[j]
        ok = bool(np.all(np.abs(got - r) <= 1e-5 * np.maximum(np.abs(r), scale)))
    if world > 1:
        t = torch.tensor([int(ok), checked], device=logits.device)
        f = torch.tensor([int(ok)], device=logits.device)
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ok, checked = bool(f.item()), int(t[1].item())
    if not ok:
        print(json.dumps({"error": f"FCN {name} logits differ from the oracle; refusing to report"}), flush=True)
        sys.exit(1)
    return f"passed ({checked} sampled logits vs the oracle's values, reading R13 tolerance)"


def fcn_layer_work(table, shape, nclass, taps=None):
    """Per layer of one forward over `shape` (n,C,D,H,W): algorithmic ternary MACs
    (taps * C_in * C_out per output voxel: 27 for the 3D FCN; 9 / 1 for Table 1's 2D 3x3 / 1x1
    layers) and algorithmic HBM bytes (each input segment's packed buffer read once at its own
    resolution -- the float input for the first layer -- plus the packed output written once;
    the last layer writes fp32 logits instead)."""
    n, C, D, H, W = shape
    cwb = lambda c: 8 * ((c + 31) // 32)
    outs, res = [], []
    for i, (kind, co, s, segs) in enumerate(table):
        if segs[0][0] < 0:
            d, h, w, cin, b_in = D, H, W, C, n * C * D * H * W * 4
        else:
            f, fz = (2 if segs[0][1] else 1), (2 if segs[0][1] == 1 else 1)
            d, h, w = outs[segs[0][0]][1] * fz, outs[segs[0][0]][2] * f, outs[segs[0][0]][3] * f
            cin = sum(outs[sj][0] for sj, _ in segs)
            b_in = sum(n * outs[sj][1] * outs[sj][2] * outs[sj][3] * cwb(outs[sj][0]) for sj, _ in segs)
        do, ho, wo = ((v - 1) // s + 1 for v in (d, h, w))
        outs.append((co, do, ho, wo))
        last = i == len(table) - 1
        b_out = n * do * ho * wo * (4 * nclass if last else cwb(co))
        tp = 27 if taps is None else taps[i]
        res.append({"layer": i + 1, "macs": n * do * ho * wo * co * tp * cin, "bytes": b_in + b_out})
    return res


def fcn_roofline(torch, net, x, logits, ws, stream, forward_ms, peaks, reps=3, taps=None):
    """Per-layer binding roofline of one FCN forward: each layer's bound is the larger of its
    algorithmic MACs at the fp4 dense tensor peak (4 x measured bf16, the guide's nominal
    ratio; every layer's ternary products are exact in E2M1) and its algorithmic bytes at the
    measured HBM bandwidth.  Layers are timed one by one (tn_fcn_forward_range, CUDA events on
    the launching stream); frac = sum of the bounds / the whole forward's device time."""
    L = len(net.table)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
    ms = np.zeros(L)
    for _ in range(reps):
        # the host queues all launches while the GPU spins, so no event pair brackets a host gap
        torch.cuda._sleep(int(2_000_000 * (2.0 + 4.0 * forward_ms)))
        ev[0].record(stream)
        for i in range(L):
            net.forward_range(x, i, i + 1 if i < L - 1 else -1, logits=logits, ws=ws, stream=stream)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        ms += [ev[i].elapsed_time(ev[i + 1]) for i in range(L)]
    ms /= reps
    hbm = peaks.get("hbm_gbs", 6548.2) * 1e9
    mac_peak = FP4_PER_BF16 * peaks.get("bf16_tflops", 1662.6) * 1e12 / 2.0
    per, bound_ms = [], 0.0
    for wk, t in zip(fcn_layer_work(net.table, tuple(x.shape), net.nclass, taps), ms):
        tt, th = wk["macs"] / mac_peak * 1e3, wk["bytes"] / hbm * 1e3
        b = max(tt, th)
        bound_ms += b
        per.append({"layer": wk["layer"], "ms": float(t), "bound_ms": b, "bound": "tensor" if tt >= th else "hbm",
                    "frac": b / float(t), "gmac": wk["macs"] / 1e9, "mb": wk["bytes"] / 1e6})
    dom = max(per, key=lambda r: r["ms"])
    dom_t = dom["bound"] == "tensor"
    achieved = dom["gmac"] * 1e9 / (dom["ms"] / 1e3) / 1e12 if dom_t else dom["mb"] * 1e6 / (dom["ms"] / 1e3) / 1e9
    return {"bound": "per-layer max(fp4 tensor, hbm)", "bound_ms": bound_ms, "achieved_ms": forward_ms,
            "frac": bound_ms / forward_ms, "layers_sum_ms": float(ms.sum()),
            "dominant": {"layer": dom["layer"], "bound": dom["bound"], "achieved": achieved,
                         "peak": mac_peak / 1e12 if dom_t else hbm / 1e9,
                         "unit": "TMAC/s (fp4 dense)" if dom_t else "GB/s", "frac": dom["frac"], "traffic": None},
            "per_layer": per,
            "peak_source": "fp4 = 4 x MEASURED_PEAKS.bf16_tflops / 2 MAC; HBM = MEASURED_PEAKS.hbm_gbs",
            "timing": "layers timed one at a time (tn_fcn_forward_range, events between launches queued behind a "
                      "device spin so no host gap falls between events); "
                      "frac uses the whole forward's time"}


def bench_c2(args, tn, torch, dev, stream):
    """configs[2]: one 1x1x96x144x144 CT-like volume through the FCN (device time per volume)."""
    cfg = synth.CONFIGS["C2"]
    shape = cfg["vol_shape"]
    p = synth.fcn_params(cfg["seed_params"])
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"], device=dev)
    x = torch.from_numpy(synth.ct_volume(shape, seed=cfg["seeds"][0])).to(dev)
    net.prepare(shape)   # filter-bank operand images, built once (tn_fcn_prepare)
    ws = net.workspace(shape, dev)
    logits = torch.empty((1, 2) + shape[2:], dtype=torch.float32, device=dev)
    net(x, logits=logits, ws=ws)
    torch.cuda.synchronize()
    parity = logits_gate(torch, logits, "c2", p)
    net(x, logits=logits, ws=ws)
    torch.cuda.synchronize()
    steps = max(3, args.fcn_steps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)          # host queues ahead of the GPU (outside the events)
    a.record(stream)
    for _ in range(steps):
        net(x, logits=logits, ws=ws)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    vox = int(np.prod(shape[2:]))
    roof = fcn_roofline(torch, net, x, logits, ws, stream, ms, bench_peaks())
    return {"metric": "FCN voxels/s", "value": vox / (ms / 1e3), "unit": "voxels/s", "ms_per_volume": ms,
            "config": "C2: one CT-like volume 1x1x96x144x144 (BASELINE configs[2]); every layer bit-exact at "
                      "this size in test_fcn_c2_full_size_matches_oracle", "steps": steps, "parity": parity,
            "roofline": roof}


FCN25_TAPS = [9, 9, 9, 9, 9, 9, 1, 1, 9, 9, 9, 9, 9, 9]      # Table 1: 3x3 layers, 1x1 at #7 / #8


def bench_fcn25(args, tn, torch, dist, world, rank, dev, stream):
    """NEXT-4: Table 1's own network (reading R18) -- the ternary 2.5D U-Net on
    15-slice stacks of 240 x 176 -- over the 138 stacks of one CT-like ROI volume,
    sharded over the ranks by stack.  Parity-gated on the oracle's logits of stacks 0-3."""
    p = synth.fcn25_params()
    x_all = synth.ct_stacks(synth.ROI_STACKS, synth.STACK_H, synth.STACK_W, seed=300)
    mine = [i for i in range(synth.ROI_STACKS) if i % world == rank]
    x = torch.from_numpy(np.ascontiguousarray(x_all[mine])).to(dev)
    del x_all
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"],
                        table=tn.fcn25_table(), device=dev, c_in=15)
    net.prepare(tuple(x.shape))
    ws = net.workspace(tuple(x.shape), dev)
    logits = torch.empty((x.shape[0], 2, 1, synth.STACK_H, synth.STACK_W), dtype=torch.float32, device=dev)
    net(x, logits=logits, ws=ws)
    torch.cuda.synchronize()
    # stacks 0-3 are this rank's local stacks 0..: rank r holds global stack r at local 0
    gold = golden()
    at, ref = gold["fcn25_at"], gold["fcn25_ref"]
    sel = np.isin(at[:, 0], mine)
    ok = True
    if sel.any():
        a = at[sel].astype(np.int64)
        a[:, 0] = [mine.index(v) for v in a[:, 0]]
        idx = tuple(torch.from_numpy(a[:, j]).to(dev) for j in range(5))
        got = logits[idx].cpu().numpy().astype(np.float64)
        r = ref[sel].astype(np.float64)
        scale = np.abs(p["pred_b"]).astype(np.float64)[a[:, 1]] + np.abs(p["pred_w"]).astype(np.float64).sum(1)[a[:, 1]]
        ok = bool(np.all(np.abs(got - r) <= 1e-5 * np.maximum(np.abs(r), scale)))
    if world > 1:
        f = torch.tensor([int(ok)], device=dev)
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
        ok = bool(f.item())
    if not ok:
        print(json.dumps({"error": "Table-1 2.5D network logits differ from the oracle; refusing to report"}), flush=True)
        sys.exit(1)
    steps = max(2, args.fcn_steps)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)          # host queues ahead of the GPU (outside the events)
    e0.record(stream)
    for _ in range(steps):
        net(x, logits=logits, ws=ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    macs = sum(w["macs"] for w in fcn_layer_work(net.table, (1, 15, 1, synth.STACK_H, synth.STACK_W), 2, FCN25_TAPS))
    roof = fcn_roofline(torch, net, x, logits, ws, stream, ms, bench_peaks(), taps=FCN25_TAPS) if world == 1 else None
    return {"metric": "Table-1 2.5D U-Net stacks/s", "value": synth.ROI_STACKS / (ms / 1e3), "unit": "stacks/s",
            "ms_per_volume": ms, "effective_gmacs": synth.ROI_STACKS * macs / (ms / 1e3) / 1e9,
            "macs_per_stack": macs, "roofline": roof, "steps": steps,
            "parity": f"passed ({int(sel.sum())} sampled logits of stacks 0-3 vs the oracle's values, R13)",
            "config": f"{synth.ROI_STACKS} stacks of 15 x {synth.STACK_H} x {synth.STACK_W} (one 138-slice ROI), "
                      "Table 1 channels 32-64-128-256, 2D convs (3x3, 1x1 at the lowest level), stride-2 rows "
                      "for AvgPool2D, nearest x2 Upsample2D; #1-#3 on the TZ tensor-core kernel, #4-#14 on the wide one-plane tensor-core kernel"}


def bench_c0(args, tn, torch, dev):
    """configs[0] (1x16x32x32x32, 16 -> 16, int32 channel-last output): 226 M MAC per launch is a
    few microseconds of work, so it is timed as CUDA-graph replays of 100 back-to-back launches
    (SURVEY 8(d)); parity-checked first (sampled outputs vs the oracle's values)."""
    x, w, _, _ = synth.conv_config("C0")
    xd = tn.dims(*x.shape)
    xp = tn.tn_pack_i8(torch.from_numpy(x).to(dev))
    wp = tn.tn_pack_weights(torch.from_numpy(w).to(dev))
    segs = [(xp, xd, 0, wp)]
    prep = tn.tn_conv_prepare(segs, 16, tn.geom(), requant=False)   # filter bank prepared once, as in C1
    y = tn.tn_conv3d_seg_prepared(prep, segs, 16, tn.geom(), requant=False)
    torch.cuda.synchronize()
    gold = golden()
    n_, k_, z_, y_, x_ = gold["c0_at"].T
    if not np.array_equal(y.cpu().numpy()[n_, z_, y_, x_, k_], gold["c0_ref"]):
        print(json.dumps({"error": "C0 parity check failed; refusing to report"}), flush=True)
        sys.exit(1)
    st = torch.cuda.Stream(device=dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(100):
            tn.tn_conv3d_seg_prepared(prep, segs, 16, tn.geom(), y=y, requant=False, stream=st)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 500
    macs = 32 * 32 * 32 * 16 * 16 * 27
    return {"metric": "ternary conv3d effective GMAC/s (C0, int32 output)", "unit": "GMAC/s",
            "value": macs / (us / 1e6) / 1e9, "us_per_launch": us,
            "config": "C0: 1x16x32x32x32 16->16 3x3x3 s1 p1, int32 channel-last output (BASELINE configs[0]); "
                      "tn_conv3d_seg_prepared (filter bank prepared once, as in C1); "
                      "CUDA-graph replays of 100 launches, L2-resident (2.3 MB working set)",
            "parity": f"passed ({len(gold['c0_ref'])} sampled int32 outputs vs the oracle's values)"}


def bench_binary(args, tn, torch, dist, world, rank, dev, stream, flush):
    """Binary XNOR variant (Eq. 8): C1's shape with binary
    activations and weights (ternary codes with all-ones masks) and the sign activation
    lo = hi - 1; the same pack + fused conv/requant step, sampled parity against the oracle."""
    shape = (1, 64, 64, 128, 128)
    x, w, lo, hi = synth.binary_config()
    x_d = torch.from_numpy(x).to(dev)
    lo_d, hi_d = torch.from_numpy(lo).to(dev), torch.from_numpy(hi).to(dev)
    wp = tn.tn_pack_weights(torch.from_numpy(w).to(dev))
    xd, g = tn.dims(*shape), tn.geom(1, 1, 1)
    xp = tn.packed_empty(*shape, device=dev)
    yp = tn.packed_empty(*shape, device=dev)

    def step():
        tn.tn_pack_i8(x_d, xp)
        tn.tn_conv3d_requant(xp, xd, wp, 64, g, lo_d, hi_d, yp)

    step()
    torch.cuda.synchronize()
    gold = golden()
    if not np.array_equal(ternary_at(yp, gold["bin_at"]), gold["bin_ref"]):
        print(json.dumps({"error": "binary parity check failed; refusing to report"}), flush=True)
        sys.exit(1)
    parity = f"passed ({len(gold['bin_ref'])} sampled outputs vs the oracle's values)"
    for _ in range(max(3, args.warmup)):
        step()
    steps = max(5, min(args.steps, 20))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)          # host queues ahead of the GPU (outside the events)
    for i in range(steps):
        flush()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"metric": "binary conv3d effective GMAC/s", "unit": "GMAC/s",
            "value": world * steps * C1_MACS / (ms / 1e3) / 1e9, "ms_per_step": ms / steps, "steps": steps,
            "config": "C1 shape, binary {-1,+1} activations and weights (all-ones masks), sign requant "
                      "lo = hi - 1, pack + fused conv/requant, L2 flushed between steps",
            "parity": parity}


def bench_fcn(args, tn, torch, dist, world, rank, dev, stream):
    cfg = synth.CONFIGS["C3"]
    p = synth.fcn_params(cfg["seed_params"])
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"],
                        device=dev)
    mine = [i for i in range(len(cfg["seeds"])) if i % world == rank]
    shape = cfg["vol_shape"]
    # this rank's volumes go through ONE batched forward (n = 8 / world): every layer is a
    # single launch over all of them, so partition tails and kernel prologues are paid once
    xb = torch.cat([torch.from_numpy(synth.ct_volume(shape, seed=cfg["seeds"][i])) for i in mine], 0).to(dev)
    bshape = (len(mine),) + tuple(shape[1:])
    net.prepare(bshape)
    ws = net.workspace(bshape, dev)
    logits = torch.empty((len(mine), 2) + shape[2:], dtype=torch.float32, device=dev)
    net(xb, logits=logits, ws=ws)
    torch.cuda.synchronize()
    # volume 0 (seed 100) is always this rank-0 batch's first volume
    parity = logits_gate(torch, logits[:1] if rank == 0 else logits[:0], "c3", p, dist=dist, world=world)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)          # host queues ahead of the GPU (outside the events)
    e0.record(stream)
    for _ in range(args.fcn_steps):
        net(xb, logits=logits, ws=ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    vox = int(np.prod(shape[2:]))
    total_vox = args.fcn_steps * len(cfg["seeds"]) * vox
    roof = fcn_roofline(torch, net, xb, logits, ws, stream, ms / args.fcn_steps, bench_peaks())
    return {"metric": "FCN voxels/s", "value": total_vox / (ms / 1e3), "unit": "voxels/s", "parity": parity,
            "roofline": roof,
            "config": "C3: 8 CT-like volumes 1x1x128x256x256 sharded over the ranks (8 / N each), one batched "
                      "forward per rank (BASELINE configs[3])",
            "ms_per_batch": ms / args.fcn_steps, "effective_gmacs": total_vox * FCN_MACS_PER_VOXEL / (ms / 1e3) / 1e9,
            "steps": args.fcn_steps, "gpu_launches_per_forward": 14, "scaling": "strong (fixed batch of 8)"}


def bench_c4(args, tn, torch, dist, world, rank, dev, stream):
    cfg = synth.CONFIGS["C4"]
    shape = cfg["vol_shape"]
    D, H, W = shape[2:]
    p = synth.fcn_params(cfg["seed_params"])
    net = tn.TernaryFCN(p["weights"], p["lo"], p["hi"], p["pred_w"], p["pred_b"], p["t_lo"], p["t_hi"], device=dev)
    net.prepare(shape)
    z0, z1 = rank * D // world, (rank + 1) * D // world
    vol = synth.ct_volume(shape, seed=cfg["seeds"][0])
    x = torch.from_numpy(np.ascontiguousarray(vol[:, :, z0:z1])).to(dev)
    del vol
    if world > 1:
        comm = tn.Comm(rank, world)
        nb = int(tn.lib.tn_fcn_slab_workspace_bytes(net.handle, tn.dims(*shape), z0, z1))
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        logits = torch.empty((1, 2, z1 - z0, H, W), dtype=torch.float32, device=dev)
        if args.c4_halo == "p2p":
            halo = tn.HaloP2P(net, shape, rank, world)
            run = lambda: halo.forward(x, logits=logits)
            mode = (f"z-slabs of {D // world} planes per rank, halos stored by the conv epilogues into the "
                    "neighbours' memory (CUDA IPC / NVLink) + device flags (NEXT-1)")
        else:
            run = lambda: net.forward_slab(comm, x, shape, z0, z1, logits=logits, ws=ws)
            mode = f"z-slabs of {D // world} planes per rank, NCCL halo exchange per layer"
    else:
        ws = net.workspace(shape, dev)
        logits = torch.empty((1, 2, D, H, W), dtype=torch.float32, device=dev)
        run = lambda: net(x, logits=logits, ws=ws)
        mode = "whole volume on one GPU"
    run()
    torch.cuda.synchronize()
    parity = logits_gate(torch, logits, "c4", p, z0=z0, z1=z1, dist=dist, world=world)
    steps = max(2, args.fcn_steps)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)          # host queues ahead of the GPU (outside the events)
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    vox = D * H * W
    sched = None
    if world == 1 and not args.no_slab_schedules:
        # single-GPU view of the two halo schedules: 8 slabs run layer-major on this device
        # (the same kernels and halo traffic as 8 ranks, serialised), copies vs NEXT-1
        del ws
        nsl = 8
        nb = int(tn.lib.tn_fcn_slabs_local_workspace_bytes(net.handle, tn.dims(*shape), nsl))
        wsl = torch.empty(nb, dtype=torch.uint8, device=dev)
        whole = logits.clone()
        sched = {"slabs": nsl}
        for name, fn in (("copies", net.forward_slabs_local), ("p2p_epilogue", net.forward_slabs_local_p2p)):
            fn(x, nsl, logits=logits, ws=wsl)
            torch.cuda.synchronize()
            if not torch.equal(logits, whole):
                print(json.dumps({"error": f"slab schedule {name} differs from the whole volume"}), flush=True)
                sys.exit(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(steps):
                fn(x, nsl, logits=logits, ws=wsl)
            b.record(stream)
            torch.cuda.synchronize()
            sched[name + "_ms_per_volume"] = a.elapsed_time(b) / steps
        sched["note"] = "bit-identical to the whole-volume logits (checked before timing)"
        del wsl
    roof = None
    if world == 1:
        wsr = net.workspace(shape, dev)
        roof = fcn_roofline(torch, net, x, logits, wsr, stream, ms, bench_peaks())
        del wsr
    return {"metric": "FCN voxels/s", "value": vox / (ms / 1e3), "unit": "voxels/s", "parity": parity,
            "roofline": roof, "slab_schedules_1gpu": sched,
            "config": f"C4: one CT-like volume 1x1x{D}x{H}x{W} (BASELINE configs[4]); {mode}",
            "ms_per_volume": ms, "effective_gmacs": vox * FCN_MACS_PER_VOXEL / (ms / 1e3) / 1e9,
            "steps": steps, "scaling": "strong (fixed volume)"}


if __name__ == "__main__":
    main()
