"""Sync-EASGD throughput on B200 (BASELINE.json: "Sync EASGD samples/s at
1/2/4/8 B200; elastic-update HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model lenet|cifar-quick|alexnet]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --impl reference ...                      (CPU reference arm)

A step is one Sync-EASGD round: every worker (one per GPU) samples b images
from its HBM-resident synthetic dataset, runs forward/backward, the packed
weights are summed (NCCL allreduce over NVLink, overlapped with the
round's forward/backward: sync-easgd3) and the fused elastic update runs.
``value`` = all ranks' samples / max-over-ranks device time of K graph-
replayed rounds. ``e2e`` = the same through run_trainer's host data path
(pinned host batch -> H2D every round, loss D2H every round).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # C1/C2 synthetic MNIST for LeNet, C3 CIFAR, C5 ImageNet-shaped
    "lenet": dict(classes=10, per_class=6000, b=64, eta=0.05, rho=0.25, test_per_class=100),
    "cifar-quick": dict(classes=10, per_class=5000, b=64, eta=0.05, rho=0.25, test_per_class=100),
    "alexnet": dict(classes=1000, per_class=1, b=128, eta=0.01, rho=0.1, test_per_class=0),
}


METRIC = "Sync EASGD samples/s (elastic-averaging round, 1 worker per B200)"
CONFIG_NAME = {"lenet": "configs[1]: Sync EASGD, LeNet synthetic MNIST, 1 worker per GPU",
               "cifar-quick": "Sync EASGD, CIFAR-quick synthetic CIFAR-10, 1 worker per GPU",
               "alexnet": "configs[4]: Sync EASGD, AlexNet synthetic ImageNet 224x224, weak scaling"}


def workload_config(args, b: int, world: int) -> dict:
    return {"workload": f"{CONFIG_NAME[args.model]} (sync-easgd3, b={b}/worker)", "model": args.model,
            "global_batch": world * b, "per_worker_batch": b, "parallelism": f"dp{world}",
            "l2": "update kernel timed with L2 flushed; step inputs resident"}


def traffic(kernel: str, model: str):
    """Per-launch DRAM bytes (read + write) of a roofline kernel from the
    committed ncu --set full capture summary (profiles/traffic.json)."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return t.get(f"{kernel}:{model}", t.get(kernel))
    except Exception:
        return None


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def make_data(model: str, spec, seed: int = 0):
    from paper_1708_02983_b200.datasets import Dataset, gen_synthetic, normalize

    wl = WORKLOADS[model]
    d = spec.input_dim
    if model == "alexnet":
        # 1000 x 150528 fp32 (0.6 GB); per-class blobs, features already unit-variance
        train = gen_synthetic(wl["classes"], d, wl["per_class"], seed=seed, separation=5.0, dtype=np.float32)
        return train, None
    train = normalize(gen_synthetic(wl["classes"], d, wl["per_class"], seed=seed, separation=5.0))
    return train, None


class ClockSampler:
    """SM clock + throttle reasons during the timed region: NVML every 10 ms
    (the device matched by PCI bus id), nvidia-smi every 0.2 s if NVML is
    unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.nvml = None
        try:
            import pynvml as N

            N.nvmlInit()
            try:
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                try:
                    h = N.nvmlDeviceGetHandleByPciBusId(bus)
                except Exception:
                    h = N.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = N.nvmlDeviceGetHandleByIndex(index)
            self.nvml = (N, h, N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    def _run(self):
        if self.nvml is not None:
            N, h, mx = self.nvml
            while not self._stop.is_set():
                try:
                    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                    bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append([str(sm), str(mx)] + [
                        "Active" if bits & m else "Not Active" for m in (0x8, 0x40, 0x20, 0x4)])
                except Exception:
                    pass
                self._stop.wait(0.01)
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.th.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


class NvlinkCounter:
    """NVLink bytes this GPU sent / received over a region, from NVML's
    per-link data counters (NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES, summed
    over links; throughput counters in KiB as a fallback). None when the
    driver exposes neither."""

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            try:
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.fields = None
            for tx, rx, scale in ((getattr(N, "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", None),
                                   getattr(N, "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", None), 1),
                                  (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                                   1024)):
                if tx is None:
                    continue
                self.fields = (tx, rx, scale)
                v = self.read()
                if v is not None and (v[0] > 0 or v[1] > 0):
                    break
            self.ok = self.fields is not None and self.read() is not None
        except Exception:
            self.ok = False

    def read(self):
        N = self.N
        tx, rx, scale = self.fields
        tot = [0, 0]
        try:
            for link in range(18):
                vals = N.nvmlDeviceGetFieldValues(self.h, [(tx, link), (rx, link)])
                for i, v in enumerate(vals):
                    if v.nvmlReturn == 0:
                        tot[i] += int(v.value.ullVal) * scale
            return tot
        except Exception:
            return None


def dist_setup(n_gpus: int):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def time_update_kernel(eng, reps: int = 20):
    """Live CUDA-event timing of the round's elastic-update kernel on the
    training stream with copies of the engine's buffers, L2 flushed before
    each launch. Algorithmic bytes per param: one worker in total (P = 1):
    W, C read+write and G read = 20 (S = W(t), esgd_sync_update_solo_f32);
    otherwise C read+write and S read (12) + 12 per local replica (W
    read+write, G read), plus the S_next write (4) when the update also forms
    the next round's replica sum (esgd_sync_update_sum_f32)."""
    import torch

    from paper_1708_02983_b200.updates import sync_update_, sync_update_solo_, sync_update_sum_

    n, nrep = eng.n, eng.nrep
    solo = getattr(eng, "solo", False)
    fused = getattr(eng, "fused_sum", False) and not solo
    # work on copies so the training state is untouched
    W, G, C, S = eng.W.clone(), eng.G.clone(), eng.C.clone(), eng.S.clone()
    flush = torch.empty(int(256e6) // 4, device=W.device)
    times = []
    for i in range(reps + 3):
        flush.zero_()  # evict L2 (126 MB) so the stream comes from HBM
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if solo:
            sync_update_solo_(W, G, C, n, eng.cfg.hyper)
        elif fused:
            sync_update_sum_(W, G, C, S, S, n, eng.P, eng.cfg.hyper)
        else:
            sync_update_(W, G, C, S, n, eng.P, eng.cfg.hyper)
        b.record()
        b.synchronize()
        if i >= 3:
            times.append(a.elapsed_time(b) / 1e3)
    if solo:
        return n * 20, float(np.mean(times)), "esgd_sync_update_solo_f32 (k_sync_update_solo4)", "sync_update_solo"
    bytes_ = n * (12 + 12 * nrep + (4 if fused else 0))
    name = "esgd_sync_update_sum_f32 (k_sync_update_sum4)" if fused else "esgd_sync_update_f32 (k_sync_update<4>)"
    return bytes_, float(np.mean(times)), name, ("sync_update_sum" if fused else "sync_update")


def time_dominant_gemm(eng, reps: int = 10):
    """Record one eager gradient pass, re-launch its largest tcgen05 GEMM
    alone with CUDA events (warm). Returns (desc-summary, flops, seconds)."""
    import ctypes as C

    import torch

    from paper_1708_02983_b200 import _lib
    from paper_1708_02983_b200.device import stream_ptr

    net = eng.plan.net
    net.record = []
    eng.plan.gradient(eng.G.clone(), eng.W.clone(), stream_ptr())
    torch.cuda.synchronize()
    recs, net.record = net.record, None
    tcs = [r for r in recs if r[0] == "tc"]
    if not tcs:
        return None
    lib = _lib.load()
    best = None
    for kind, d, flops in tcs:
        for _ in range(2):
            _lib.check(lib.esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            _lib.check(lib.esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / reps / 1e3
        if best is None or t > best[2]:
            best = (f"m={d.m} n={d.n} k={d.k} batch={d.batch} a_major={d.a_major} b_major={d.b_major}",
                    flops, t, d.precision, f"tc_gemm:{d.m}x{d.n}x{d.k}")
    return best


def run_device(args):
    import torch
    import torch.distributed as dist

    from paper_1708_02983_b200 import HyperParams, make_config, network
    from paper_1708_02983_b200.trainers import NetworkProblem
    from paper_1708_02983_b200.trainers.synchronous import SyncEngine

    world, rank, local = dist_setup(args.gpus)
    wl = WORKLOADS[args.model]
    b = args.batch or wl["b"]
    spec = network.MODELS[args.model](seed=0)
    train, test = make_data(args.model, spec)
    prob = NetworkProblem(spec, train, test)
    P = world  # one worker per GPU (weak scaling)
    cfg = make_config("sync-easgd3", workers=P, iterations=args.steps + args.warmup, batch_size=b,
                      hyper=HyperParams(eta=wl["eta"], rho=wl["rho"]), seed=3)
    eng = SyncEngine(cfg, prob, use_graph=True, profile_rounds=min(2, args.warmup))
    for _ in range(args.warmup):
        eng.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvl = NvlinkCounter(local) if world > 1 else None
    nvl0 = nvl.read() if (nvl is not None and nvl.ok) else None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ -> the step's launch list
        t0.record()
        for _ in range(args.steps):
            eng.step()
        t1.record()
        torch.cuda.nvtx.range_pop()
        t1.synchronize()
        if world > 1:
            dist.barrier()
    dt = t0.elapsed_time(t1) / 1e3
    nvlink = None
    if nvl0 is not None:
        nvl1 = nvl.read()
        if nvl1 is not None:
            # algorithmic NVLink bytes per GPU per round: NVLS ld_reduce of 1/N of S from the
            # N-1 peers + multicast of that slice of C to them: 2 (N-1)/N * 4|W| each way
            # (the same as a ring allreduce's 2 (N-1)/N * 4|W|)
            alg = 2.0 * (world - 1) / world * 4 * eng.ldw
            nvlink = {"tx_bytes_per_step": (nvl1[0] - nvl0[0]) / args.steps,
                      "rx_bytes_per_step": (nvl1[1] - nvl0[1]) / args.steps,
                      "algorithmic_bytes_per_step_each_way": alg, "source": "nvml per-link counters, rank 0 GPU"}
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    samples = args.steps * P * b
    value = samples / dt

    # elastic-update kernel roofline (live, CUDA events, L2 flushed)
    upd_bytes, upd_s, upd_name, upd_key = time_update_kernel(eng)
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    src = "MEASURED_PEAKS.json" if not pk.get("_fallback") else "fallback (B200_PROFILING.md)"
    roof_upd = {"kernel": upd_name, "bound": "hbm",
                "achieved": round(upd_bytes / upd_s / 1e9, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(upd_bytes / upd_s / 1e9 / hbm, 4), "traffic": traffic(upd_key, args.model),
                "algorithmic_bytes_per_launch": upd_bytes, "launch_s": upd_s,
                "peak_source": f"{src} hbm_gbs (copy)"}
    # dominant kernel of the step: the largest tcgen05 3xTF32 GEMM launch,
    # re-launched alone (warm) with CUDA events; tf32-pipe rate = 3 x 2MNK / t
    # against the measured bf16 peak / 2 (nominal dense tf32 = bf16 / 2)
    dom = time_dominant_gemm(eng)
    if dom is not None:
        desc, fl, t, prec, tkey = dom
        tf32_peak = pk.get("bf16_tflops", 1590.0) / 2
        ach = prec * fl / t / 1e12
        # achieved = ALGORITHMIC flops (2MNK, the fp32 product the GEMM delivers) per
        # launch / launch time, against the tensor-core peak of the kind the kernel
        # issues (tf32 = bf16 / 2). 3xTF32 issues 3 tf32 MMAs per product, so the
        # algorithmic fraction is at most 1/3; the same launch is also given as a
        # fraction of the 3xTF32 emulation peak (peak / 3) and of the kind::tf32
        # issue-rate floor (tensor-pipe work = 3 x algorithmic)
        alg = fl / t / 1e12
        floor = 148 * 4096 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        roof = {"kernel": f"esgd_tc_gemm_f32 (k_tc_gemm, {desc})", "bound": "tensor",
                "achieved": round(alg, 1), "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
                "frac": round(alg / tf32_peak, 4), "traffic": traffic(tkey, args.model),
                "launch_s": t, "algorithmic_flops_per_launch": fl,
                "peak_source": f"{src} bf16_tflops / 2 (tf32 = half the bf16 rate)",
                "emulation_peak_tflops": round(tf32_peak / prec, 1),
                "frac_of_emulation_peak": round(alg * prec / tf32_peak, 4),
                "tf32_pipe_tflops": round(ach, 1),
                # the issue-rate floor of kind::tf32 MMAs (4096 flop/cycle/SM, measured at the
                # floor in isolation by tools/probe_mma_rate.cu) at the max SM clock
                "tensor_floor_tflops": round(floor, 1),
                "frac_of_floor": round(ach / floor, 4)}
    else:  # no GEMM reaches the tensor-core threshold (LeNet): the round is launch/latency-bound
        roof = dict(roof_upd, note="no tcgen05 GEMM in this round (all GEMMs below the tensor-core "
                    "threshold run on the FFMA kernel); the round is launch/latency-bound "
                    "(profiles/r01_launches_lenet.md), the update kernel is the one HBM-bound launch")

    # e2e: run_trainer's host data path (pinned batch H2D + loss D2H every round)
    e2e = run_e2e(args, spec, train, cfg, world) if not args.no_e2e else None

    # exposed communication of the graph-replayed round (its twin without the
    # collective, replayed the same way), measured after the timed rounds
    comm = eng.exposed_comm(rounds=max(5, min(20, args.steps)))
    comm_frac = comm["fraction"]
    if world > 1:  # the collective alone: achieved NVLink bandwidth (NVML link counters read N/A here)
        comm["alone"] = eng.time_collective(reps=10)
    cpu = cpu_baseline(args, spec, train) if (rank == 0 and world == 1 and not args.no_cpu) else None
    out = {
        "metric": METRIC,
        "value": round(value, 1), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core GEMMs)",
        "data": "synthetic (gen_synthetic blobs, HBM-resident)",
        "config": dict(workload_config(args, b, world), params=eng.n, graph=eng.graph is not None,
                       collective=eng.collective),
        "roofline": roof,
        "roofline_update": roof_upd,
        "comm_fraction_exposed": round(comm_frac, 4),
        "comm": comm,
        "nvlink": nvlink,
        "gpu_launches": launches_per_step(eng) * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        # captured graphs hold NCCL work; tearing the communicator down under
        # them can hang, so release them, sync, and leave without a teardown
        eng.graph, eng.graphs = None, [None, None]
        torch.cuda.synchronize()
        dist.barrier()
        sys.stdout.flush()
        os._exit(0)


def launches_per_step(eng) -> int:
    """libesgd kernels in one round, counted from a CUPTI trace of one eager
    round (torch.profiler; outside the timed region)."""
    import torch

    from paper_1708_02983_b200.device import stream_ptr

    W, G = eng.W.clone(), eng.G.clone()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        eng.plan.gradient(G, W, stream_ptr())
        from paper_1708_02983_b200.fabric.collectives import replica_sum_
        from paper_1708_02983_b200.updates import sync_update_, sync_update_solo_, sync_update_sum_
        if getattr(eng, "solo", False):
            sync_update_solo_(W, G, eng.C.clone(), eng.n, eng.cfg.hyper)
        elif getattr(eng, "fused_sum", False):
            S = eng.S.clone()
            sync_update_sum_(W, G, eng.C.clone(), S, S, eng.n, eng.P, eng.cfg.hyper)
        else:
            replica_sum_(eng.S.clone(), W, eng.n)
            sync_update_(W, G, eng.C.clone(), eng.S.clone(), eng.n, eng.P, eng.cfg.hyper)
        torch.cuda.synchronize()
    n = 0
    for e in prof.events():
        if getattr(e, "device_type", None) is not None and "esgd" in e.name and "Memcpy" not in e.name:
            if str(e.device_type).endswith("CUDA"):
                n += 1
    return n


def run_e2e(args, spec, train, cfg, world):
    """End to end through the package's host-fed runner (trainers.HostFedRun):
    the dataset in pinned host memory, every round's batch H2D inside the
    round, the round's loss read back to the host after every round."""
    import torch

    from paper_1708_02983_b200.trainers import HostFedRun, NetworkProblem

    run = HostFedRun(cfg, NetworkProblem(spec, train, None))
    for _ in range(max(1, args.warmup)):
        run.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run.step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    b = cfg.batch_size
    return {"value": round(args.steps * cfg.cluster.workers * b / dt, 1), "unit": "samples/s",
            "h2d_bytes_per_step": run.h2d_bytes, "d2h_bytes_per_step": run.d2h_bytes, "path": run.path}


class CpuRound:
    """The CPU oracle (numpy restatement of the reference's sync round,
    trainers/synchronous.py:57-64, simulated engine) on this host's cores, at
    the native arm's per-worker batch: P workers' gradients, the tree sum and
    the elastic worker / center steps."""

    def __init__(self, args, train, workers: int = 1):
        from oracle import esgd_oracle as O

        self.O = O
        layers = {"lenet": O.LENET, "cifar-quick": O.CIFAR_QUICK, "alexnet": O.alexnet_layers(1000)}[args.model]
        self.wl = WORKLOADS[args.model]
        self.b = args.batch or self.wl["b"]
        self.P = workers
        self.model = args.model
        self.prob = O.NetProblem(*layers, train.samples, train.labels, seed=0, dtype=np.float32)
        self.rngs = [O.worker_rng(3, w) for w in range(workers)]
        w0 = self.prob.init_weights()
        self.w = [w0.copy() for _ in range(workers)]
        self.c = w0.copy()
        self.cores = host_info()["threads"]
        self.round()  # warm-up (BLAS init, page faults)

    def round(self):
        O, wl = self.O, self.wl
        g = [self.prob.gradient(w, r, self.b) for w, r in zip(self.w, self.rngs)]
        s = O.tree_sum(self.w)
        self.w = [O.easgd_worker_step(w, gi, self.c, wl["eta"], wl["rho"]) for w, gi in zip(self.w, g)]
        self.c = O.easgd_center_step_from_sum(self.c, s, self.P, wl["eta"], wl["rho"])

    def sample(self, budget_s: float, max_rounds: int = 1 << 30):
        """Whole rounds until ~budget_s has passed (at least one): (rounds, seconds)."""
        rounds, t0 = 0, time.perf_counter()
        while True:
            self.round()
            rounds += 1
            elapsed = time.perf_counter() - t0
            if elapsed >= budget_s or rounds >= max_rounds:
                return rounds, elapsed

    def describe(self, rounds: int) -> str:
        return (f"{rounds} full sync-easgd rounds of {self.model}, P={self.P}, b={self.b}/worker (the native "
                f"arm's per-worker batch), numpy/OpenBLAS fp32 (oracle/esgd_oracle.py restating "
                f"trainers/synchronous.py:57-64, simulated engine)")


def host_info() -> dict:
    """CPU model, thread counts and the BLAS the oracle runs on."""
    model = None
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info

        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads"), "version": i.get("version")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:
        pass
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
                  or len(os.sched_getaffinity(0)))
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "threads": threads, "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"), "blas": blas}


def update_rules_gbs(n: int = 61_100_840, reps: int = 3) -> dict:
    """The reference's numpy update rules (updates.py:85-140, via the oracle's
    restatement) on n fp32 parameters: algorithmic GB/s (worker 16 B, center
    from sum 12 B, MEASGD 24 B per parameter), best of reps."""
    from oracle import esgd_oracle as O

    rng = np.random.default_rng(0)
    w, g, c, s, v = (rng.standard_normal(n, dtype=np.float32) for _ in range(5))
    out = {}
    for name, fn, bpp in (("easgd_worker_step", lambda: O.easgd_worker_step(w, g, c, 0.01, 0.1), 16),
                          ("easgd_center_step_from_sum", lambda: O.easgd_center_step_from_sum(c, s, 1, 0.01, 0.1), 12),
                          ("measgd_worker_step", lambda: O.measgd_worker_step(w, v, g, c, 0.01, 0.9, 0.1), 24)):
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t = time.perf_counter() - t0
            best = t if best is None else min(best, t)
        out[name] = round(bpp * n / best / 1e9, 2)
    out["params"] = n
    out["unit"] = "GB/s (algorithmic bytes)"
    return out


def threaded_round(args, train, workers: int) -> dict:
    """One round of the reference's threaded engine (trainers/synchronous.py:
    156-219, restated as oracle.run_sync_threaded): P OS threads, 3 barriers."""
    from oracle import esgd_oracle as O

    layers = {"lenet": O.LENET, "cifar-quick": O.CIFAR_QUICK, "alexnet": O.alexnet_layers(1000)}[args.model]
    wl = WORKLOADS[args.model]
    b = args.batch or wl["b"]
    prob = O.NetProblem(*layers, train.samples, train.labels, seed=0, dtype=np.float32)
    O.run_sync_threaded(prob, workers, 1, b, wl["eta"], wl["rho"], seed=3)  # warm-up
    t0 = time.perf_counter()
    O.run_sync_threaded(prob, workers, 1, b, wl["eta"], wl["rho"], seed=3)
    t = time.perf_counter() - t0
    return {"value": round(workers * b / t, 2), "unit": "samples/s", "workers": workers,
            "sample": f"1 round, P={workers} threads, b={b}/worker"}


def cpu_baseline(args, spec, train, budget_s: float = 12.0):
    cpu = CpuRound(args, train)
    rounds, elapsed = cpu.sample(budget_s)
    out = {"value": round(rounds * cpu.b / elapsed, 2), "unit": "samples/s", "cores": cpu.cores,
           "kind": "port", "sample": cpu.describe(rounds), "host": host_info()}
    try:
        out["update_rules"] = update_rules_gbs(spec.parameter_count())
        out["threaded_engine"] = threaded_round(args, train, 2)
    except Exception as exc:  # extras only; never fail the bench over them
        out["extras_error"] = repr(exc)
    return out


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (the oracle port — the
    reference is pure Python/numpy and is not installed on the GPU box) on the
    host's cores, on the native arm's config: P = N workers (one per GPU),
    b per worker, full rounds. Rank 0 alone runs it. Each step is one full
    round; when K rounds would exceed ~150 s, fewer are timed (stated in
    the sample) so the run ends within a few minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1708_02983_b200 import network

    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    spec = network.MODELS[args.model](seed=0)
    train, _ = make_data(args.model, spec)
    cpu = CpuRound(args, train, workers=world)  # includes one warm-up round
    t_round = None
    tot_r, tot_t = 0, 0.0
    min_step = 0.25  # small models: several rounds per step so timer noise stays small
    for i in range(args.steps):
        r, t = cpu.sample(min_step)
        tot_r, tot_t = tot_r + r, tot_t + t
        t_round = tot_t / tot_r
        if i >= 2 and tot_t + t_round * (args.steps - i - 1) > 150.0:
            break
    steps_done = i + 1
    value = round(tot_r * cpu.P * cpu.b / tot_t, 2)
    out = {"impl": "reference", "metric": METRIC,
           "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(1000.0 * tot_t / steps_done, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "config": workload_config(args, cpu.b, world),
           "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cpu.cores, "kind": "port",
                            "sample": cpu.describe(tot_r) + f"; {steps_done} of {args.steps} steps timed "
                            "(1 warm-up round)", "host": host_info()},
           "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_async(args):
    """--schedule async-measgd|async-easgd|hogwild-easgd: configs[2] / [3]
     — the asynchronous schedules in ONE process over
    the visible GPUs (workers spread round-robin, master on GPU 0: the device
    master kernel for the elastic async methods). A step = one exchange
    (one worker cycle); value = exchanges x batch / device time. Under torchrun
    only rank 0 runs."""
    import torch

    from paper_1708_02983_b200 import HyperParams, make_config, network, run_trainer
    from paper_1708_02983_b200.trainers import NetworkProblem

    if int(os.environ.get("RANK", "0")) != 0:
        return
    model = args.model if args.model != "alexnet" else ("cifar-quick" if "async" in args.schedule else "lenet")
    wl = WORKLOADS[model]
    spec = network.MODELS[model](seed=0)
    train, _ = make_data(model, spec)
    prob = NetworkProblem(spec, train)
    b = args.batch or wl["b"]
    workers = args.workers or (8 if "async" in args.schedule else 16)
    mom = "measgd" in args.schedule
    hy = HyperParams(eta=wl["eta"] * (0.1 if mom else 1.0), rho=wl["rho"], mu=0.9)
    iters = max(args.steps, 1) * workers
    run_trainer(make_config(args.schedule, workers=workers, iterations=max(args.warmup, 3) * workers,
                            batch_size=b, hyper=hy, seed=3), prob)  # warm-up: allocation, graphs, kernels
    rec = run_trainer(make_config(args.schedule, workers=workers, iterations=iters, batch_size=b, hyper=hy,
                                  seed=3), prob)
    gpus = torch.cuda.device_count()
    out = {"metric": f"{args.schedule} samples/s ({workers} workers, {model})", "value": round(iters * b / rec.total_seconds, 1),
           "unit": "samples/s", "n_gpus": gpus, "steps": iters, "warmup": max(args.warmup, 3) * workers,
           "ms_per_step": round(rec.total_seconds / iters * 1e3, 5), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (gen_synthetic blobs, HBM-resident)",
           "config": {"workload": f"configs[{2 if 'async' in args.schedule else 3}]: {args.schedule}, {model}, "
                                  f"{workers} workers over {gpus} GPU(s), b={b}", "model": model,
                      "workers": workers, "per_worker_batch": b},
           "exchanges_per_s": round(iters / rec.total_seconds, 1),
           "final_train_loss": rec.train_loss[-1] if rec.train_loss else None,
           "engine": rec.engine_info}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--model", default="alexnet", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--schedule", default="sync-easgd3",
                    choices=["sync-easgd3", "async-measgd", "async-easgd", "hogwild-easgd"])
    ap.add_argument("--workers", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.schedule != "sync-easgd3" and args.impl == "native":
        run_async(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
