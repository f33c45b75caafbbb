"""Benchmark: simulation steps/s (and ADMM iterations/s) of the B200 hot path.

`python bench.py --gpus N --steps K --warmup W [--impl ours|reference]`

A step is one committed frame of the BASELINE.json workload. At N=1 that is
config[1], "1k-body random pile drop, single partition on 1 B200" (scene
`pile-1k`: 1,000 boxes, 25 x 40 lattice, run_reference semantics). Inputs are
synthetic (the deterministic lattice + splitmix64 jitter of scene.py) and
resident in HBM during the timed `value`; `e2e` times the same steps through
the public C ABI with the state copied host->device and back every step.

Untimed set-up drops the lattice for --settle frames so every timed step is
a contact-rich pile frame. The L2 is flushed (256 MiB write) between timed
steps, outside the per-step CUDA events. Rank 0 prints ONE JSON line.
Under torchrun (N > 1) the run is partition-per-GPU consensus ADMM with weak
scaling: the scene is N pile-1k slabs side by side (N x 1,000 bodies, N
partitions separated by interface planes), rank r owns partition r, split
bodies are exchanged with the neighbouring ranks over NCCL (dist.TorchComm).
`value` counts pile-1k-equivalent steps: N x committed frames/s, so N=1 and
N>1 share a unit (one partition of 1,000 bodies stepped once). At N=1 the
single partition is the run_reference path (1-worker ADMM is bitwise the
same algorithm, tests/test_gpu_admm.py). DABD_BENCH_SHARE_GPU=1 maps every
rank to cuda:0 over gloo (a functional check of the N>1 path on one GPU; its
timings are not scaling numbers).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_N1 = "pile-1k"


def _ncu_traffic(kernel: str = "k_pcg_cluster"):
    """DRAM bytes per launch (read + write) of `kernel` from the newest committed
    `ncu --set full` summary under profiles/ (tools/ncu_summary.py output)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{kernel}_ncu_full.txt")))
    if not files:
        return None, None
    units = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    seen = 0
    with open(files[-1]) as f:
        for line in f:
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if line.startswith(key + " ="):
                    parts = line.split("=")[1].split()
                    total += float(parts[0].replace(",", "")) * units.get(parts[1] if len(parts) > 1 else "byte", 1.0)
                    seen += 1
    return (total if seen == 2 else None), os.path.relpath(files[-1], ROOT)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int) -> None:
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
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
                "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    return O


def _settled_state(O, sd, settle: int):
    """The oracle's own drop of the lattice (used by the CPU arm only)."""
    o = O.Scene(sd)
    if settle > 0:
        r = o.run(settle, workers=0)
        return o, r["q"][-1], r["qdot"][-1]
    return o, o.q0.copy(), o.qdot0.copy()


def run_reference_arm(args) -> None:
    """CPU reference arm: the oracle port of proj/src/sim.cpp:186-249 (the
    reference itself cannot be built here: Eigen3 is absent),
    single-threaded like the reference worker. Each step is one
    frame of the same settled pile, continued from the previous step."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    O = _oracle()
    from paper_2605_15875_b200.scene import make_scenario

    sd = make_scenario(args.config)
    o, q, qd = _settled_state(O, sd, args.settle)
    times, admm = [], 0
    for i in range(args.warmup + args.steps):
        o.set_state(q, qd)
        t0 = time.perf_counter()
        r = o.run(1, workers=0)
        dt = time.perf_counter() - t0
        q, qd = r["q"][0], r["qdot"][0]
        if i >= args.warmup:
            times.append(dt)
            admm += int(r["admm"][0])
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": "sim_steps_per_sec", "value": value, "unit": "steps/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "bodies": o.n, "partitions": 1,
                   "semantics": "run_reference (sim.cpp:186-249)",
                   "start": f"lattice dropped for {args.settle} untimed frames (contact-rich pile)"},
        "admm_iters_per_sec": admm / total,
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": 1, "kind": "port",
                         "sample": f"{args.steps} consecutive frames of {args.config} after "
                                   f"{args.warmup} warm-up frames, oracle/ C++ restatement"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if ws > 1:
        line["config"]["note"] = (
            f"N={ws}: the reference arm times the single-domain pile-1k step (one pile-1k-equivalent "
            f"unit, as the GPU arm counts them); the CPU consensus run of pile-1k-x{ws} needs ~150 ADMM "
            "iterations of 1,000-body Newton solves per frame and partition, minutes per frame")
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(sd, q, qd, budget_s: float = 20.0, max_frames: int = 3):
    """Oracle (port) steps/s on the host, continuing from the GPU's warm state."""
    O = _oracle()
    o = O.Scene(sd)
    frames = 0
    t0 = time.perf_counter()
    while True:
        o.set_state(q, qd)
        r = o.run(1, workers=0)
        q, qd = r["q"][0], r["qdot"][0]
        frames += 1
        if time.perf_counter() - t0 > budget_s or frames >= max_frames:
            break
    dt = time.perf_counter() - t0
    return {"value": frames / dt, "unit": "steps/s", "cores": 1, "kind": "port",
            "sample": f"{frames} frame(s) of the same settled pile, continued from the GPU run's "
                      f"warm state, single-threaded oracle/ restatement ({dt:.1f} s)"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CONFIG_N1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle", type=int, default=40,
                    help="untimed frames that turn the lattice into a pile before warm-up")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch

    ws, rank, local = _dist()
    share = os.environ.get("DABD_BENCH_SHARE_GPU", "0") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_15875_b200 import _lib as L
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario, pile_slabs

    lib = L.load()
    workers = 0 if ws == 1 else ws
    sd = make_scenario(args.config) if ws == 1 else pile_slabs(ws)
    scene = api.Scene(sd)
    comm = None
    if ws > 1:
        from paper_2605_15875_b200.dist import TorchComm

        comm = TorchComm(workers, device=local)
    def make_ctx():
        c = api.Context(scene, device=local, num_workers=workers,
                        part_begin=comm.part_begin if comm else 0,
                        part_end=comm.part_end if comm else None)
        if comm:
            c.set_comm(comm)
        return c

    ctx = make_ctx()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    if args.settle > 0:
        ctx.run_frames(args.settle)
    for _ in range(args.warmup):
        ctx.run_frames(1)
    torch.cuda.synchronize()
    q_warm, qd_warm = ctx.state()

    def perf(reset):
        ns, n, b, it = C.c_double(), C.c_longlong(), C.c_double(), C.c_longlong()
        L.check(lib.dabd_gpu_ctx_pcg_perf(ctx.h, int(reset), C.byref(ns), C.byref(n), C.byref(b),
                                          C.byref(it)))
        return ns.value, n.value, b.value, it.value

    perf(True)
    n0 = C.c_longlong()
    lib.dabd_gpu_launch_count(C.byref(n0))
    step_ms, stats = [], []
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = ctx.run_frames(1)[0]
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            stats.append(st)
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    n1 = C.c_longlong()
    lib.dabd_gpu_launch_count(C.byref(n1))
    pcg_ns, pcg_launches, pcg_bytes, pcg_iters = perf(True)
    total_ms = sum(step_ms)
    if ws > 1:
        t = torch.tensor([total_ms], device="cpu" if share else "cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = ws * args.steps / (total_ms / 1e3)
    admm = sum(s["admm_iterations"] for s in stats)

    # e2e through the public API with pinned host buffers every step
    q_h = torch.from_numpy(q_warm.copy()).pin_memory()
    qd_h = torch.from_numpy(qd_warm.copy()).pin_memory()
    ctx2 = make_ctx()
    ctx2.set_stream(stream.cuda_stream)
    qp = C.cast(q_h.data_ptr(), C.POINTER(C.c_double))
    qdp = C.cast(qd_h.data_ptr(), C.POINTER(C.c_double))
    st_arr = (L.FrameStats * 1)()
    L.check(lib.dabd_gpu_set_state(ctx2.h, qp, qdp))
    L.check(lib.dabd_gpu_run_frames(ctx2.h, 1, st_arr))  # graph capture outside the timing
    q_h.copy_(torch.from_numpy(q_warm))
    qd_h.copy_(torch.from_numpy(qd_warm))
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        L.check(lib.dabd_gpu_set_state(ctx2.h, qp, qdp))
        L.check(lib.dabd_gpu_run_frames(ctx2.h, 1, st_arr))
        L.check(lib.dabd_gpu_get_state(ctx2.h, qp, qdp))
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64,
                         device="cpu" if share else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    nbytes = 2 * 6 * 8 * scene.n

    hbm, peak_kind = _peaks()
    roof = None
    if pcg_launches > 0 and pcg_ns > 0:
        dur = pcg_ns / pcg_launches / 1e9
        achieved = (pcg_bytes / pcg_launches) / dur / 1e9
        traffic, traffic_src = _ncu_traffic()
        roof = {"bound": "hbm", "kernel": "k_pcg_cluster", "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "traffic_source": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, {traffic_src}"
                                  if traffic is not None else None,
                "peak_kind": peak_kind, "launches": pcg_launches,
                "avg_launch_us": 1e6 * dur, "iterations_per_launch": pcg_iters / pcg_launches,
                "share_of_step": (pcg_ns / 1e6) / total_ms,
                "algorithmic_bytes_per_launch": pcg_bytes / pcg_launches,
                "timing": "device %globaltimer per launch inside the captured graph "
                          "(CUDA events cannot bracket a conditional-graph node)",
                "bytes_model": "SURVEY.md 8(d): I_pcg * [288 (N_b + 2 E_o) + 504 N_b]"}
    line = {
        "metric": "sim_steps_per_sec", "value": value, "unit": "steps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.config if ws == 1 else sd.name, "bodies": scene.n,
                   "partitions": max(workers, 1),
                   "semantics": "run_reference (sim.cpp:186-249)" if ws == 1 else
                                "consensus ADMM, one partition per GPU (runtime.cpp:110-694)",
                   "unit_of_work": "one 1,000-body pile partition stepped one frame",
                   "start": f"lattice dropped for {args.settle} untimed frames (contact-rich pile)",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "parallelism": "single" if ws == 1 else
                                  f"partition-per-GPU x{ws} ({'gloo, shared GPU' if share else 'NCCL'})"},
        "admm_iters_per_sec": admm * ws / (total_ms / 1e3),
        "newton_iters_per_step": sum(s["newton_iterations"] for s in stats) / len(stats),
        "pcg_iters_per_step": sum(s["pcg_iterations"] for s in stats) / len(stats),
        "max_contacts": max(s["max_contacts"] for s in stats),
        "e2e": {"value": ws * args.steps / (e2e_ms / 1e3), "unit": "steps/s",
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
        "gpu_launches": int(n1.value - n0.value),
        "roofline": roof,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(sd, q_warm, qd_warm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
