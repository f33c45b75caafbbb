"""Benchmark: simulation steps/s (and ADMM iterations/s) of the B200 hot path.

`python bench.py --gpus N --steps K --warmup W [--impl ours|reference]`

A step is one committed frame of the BASELINE.json workload. At N=1 that is
config[1], "1k-body random pile drop, single partition on 1 B200" (scene
`pile-1k`: 1,000 boxes, 25 x 40 lattice, run_reference semantics). Inputs are
synthetic (the deterministic lattice + splitmix64 jitter of scene.py) and
resident in HBM during the timed `value`; `e2e` times the same steps through
the public C ABI with the state copied host->device and back every step.

Both arms start from the same contact-rich pile: the CPU oracle's own
40-frame drop of the lattice (tests/golden/pile-1k_settled40.npz, made by
tools/make_bench_fixture.py), tiled into the N slabs of pile_slabs(N) when
N > 1. The L2 is flushed (256 MiB write) between timed steps, outside the
per-step CUDA events, in the device-timed loop and in the e2e loop alike.
Rank 0 prints ONE JSON line.
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

`--mode strong` (a second, opt-in mode for the C3/C5 story): the same
pour-10k scene with 8 consensus partitions at every N, rank r owning
partitions [8r/N, 8(r+1)/N); N=1 runs all 8 partitions batched on one GPU
(the device-side ADMM frame), so N=1,2,4,8 run the same algorithm and
`value` is whole-scene frames/s ("scaling": "strong"). Both modes start
from a state the GPU reached itself in strong mode (30 single-domain frames
of the pour, then 2 consensus frames), and the N=1 strong line also reports
the undivided single-domain frame rate of the same state. The reference arm
has no strong mode (an 8-partition pour frame costs the CPU oracle tens of
minutes) and says so.
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
STRONG_SCENE, STRONG_PARTS, STRONG_SETTLE, STRONG_SPLIT = "pour-10k", 8, 30, 2


def _ncu_traffic(kernel: str = "k_pcg_cluster"):
    """DRAM bytes per launch (read + write) of `kernel` from the newest committed
    `ncu --set full` summary under profiles/ (tools/ncu_summary.py output)."""
    import glob

    def tag_key(path):  # r01 < r01b < r02a < r02z < r02aa < r02bk (spreadsheet-column order)
        tag = os.path.basename(path).split("_")[0]
        rnd, suf = tag[:3], tag[3:]
        return (rnd, len(suf), suf)

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{kernel}_ncu_full.txt")), key=tag_key)
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


FIXTURE = os.path.join(ROOT, "tests", "golden", "pile-1k_settled40.npz")


def start_state(sd, ws: int):
    """The bench's start state: the oracle-settled pile-1k (FIXTURE); for
    N > 1 slab k of pile_slabs(N) holds a copy of it shifted by the slab's
    centre (slabs are 5.2 wide, the pile-1k container too). Body 0 (the
    container) stays where the scene puts it."""
    import numpy as np

    z = np.load(FIXTURE)
    q1, qd1 = z["q"], z["qdot"]
    if ws == 1:
        return q1.copy(), qd1.copy()
    per = q1.shape[0] - 1
    width = 5.2 * ws
    q = np.zeros((1 + ws * per, 6))
    qd = np.zeros_like(q)
    q[0] = q1[0]
    for k in range(ws):
        sl = slice(1 + k * per, 1 + (k + 1) * per)
        q[sl] = q1[1:]
        q[sl, 0] += -width / 2.0 + 5.2 * k + 2.6
        qd[sl] = qd1[1:]
    return q, qd


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def bench_config(ws: int, share: bool = False):
    """The `config` both arms print (identical dicts for the same N)."""
    from paper_2605_15875_b200.scene import make_scenario, pile_slabs

    sd = make_scenario(CONFIG_N1) if ws == 1 else pile_slabs(ws)
    return sd, {
        "workload": CONFIG_N1 if ws == 1 else sd.name, "bodies": len(sd.bodies),
        "partitions": ws,
        "semantics": "run_reference (sim.cpp:186-249)" if ws == 1 else
                     "consensus ADMM, one partition per GPU (runtime.cpp:110-694)",
        "unit_of_work": "one 1,000-body pile partition stepped one frame",
        "start": "pile-1k settled 40 frames by the CPU oracle (tests/golden/pile-1k_settled40.npz)"
                 + ("" if ws == 1 else f", tiled into {ws} slabs"),
        "l2": "flushed (256 MiB write) between timed steps (GPU arm)",
        "parallelism": "single" if ws == 1 else
                       f"partition-per-GPU x{ws} ({'gloo, shared GPU' if share else 'NCCL'})",
    }


def strong_config(ws: int, share: bool = False):
    """Strong-scaling workload: pour-10k, 8 partitions over ws GPUs."""
    from paper_2605_15875_b200.scene import make_scenario

    sd = make_scenario(STRONG_SCENE)
    return sd, {
        "workload": STRONG_SCENE, "bodies": len(sd.bodies), "partitions": STRONG_PARTS,
        "semantics": "consensus ADMM (runtime.cpp:110-694), the same 8 partitions at every N",
        "unit_of_work": "one 10,000-body frame of the whole scene",
        "start": f"pour-10k: {STRONG_SETTLE} single-domain + {STRONG_SPLIT} 8-partition frames on the GPU",
        "l2": "flushed (256 MiB write) between timed steps (GPU arm)",
        "parallelism": f"{STRONG_PARTS // ws} partition(s) per GPU x{ws}"
                       + (" (gloo, shared GPU)" if share else (" (NCCL)" if ws > 1 else " (batched)")),
    }


def strong_start_state(api, sd):
    """The strong mode's start state: every rank computes it itself (the
    frames are deterministic, so all ranks hold the same bits)."""
    ctx = api.Context(api.Scene(sd))
    ctx.run_frames(STRONG_SETTLE)
    q, qd = ctx.state()
    c8 = api.Context(api.Scene(sd), num_workers=STRONG_PARTS)
    c8.set_state(q, qd)
    c8.run_frames(STRONG_SPLIT)
    return c8.state()


def run_reference_arm(args) -> None:
    """CPU reference arm: the oracle port of proj/src/sim.cpp:186-249 (N=1,
    single-threaded like the reference worker) or of the
    consensus runtime (N > 1: runtime.cpp:110-694 with one std::thread per
    partition, sim.cpp:281-322) on the same scene and start state as the GPU
    arm. The reference itself cannot be built here (Eigen3 is absent,
    SURVEY.md 8c). N=1: each step is one frame, continued from the previous
    one, after the same warm-up frames. N > 1: a consensus frame of N
    1,000-body partitions costs the CPU about a minute, so the sample is the
    frames that complete within --ref-budget seconds (at least one, no
    warm-up)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    if args.mode == "strong":
        print(json.dumps({"impl": "reference", "unavailable": "strong mode: one 8-partition pour-10k frame "
                          "costs the CPU oracle tens of minutes; the reference arm runs the default mode"}))
        return
    O = _oracle()
    sd, config = bench_config(ws)
    o = O.Scene(sd)
    q, qd = start_state(sd, ws)
    times, admm = [], 0
    if ws == 1:
        for i in range(args.warmup + args.steps):
            o.set_state(q, qd)
            t0 = time.perf_counter()
            r = o.run(1, workers=0)
            dt = time.perf_counter() - t0
            q, qd = r["q"][0], r["qdot"][0]
            if i >= args.warmup:
                times.append(dt)
                admm += int(r["admm"][0])
        sample = (f"{args.steps} consecutive frames of {config['workload']} after {args.warmup} "
                  "warm-up frames, oracle/ C++ restatement, one thread")
    else:
        t_start = time.perf_counter()
        while not times or (len(times) < args.steps and time.perf_counter() - t_start < args.ref_budget):
            o.set_state(q, qd)
            t0 = time.perf_counter()
            r = o.run(1, workers=ws)
            times.append(time.perf_counter() - t0)
            q, qd = r["q"][0], r["qdot"][0]
            admm += int(r["admm"][0])
        sample = (f"{len(times)} consecutive consensus frame(s) of {config['workload']} from the start "
                  f"state (bounded by {args.ref_budget:.0f} s), oracle/ C++ restatement, "
                  f"{ws} partition threads")
    total = sum(times)
    value = len(times) / total
    line = {
        "impl": "reference", "metric": "sim_steps_per_sec", "value": ws * value, "unit": "steps/s",
        "n_gpus": ws, "steps": len(times), "warmup": args.warmup if ws == 1 else 0,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config,
        "admm_iters_per_sec": ws * admm / total,
        "cpu_baseline": {"value": ws * value, "unit": "steps/s", "cores": ws, "kind": "port",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": ws * value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(sd, q, qd, budget_s: float = 20.0, max_frames: int = 6):
    """Oracle (port) steps/s on the host, single-threaded like the reference's
    run_reference, continuing from the GPU's warm state (~20 s sample)."""
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
                      f"warm state, single-threaded oracle/ restatement ({dt:.1f} s)",
            "host": host_info()}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle", type=int, default=0,
                    help="extra untimed GPU frames after loading the start state")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="reference arm at N > 1: wall-clock bound of the CPU sample (s)")
    ap.add_argument("--mode", default="weak", choices=["weak", "strong"],
                    help="weak: pile-1k slabs (default); strong: pour-10k, 8 partitions at every N")
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
    lib = L.load()
    strong = args.mode == "strong"
    if strong:
        workers = STRONG_PARTS
        sd, config = strong_config(ws, share)
    else:
        workers = 0 if ws == 1 else ws
        sd, config = bench_config(ws, share)
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

    q0, qd0 = strong_start_state(api, sd) if strong else start_state(sd, ws)
    ctx.set_state(q0, qd0)
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
    value = (1 if strong else ws) * args.steps / (total_ms / 1e3)
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
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.check(lib.dabd_gpu_set_state(ctx2.h, qp, qdp))
        L.check(lib.dabd_gpu_run_frames(ctx2.h, 1, st_arr))
        L.check(lib.dabd_gpu_get_state(ctx2.h, qp, qdp))
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
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
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config,
        "admm_iters_per_sec": admm * (1 if strong else ws) / (total_ms / 1e3),
        "newton_iters_per_step": sum(s["newton_iterations"] for s in stats) / len(stats),
        "pcg_iters_per_step": sum(s["pcg_iterations"] for s in stats) / len(stats),
        "max_contacts": max(s["max_contacts"] for s in stats),
        "e2e": {"value": (1 if strong else ws) * args.steps / (e2e_ms / 1e3), "unit": "steps/s",
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
        "gpu_launches": int(n1.value - n0.value),
        "roofline": roof,
        "clocks": clk.summary(),
    }
    if strong:
        line["t_frame_split_ms"] = {  # host wall split of the timed frames (FrameStats)
            "frame": 1e3 * sum(s["t_frame"] for s in stats) / len(stats),
            "solve": 1e3 * sum(s["t_solve"] for s in stats) / len(stats),
            "sync": 1e3 * sum(s["t_sync"] for s in stats) / len(stats)}
        if ws == 1:  # the undivided single-domain frame rate of the same start state
            c1 = api.Context(scene, device=local)
            c1.set_stream(stream.cuda_stream)
            c1.set_state(q_warm, qd_warm)
            c1.run_frames(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c1.run_frames(args.steps)
            e1.record(stream)
            e1.synchronize()
            line["single_domain_steps_per_s"] = args.steps / (e0.elapsed_time(e1) / 1e3)
        line["cpu_baseline"] = None  # see the reference arm
    elif rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(sd, q_warm, qd_warm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
