#!/usr/bin/env python3
"""Benchmark of the kcg hot path (BASELINE.json metric: predicted
(kernel,size) points/sec; % HBM roofline; fit rows/sec).

Headline workload (config 4, materialised mode): the 6 matmul variants of
the bundled suite (matmul_tiled_g{12,14,16}, matmul_naive_g16x{12,14,16})
at every size (n,m,l) = 336*(u,v,w), u,v,w in [1,551] -- 551^3 =
1.673e8 sizes x 6 variants = 1.004e9 (variant, size) points. A step is one
exact evaluate_properties + predict of every point: ONE launch of the
one-pass multi-program kernel (kcg_eval_predict_multi) reads each size's SoA
int64 bindings once (24 B) and writes all six fp64 predictions (48 B).
Inputs (4.0 GB) and outputs (8.0 GB) exceed L2, so no flush is needed.
Sizes shard contiguously across ranks (strong scaling, no collective on the
data path). The default line also carries the fused argmin (config 4),
config 2 (1e6 points of the four test kernels) and the config-3 Gram.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

VARIANTS = ["matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
            "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16"]
SIDE = 551
UNIT = 336
METRIC = "predicted (kernel,size) points/sec"
PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"


def peaks():
    try:
        d = json.loads(PEAKS_PATH.read_text())
        return d["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


CPU_SAMPLE_SIZES = 1_000_000  # sizes per CPU sample (x 6 variants): ~5 s on 16 threads


def cpu_reference(threads: int, n_sizes: int, offset: int = 0):
    exe = ROOT / "oracle" / "_ref" / "kcref_bench"
    if not exe.exists():
        return None
    out = subprocess.run([str(exe), "autotune", str(threads), str(n_sizes), str(offset)],
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out)


def host_info(threads: int) -> dict:
    model = ""
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_used": threads,
            "build": "oracle/_ref: the reference's own core sources compiled in place, g++ -std=c++20 -O3 "
                     "-DNDEBUG -ffp-contract=off (CMake Release, the reference default), against the repo's "
                     "shims: bigint (cpp_int/cpp_rational) instead of Boost.Multiprecision, COD instead of Eigen"}


def cpu_reference_line(threads: int, offset: int = 0) -> dict | None:
    """The one CPU routine behind both the in-line cpu_baseline and the
    --impl reference arm: the reference's evaluate_properties + predict per
    (variant, size) point (bench.cpp:47-56 pattern) over CPU_SAMPLE_SIZES
    sizes of the headline lattice, std::thread fan-out over `threads`."""
    r = cpu_reference(threads, CPU_SAMPLE_SIZES, offset)
    if r is None:
        return None
    return {"value": r["points_per_s"], "unit": "points/s", "cores": threads, "kind": "reference",
            "seconds": r["seconds"], "points": r["points"],
            "sample": f"{r['points'] // len(VARIANTS)} sizes x {len(VARIANTS)} variants of the headline lattice "
                      f"(from size {offset}), evaluate_properties+predict per point",
            "host": host_info(threads)}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path (oracle/_ref: reference
    sources + shim bigint/COD), all host threads, a fixed sample of
    CPU_SAMPLE_SIZES sizes per step (warm-up steps: a tenth of it)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if cpu_reference(threads, 1000) is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/kcref_bench not built"}))
        return
    for w in range(args.warmup):
        cpu_reference(threads, CPU_SAMPLE_SIZES // 10, offset=w * 7919)
    times, pts, last = [], 0, None
    for s in range(args.steps):
        last = cpu_reference_line(threads)  # the in-line cpu_baseline's sample, every step
        times.append(last["seconds"])
        pts = last["points"]
    sec = sum(times) / len(times)
    value = pts / sec
    cb = dict(last)
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bigint", "data": "synthetic",
        "config": {"workload": "config4 autotune sample: 6 matmul variants x sizes 336*(u,v,w)",
                   "points_per_step": pts, "threads": threads},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--side", type=int, default=SIDE, help="u,v,w in [1, side]")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fit", action="store_true", help="skip the sharded fit (config 5)")
    ap.add_argument("--fit-rows", type=int, default=10**9, help="fit rows per rank")
    ap.add_argument("--extras", action="store_true", help="also time config 5 on one GPU, the grid "
                    "descriptor path and the enumeration oracle")
    ap.add_argument("--no-configs", action="store_true", help="skip argmin / config 2 / config 3 in the line")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1604_04997_b200 as kc

    # one process per GPU; KCG_DIST_BACKEND=gloo lets several ranks share
    # one device for a functional dry run of the multi-rank path
    backend = os.environ.get("KCG_DIST_BACKEND", "nccl")
    if world > 1 and backend == "nccl":  # init lines (ring / NVLS / P2P) for the driver's rank check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)

    progs = [kc.load_program(v) for v in VARIANTS]
    sim_alpha = _simdev_alpha(kc)
    w = kc.ModelWeights(device="simdev-v1", alpha=sim_alpha, covered=[a != 0 for a in sim_alpha])

    total = args.side ** 3
    r0, r1 = total * rank // world, total * (rank + 1) // world
    n = r1 - r0
    idx = torch.arange(r0, r1, dtype=torch.int64, device=dev)
    s2 = args.side * args.side
    cols = {"n": (idx // s2 + 1) * UNIT, "m": ((idx // args.side) % args.side + 1) * UNIT,
            "l": (idx % args.side + 1) * UNIT}
    del idx
    cols = {k: v.contiguous() for k, v in cols.items()}
    # rows padded to a 16-byte multiple so every variant's output row is
    # aligned (the kernels also accept unaligned rows)
    ld = (n + 1) // 2 * 2
    preds = torch.empty((len(VARIANTS), ld), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    handles = (ctypes.c_void_p * len(progs))(*[p.handle.value for p in progs])
    carr = _colarr(progs[0], cols)
    alpha_arr = w.alpha_array()

    def step(ev=None):
        # one launch: every variant's evaluate + predict, bindings read once
        if ev is not None:
            ev[0].record(stream)
        kc.api.check(kc.api.lib().kcg_eval_predict_multi(handles, len(progs), carr, n, alpha_arr, preds.data_ptr(),
                                                         ld, None, 0, stream.cuda_stream))
        if ev is not None:
            ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = kc.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        start.record(stream)
        for s in range(args.steps):
            step(evs[s])
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = kc.launch_count() - launches0
    elapsed = start.elapsed_time(end) / 1e3
    kern_ms = [e[0].elapsed_time(e[1]) for e in evs]
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    points = total * len(VARIANTS) * args.steps
    value = points / elapsed

    # sanity: a few points against the oracle (checker only)
    checked = _spot_check(kc, progs, cols, preds[:, :n], sim_alpha, r0, args.side) if rank == 0 else 0

    # the same step as six kcg_eval_predict launches (one per variant, the
    # bindings re-read six times): context for the one-pass kernel
    six = _timed(torch, lambda: [kc.api.check(kc.api.lib().kcg_eval_predict(
        p.handle, _colarr(p, cols), n, alpha_arr, preds[v].data_ptr(), None, None, None, 0, stream.cuda_stream))
        for v, p in enumerate(progs)], reps=3, warm=1)
    step()
    torch.cuda.synchronize()

    hbm, peak_kind = peaks()
    V = len(VARIANTS)
    traffic = None
    try:  # ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/)
        tr = json.loads((ROOT / "profiles" / "r02_traffic.json").read_text())
        traffic = tr["traffic_bytes_per_launch"] * n / tr["sizes_per_launch"]
    except Exception:
        pass
    avg_launch = statistics.mean(kern_ms) / 1e3
    bytes_per_size = 8 * 3 + 8 * V  # 8 P in (P = 3), 8 V out
    bytes_per_launch = float(bytes_per_size) * n
    achieved = bytes_per_launch / avg_launch / 1e9
    mix = kc.measure_stream(3, V, 1 << 27) / 1e9
    pipes = _pipe_peaks(kc)

    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": "config4 materialised evaluate+predict: 6 matmul variants x "
                               f"{total} sizes (n,m,l)=336*(u,v,w), u,v,w<= {args.side}, one multi-program "
                               "launch per step",
                   "points_per_step": total * V, "bytes_per_size": bytes_per_size,
                   "bytes_per_point": bytes_per_size / V,
                   "l2": "inputs 4.0 GB + outputs 8.0 GB per step exceed the 126 MB L2 (no flush)",
                   "parallelism": f"dp{world} (contiguous size shards)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes": "8 P + 8 V per size (P = 3 binding columns read once, V = 6 "
                                          "predictions written) = 72 B per size, 12 B per (variant, size) point",
                     "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch * 1e3,
                     "same_mix_stream_gbs": mix, "frac_of_same_mix": achieved / mix,
                     "same_mix_note": "kcg_measure_stream(3, 6): a plain kernel reading 3 int64 and writing 6 "
                                      "fp64 columns (this kernel's 1:2 read:write mix), the best of 16-byte "
                                      "streaming stores and smem-staged cp.async.bulk stores, measured live",
                     "traffic_source": "profiles/r02_traffic.json (ncu dram bytes of the same launch)",
                     "kernel": "kcg_multi_v6_tmab (NVRTC sm_100a: TMA-ring loads, per-warp cp.async.bulk stores)",
                     "per_point_8P_plus_8_GBps": 32.0 * n * V / avg_launch / 1e9,
                     "per_point_note": "SURVEY 8(d)'s per-point figure (8 P + 8 = 32 B per point, bindings "
                                       "counted once per variant) over the same launch time: what six "
                                       "per-variant launches would have to stream"},
        "instruction_roofline": _instr_roofline(_ncu_lane_instr("r02_multi_ncu.txt"),
                                                avg_launch and n * V / avg_launch, pipes,
                                                "profiles/r02_multi_ncu.txt (ncu, same kernel)"),
        "pipe_peaks_lane_ops_per_s": pipes,
        "six_launch_step_ms": six * 1e3,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "spot_checked_points": checked,
    }
    if rank == 0 and not args.no_configs:
        del preds
        line["configs"] = _configs(kc, torch, dev, args, cols, progs, w)
    else:
        del preds
    if not args.no_fit:
        del cols
        line["fit"] = _sharded_fit(kc, torch, dev, world, rank, args.fit_rows)
    if not args.no_e2e:  # every rank streams its own shard over its own PCIe link
        e2e = _e2e(kc, progs, w, args, torch, dev, world, rank)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and not args.no_cpu:
        threads = os.cpu_count() or 1
        cb = cpu_reference_line(threads)
        if cb:
            line["cpu_baseline"] = cb
        if "fit" in line:
            line["fit"]["cpu_reference"] = cpu_reference_fit(200_000, 40)
        line["cpu_optimized"] = cpu_lowered_baseline(kc, progs, sim_alpha, threads, args.side)
    if rank == 0 and args.extras:
        line["extras"] = _extras(kc, torch, dev, args)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))


def cpu_lowered_baseline(kc, progs, alpha, threads, side, sizes=4_000_000):
    """the optimised CPU baseline -- this repo's own lowered
    program for each variant compiled for the host (g++ -O3 -march=native
    -ffp-contract=off, kcg_program_jit_source_kind kind 4), all host
    threads, over the first `sizes` sizes of the headline lattice; its
    predictions are checked bitwise against the GPU's on a sample."""
    import numpy as np
    try:
        from tools.hostbuild import HostEvaluator
        idx = np.arange(sizes, dtype=np.int64)
        cols = {"n": (idx // (side * side) + 1) * UNIT, "m": ((idx // side) % side + 1) * UNIT,
                "l": (idx % side + 1) * UNIT}
        hs = [HostEvaluator(p) for p in progs]
        hs[0].predict(alpha, {k: v[:1000] for k, v in cols.items()}, threads=threads)
        t0 = time.perf_counter()
        preds = [h.predict(alpha, cols, threads=threads)[0] for h in hs]
        sec = time.perf_counter() - t0
        import torch
        w = kc.ModelWeights(device="simdev-v1", alpha=alpha, covered=[a != 0 for a in alpha])
        sl = slice(0, sizes, max(1, sizes // 4096))
        dc = {k: torch.from_numpy(np.ascontiguousarray(v[sl])).cuda() for k, v in cols.items()}
        same = all(np.array_equal(kc.predict(w, p, dc).cpu().numpy().view(np.int64), pr[sl].view(np.int64))
                   for p, pr in zip(progs, preds))
        return {"value": len(progs) * sizes / sec, "unit": "points/s", "cores": threads, "kind": "port",
                "sample": f"{sizes} sizes x {len(progs)} variants of the headline lattice",
                "bitwise_equal_to_gpu_on_sample": bool(same),
                "note": "the repo's lowered integer program compiled for the host (not the reference); "
                        "the reference CPU path is cpu_baseline"}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:300]}


def cpu_reference_fit(rows, cols):
    """The reference's own build_design_matrix + fit_weights (model.cpp:11-93,
    shim COD) on a config-3-shaped synthetic sample, 1 host thread."""
    exe = ROOT / "oracle" / "_ref" / "kcref_bench"
    if not exe.exists():
        return None
    try:
        r = subprocess.run([str(exe), "fit", str(rows), str(cols)], capture_output=True, text=True, timeout=300)
        d = json.loads(r.stdout)
        d["unit"] = "rows/s"
        d["sample"] = f"{rows} synthetic rows x {cols} keys (test_model.cpp pattern), build_design_matrix + fit_weights"
        return d
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:200]}


def _simdev_alpha(kc):
    sys.path.insert(0, str(ROOT / "oracle"))
    keys = kc.schema_keys()
    table = {
        "flop.f32.addsub": 6.81e-13, "flop.f32.mul": 5.68e-13, "flop.f32.pow": 3.91e-13,
        "flop.f32.special": 1.61e-12, "mem.local.load": -1.76e-12,
        "mem.global.load.s32.1/1": 8.27e-12, "mem.global.load.s32.2/2": 9.82e-13,
        "mem.global.load.s32.2/3": 2.89e-11, "mem.global.load.s32.3/3": 9.30e-13,
        "mem.global.load.s32.4/>4": 2.67e-12, "mem.global.store.s32.1/1": 6.52e-12,
        "mem.global.store.s32.4/>4": 3.55e-10, "mem.minls.s32.1/1": -6.63e-12,
        "sync.barrier": 4.26e-11, "launch.groups": 3.75e-09, "launch.const": 1.29e-04}
    return [table.get(k, 0.0) for k in keys]


_COLS_CACHE = {}


def _colarr(p, cols):
    import ctypes
    key = (id(p), tuple(c.data_ptr() for c in cols.values()))
    if key not in _COLS_CACHE:
        _COLS_CACHE[key] = (ctypes.c_void_p * len(p.params))(*[cols[q].data_ptr() for q in p.params])
    return _COLS_CACHE[key]


def _pipe_peaks(kc):
    """Measured lane-op rates of the pipes the exact evaluation runs on
    (csrc/peaks.cu via kcg_measure_pipe_peak): the instruction roofline's
    denominators (MEASURED_PEAKS has no INT32 / FP64 figures)."""
    return {k: kc.measure_pipe_peak(k) for k in ("imad", "lop3", "dfma", "issue")}


def _ncu_lane_instr(name):
    """Lane instructions per point of a kernel, from its committed ncu
    capture (profiles/<name>: SASS instructions executed / points)."""
    try:
        for ln in (ROOT / "profiles" / name).read_text().splitlines():
            if ln.strip().startswith("lane instructions per point:"):
                return float(ln.split(":")[1])
    except OSError:
        pass
    return None


def _instr_roofline(lane_instr, points_per_s, peaks, source):
    if lane_instr is None:
        return None
    achieved = lane_instr * points_per_s
    return {"bound": "issue", "lane_instr_per_point": lane_instr, "achieved_lane_ops_per_s": achieved,
            "peak_lane_ops_per_s": peaks["issue"], "frac": achieved / peaks["issue"],
            "peak_note": "measured: IMAD and LOP3 alternating at full occupancy (kcg_measure_pipe_peak kind 3)",
            "lane_instr_source": source}


def _same_mix_stream(torch, dev, n, stream, reps=10):
    """GB/s of a plain streaming kernel with the headline kernel's traffic
    mix (3 x 8 B read, 8 B written per element), timed like it: the
    bandwidth this read:write ratio gets from HBM on this box."""
    a, b, c = (torch.rand(n, dtype=torch.float64, device=dev) for _ in range(3))
    d = torch.empty_like(a)
    for _ in range(3):
        torch.addcmul(a, b, c, out=d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        e0.record(stream)
        torch.addcmul(a, b, c, out=d)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in ev)
    del a, b, c, d
    return 32.0 * n / (ms / 1e3) / 1e9


def _spot_check(kc, progs, cols, preds, alpha, r0, side):
    sys.path.insert(0, str(ROOT / "oracle"))
    import kc_oracle as ko
    n = preds.shape[1]
    picks = sorted({0, n - 1, n // 2, n // 3, 7 * n // 11})
    done = 0
    for i in picks:
        b = {k: int(v[i]) for k, v in cols.items()}
        for v, p in enumerate(progs):
            op = ko.Program(p.text)
            want = ko.predict(alpha, op.evaluate_properties(b))
            got = float(preds[v, i])
            if got != want:
                raise SystemExit(f"bench spot check failed: {p.name} {b}: {got!r} != {want!r}")
            done += 1
    return done


def _e2e(kc, progs, w, args, torch, dev, world, rank):
    """Same workload through the public C ABI with HOST buffers:
    kcg_eval_predict_host (pinned SoA bindings in, every variant's
    predictions out; the library pipelines H2D / kernels / D2H over its own
    streams), copies inside the timed region. Also reported: the same call
    on pageable buffers (staged through the library's pinned ring)."""
    import ctypes
    total = args.side ** 3
    r0 = total * rank // world
    n = total * (rank + 1) // world - r0
    idx = torch.arange(r0, r0 + n, dtype=torch.int64)
    s2 = args.side * args.side
    host_cols = {"n": ((idx // s2 + 1) * UNIT), "m": (((idx // args.side) % args.side + 1) * UNIT),
                 "l": ((idx % args.side + 1) * UNIT)}
    del idx
    pinned_cols = {k: v.pin_memory() for k, v in host_cols.items()}
    host_pred = torch.empty((len(progs), n), dtype=torch.float64).pin_memory()
    handles = (ctypes.c_void_p * len(progs))(*[p.handle.value for p in progs])
    alpha = w.alpha_array()

    def call(cols, out, flags):
        arr = (ctypes.c_void_p * 3)(*[cols[q].data_ptr() for q in progs[0].params])
        kc.api.check(kc.api.lib().kcg_eval_predict_host(handles, len(progs), arr, n, alpha, out.data_ptr(),
                                                        None, flags))

    import torch.distributed as dist
    call(pinned_cols, host_pred, kc._capi.HOST_PINNED)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    reps = max(1, min(3, args.steps))
    for _ in range(reps):
        call(pinned_cols, host_pred, kc._capi.HOST_PINNED)
    sec = (time.perf_counter() - t0) / reps
    # pageable caller buffers (a std::vector-style caller), one call
    page_pred = torch.empty((len(progs), n), dtype=torch.float64)
    call(host_cols, page_pred, 0)
    t1 = time.perf_counter()
    call(host_cols, page_pred, 0)
    sec_page = time.perf_counter() - t1
    same = bool(torch.equal(page_pred.view(torch.int64), host_pred.view(torch.int64)))
    del page_pred
    if world > 1:  # whole job: all shards, the slowest rank's wall clock
        t = torch.tensor([sec, sec_page], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec, sec_page = (float(x) for x in t.tolist())
    n_local = n
    n = total
    h2d = 3 * 8 * n
    d2h = 8 * n * len(progs)
    # the bound: a plain pinned D2H copy of the same size class on this box
    probe = torch.empty(1 << 27, dtype=torch.float64, device=dev)
    hp = torch.empty(1 << 27, dtype=torch.float64).pin_memory()
    hp.copy_(probe)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(3):
        hp.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    d2h_bw = 3 * 8 * (1 << 27) / (time.perf_counter() - t1)
    chunk = int(os.environ.get("KCG_HOST_CHUNK", 1 << 22))
    nstreams = int(os.environ.get("KCG_HOST_STREAMS", 3))
    return {"value": n * len(progs) / sec, "unit": "points/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": sec * 1e3,
            "pcie_d2h_GBps_measured": d2h_bw / 1e9,
            "d2h_frac_of_measured": 8 * n_local * len(progs) / sec / d2h_bw,  # per rank / per link
            "pageable": {"value": n * len(progs) / sec_page, "ms_per_step": sec_page * 1e3,
                         "bitwise_equal_to_pinned": same},
            "note": "kcg_eval_predict_host (C ABI): pinned host SoA bindings -> 6 variants -> pinned host "
                    f"predictions; library-internal {nstreams} streams, {chunk >> 20}M-size chunks; "
                    "wall clock incl. all copies"}


def _sharded_fit(kc, torch, dev, world, rank, rows):
    """Config 5: every rank forms `rows` design rows (matmul_tiled_g16x16 at
    its own block of sizes, T = noiseless_time on the GPU) and reduces them
    through the fused evaluate -> row -> Gram kernel; G / Xᵀ1 / colmax are
    all-reduced over NCCL, every rank solves the same small system, then
    takes one refinement step whose pass also sums the squared residuals, so
    the objective at the refined weights follows from the all-reduced sums
    and the Gram (api.refined_objective) without a third pass.
    Timed on the device from the Gram launch to the reduced objective, max
    over ranks (host solve included)."""
    import torch.distributed as dist

    from paper_1604_04997_b200.dist import allreduce_gram, allreduce_sum
    prog = kc.load_program("matmul_tiled_g16x16")
    alpha = _simdev_alpha(kc)
    g = torch.arange(0, rows, dtype=torch.int64, device=dev)
    cols = {"n": (16 * (g // 1_000_000 % 1000 + 1 + 1000 * rank)).contiguous(),
            "m": (16 * (g // 1000 % 1000 + 1)).contiguous(),
            "l": (16 * (g % 1000 + 1)).contiguous()}
    del g
    T = kc.noiseless_time(alpha, prog, cols)
    arr = _colarr(prog, cols)
    stream = torch.cuda.current_stream(dev).cuda_stream

    def once():
        st = kc.GramStats.zeros(len(prog.props), dev)
        kc.api.check(kc.api.lib().kcg_gram_fused(prog.handle, arr, T.data_ptr(), rows, st.G.data_ptr(),
                                                 st.xt1.data_ptr(), st.colmax.data_ptr(), None, stream))
        st.n_rows = rows
        allreduce_gram(st)
        a, rank_ = kc.solve_gram(st)

        def full(x):
            out = [0.0] * kc.schema_size()
            for j, k in enumerate(prog.props):
                out[k] = x[j]
            return out
        import ctypes
        # one refinement step: the double-double gradient over the rows the
        # reference would form (fused, never materialised), all-reduced
        # and the sum of squared residuals, which with the Gram gives the
        # objective at the refined weights (api.refined_objective)
        g = torch.zeros(len(prog.props), dtype=torch.float64, device=dev)
        r2 = torch.zeros(1, dtype=torch.float64, device=dev)
        fa = full(a)
        kc.api.check(kc.api.lib().kcg_residual_grad_obj_fused(prog.handle, arr, T.data_ptr(), rows,
                                                              (ctypes.c_double * len(fa))(*fa), g.data_ptr(),
                                                              r2.data_ptr(), stream))
        g = allreduce_sum(g)
        r2 = allreduce_sum(r2)
        a2 = kc.refine_gram(st, a, g)
        obj = kc.refined_objective(st, a, a2, g, r2)
        return rank_, obj, st.n_rows

    once()  # JIT + warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    rk, obj, total_rows = once()
    t1.record()
    torch.cuda.synchronize()
    sec = t0.elapsed_time(t1) / 1e3
    if world > 1:
        t = torch.tensor([sec], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    return {"metric": "fit rows/sec", "rows": total_rows, "value": total_rows / sec, "ms": sec * 1e3,
            "rank": rk, "objective": obj, "scaling": "weak",
            "workload": f"config5: {rows} rows/rank (matmul_tiled_g16x16, T = noiseless_time), fused "
                        "evaluate->row->Gram (monomial basis) + NCCL all-reduce + host min-norm solve + one "
                        "refinement step (fused gradient over the reference's rows with the residual in twice "
                        "the working precision, and its sum of squares, all-reduced); the objective at the "
                        "refined weights from those sums and the Gram (no third pass)",
            # two streaming passes over the rows (Gram, refinement gradient),
            # 8*P + 8 = 32 B per row each
            "bytes_per_row": 64,
            "hbm_frac": 64.0 * rows / sec / 1e9 / peaks()[0],
            "peak_note": "the peak is MEASURED_PEAKS' copy rate (read + write); these passes only read, "
                         "and read streams run above it"}


def _timed(torch, fn, reps=5, warm=2):
    """CUDA-event timing on the current stream: mean seconds per call."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def _fp64_peak(torch, dev):
    """Measured dense fp64 throughput (cuBLAS DGEMM 8192^3), TFLOP/s."""
    n = 8192
    A = torch.rand(n, n, dtype=torch.float64, device=dev)
    B = torch.rand(n, n, dtype=torch.float64, device=dev)
    sec = _timed(torch, lambda: torch.mm(A, B), reps=5, warm=2)
    return 2 * n ** 3 / sec / 1e12


def _configs(kc, torch, dev, args, cols, progs, w):
    """Configs the default line carries beside the headline:
    config 1 (the reference's campaign CSV -> fit -> test predictions, with
    the reference CLI path timed beside it), the fused config-4 argmin over
    the same lattice, config 2 (1e6 points of the four test kernels) and the
    config-3 Gram (1e8 x 40 fp64 rows)."""
    out = {}
    hbm, _ = peaks()
    stream = torch.cuda.current_stream(dev).cuda_stream
    sim_alpha = w.alpha

    # ---- config 1: the reference's own campaign CSV (390 measurement cases,
    # simdev-v1, sigma 0) -> fit -> predict the 16 test cases (suite.cpp
    # test sizes, incl. fd_stencil n=512 and nbody n=2048) on the GPU; the
    # reference CLI path (campaign + bound extraction + fit + eval) beside it
    golden = ROOT / "tests" / "golden"
    tests = json.loads((golden / "fit_suite.json").read_text())["test_predictions"]
    tprogs = {t["kernel"]: kc.load_program(t["kernel"]) for t in tests}

    def c1():
        wf, rep = kc.fit_from_csv(golden / "meas_sigma0.csv", device="simdev-v1")
        outp = []
        for t in tests:
            p = tprogs[t["kernel"]]
            outp.append(kc.predict(wf, p, {q: torch.tensor([int(t["binding"][q])], dtype=torch.int64, device=dev)
                                           for q in p.params}))
        torch.cuda.synchronize()
        return wf, rep, outp
    c1()
    t0 = time.perf_counter()
    wf, rep, outp = c1()
    sec1 = time.perf_counter() - t0
    rel = max(abs(float(o.item()) - float.fromhex(t["predicted_s"][1])) / abs(float.fromhex(t["predicted_s"][1]))
              for o, t in zip(outp, tests))
    ref1 = None
    exe = ROOT / "oracle" / "_ref" / "kcref_bench"
    if exe.exists():
        try:
            ref1 = json.loads(subprocess.run([str(exe), "config1"], capture_output=True, text=True,
                                             timeout=300).stdout)
        except Exception as e:  # noqa: BLE001
            ref1 = {"error": str(e)[:200]}
    out["config1_suite_fit_eval"] = {
        "cases": rep["n_cases"], "test_cases": len(tests), "gpu_ms": sec1 * 1e3,
        "max_rel_diff_test_predictions_vs_reference": rel, "cpu_reference": ref1,
        "note": "GPU: kcg_measurements_read_csv + per-kernel fused Gram + solve + 2 refinement steps (objective from the last) + 16 predictions "
                "(wall clock, ~70 launches); CPU: the reference's run_campaign + extract_properties (bound, "
                "cap 2e7) + fit_weights + predict, 1 thread"}

    # ---- config 2: 1e6 points over the 4 test kernels (250k each) ----------
    U = 250_000
    u = torch.arange(1, U + 1, dtype=torch.int64, device=dev)
    specs = [("matmul_skinny_g16x16", {"n": 16 * u, "m": 128 * u, "l": 16 * u}),
             ("conv_g16x16", {"n": 16 * u}),
             ("fd_stencil_g16x16", {"n": 16 * u}),
             ("nbody_g256", {"n": 256 * u})]
    launches = []
    for kid, cdict in specs:
        p = kc.load_program(kid)
        cdict = {k: v.contiguous() for k, v in cdict.items()}
        launches.append((p, cdict, _colarr(p, cdict), torch.empty(U, dtype=torch.float64, device=dev)))

    def c2():
        for p, _, arr, out in launches:
            kc.api.check(kc.api.lib().kcg_eval_predict(p.handle, arr, U, w.alpha_array(), out.data_ptr(),
                                                       None, None, None, 0, stream))
    sec = _timed(torch, c2, reps=20)
    # the same 4 launches replayed from a CUDA graph (the C ABI launches are
    # capturable once the kernels are specialised): launch overhead removed
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        c2_stream = torch.cuda.current_stream(dev).cuda_stream
        for p, _, arr, o in launches:
            kc.api.check(kc.api.lib().kcg_eval_predict(p.handle, arr, U, w.alpha_array(), o.data_ptr(),
                                                       None, None, None, 0, c2_stream))
    sec_g = _timed(torch, g2.replay, reps=50)
    b64, _ = launches[0][0].safe_bounds()
    out["config2_suite_1e6"] = {
        "points": 4 * U, "ms": sec * 1e3, "points_per_s": 4 * U / sec, "launches": 4,
        "graph_ms": sec_g * 1e3, "graph_points_per_s": 4 * U / sec_g,
        "note": "skinny (16u,128u,16u), conv 16u, fd_stencil 16u, nbody 256u, u=1..250000; skinny counts "
                f"reach 5.8e20 (int128 path for n > {b64}); fd_stencil / nbody use the derived programs "
                "(SURVEY 8f row 1); latency-bound (4 launches)"}
    del launches, u

    # ---- config 4 fused: evaluate + predict + argmin over the 6 variants ---
    total = cols["n"].numel()
    best = torch.empty(total, dtype=torch.int32, device=dev)
    best_t = torch.empty(total, dtype=torch.float64, device=dev)
    handles = (ctypes.c_void_p * len(progs))(*[p.handle.value for p in progs])
    carr = _colarr(progs[0], cols)

    def c4():
        kc.api.check(kc.api.lib().kcg_argmin(handles, len(progs), carr, total, w.alpha_array(),
                                             best.data_ptr(), best_t.data_ptr(), None, stream))
    sec = _timed(torch, c4, reps=5)
    out["config4_argmin_fused"] = {
        "sizes": total, "points": total * len(progs), "ms": sec * 1e3,
        "points_per_s": total * len(progs) / sec, "sizes_per_s": total / sec,
        "bytes_per_size": 36, "hbm_frac": 36 * total / sec / 1e9 / hbm,
        "best_variant_histogram": torch.bincount(best.to(torch.int64) + 1, minlength=len(progs) + 1).tolist(),
        "instruction_roofline": _instr_roofline(_ncu_lane_instr("r02_argmin_ncu.txt"), total * len(progs) / sec,
                                                _pipe_peaks(kc), "profiles/r02_argmin_ncu.txt (ncu, kcg_multiam_v6_tma, default 3-CTA build)"),
        "kernel": "kcg_multiam_v6_tma (one-pass kernel, argmin epilogue)",
        "note": "one fused launch per step; 24 B bindings in, int32 + fp64 out per size"}
    # the same launch also writing every variant's prediction (variant-major):
    # all 1e9 predictions with the bindings read once (24 + 48 B per size
    # instead of 6 x 32 B for six separate launches)
    preds_all = torch.empty((len(progs), total), dtype=torch.float64, device=dev)

    def c4p():
        kc.api.check(kc.api.lib().kcg_argmin(handles, len(progs), carr, total, w.alpha_array(),
                                             best.data_ptr(), best_t.data_ptr(), preds_all.data_ptr(), stream))
    sec = _timed(torch, c4p, reps=5)
    out["config4_fused_all_predictions"] = {
        "points": total * len(progs), "ms": sec * 1e3, "points_per_s": total * len(progs) / sec,
        "bytes_per_size": 24 + 12 + 8 * len(progs), "hbm_frac": (36 + 8 * len(progs)) * total / sec / 1e9 / hbm,
        "note": "kcg_argmin with preds_out: every (variant, size) prediction plus the argmin in one launch"}
    del preds_all, best, best_t

    # ---- config 3: Gram over 1e8 x 40 fp64 materialised rows ---------------
    N, F = 100_000_000, 40
    g = torch.Generator(device=dev).manual_seed(4242)
    X = torch.rand((N, F), dtype=torch.float64, device=dev, generator=g)
    X.mul_(9999.0).add_(1.0)
    st = kc.GramStats.zeros(F, dev)

    def c3():
        st.G.zero_(); st.xt1.zero_(); st.colmax.zero_()
        kc.api.check(kc.api.lib().kcg_gram_accumulate(X.data_ptr(), N, F, F, st.G.data_ptr(),
                                                      st.xt1.data_ptr(), st.colmax.data_ptr(), stream))
    sec = _timed(torch, c3, reps=5)
    # parity at full size: Gram vs a float64 torch reference on a 1e6-row slice
    Xs = X[:1_000_000]
    st2 = kc.gram_accumulate(Xs)
    ref = Xs.T @ Xs
    rel = float(((st2.G - ref).abs().max() / ref.abs().max()).item())
    fp64 = _fp64_peak(torch, dev)
    flops = N * F * (F + 1) + 2 * N * F
    out["config3_gram_1e8x40"] = {
        "rows": N, "cols": F, "ms": sec * 1e3, "rows_per_s": N / sec,
        "hbm_achieved_GBps": 8 * F * N / sec / 1e9, "hbm_frac": 8 * F * N / sec / 1e9 / hbm,
        "fp64_tflops": flops / sec / 1e12, "fp64_peak_tflops_measured_dgemm": fp64,
        "fp64_frac": flops / sec / 1e12 / fp64, "slice_rel_err_vs_torch": rel,
        "kernel": "kcg_gram_hybrid<5,96,true> (AOT: off-diagonal 8x8 blocks on DMMA m8n8k4 f64, diagonal blocks' upper triangles on DFMA, TMA-staged rows)"}

    # the same Gram on the int8 tensor cores (tcgen05.mma kind::i8, TMEM accumulators):
    # the alternative back end kcg_gram_accumulate_sliced, not the default
    def c3s():
        st.G.zero_(); st.xt1.zero_(); st.colmax.zero_()
        kc.api.check(kc.api.lib().kcg_gram_accumulate_sliced(X.data_ptr(), N, F, F, st.G.data_ptr(),
                                                              st.xt1.data_ptr(), st.colmax.data_ptr(), stream))
    sec_s = _timed(torch, c3s, reps=3)
    st3 = kc.gram_accumulate(Xs, sliced=True)
    A = Xs.abs()
    out["config3_gram_1e8x40"]["int8_tensor_core_alternative"] = {
        "ms": sec_s * 1e3, "hbm_frac": 8 * F * N / sec_s / 1e9 / hbm,
        "slice_err_rel_to_abs_scale": float(((st3.G - ref).abs() / (A.T @ A)).max().item()),
        "kernel": "kcg_gram_sliced<40,true> (7 signed 8-bit digits per value, tcgen05.mma kind::i8 M=128 N=144/144/80 "
                  "per 32-row K step, int32 TMEM accumulators drained per segment; DESIGN.md section 4)"}
    del X, Xs, st, st2, st3, ref, A

    return out


def _extras(kc, torch, dev, args):
    """Config 5 on one GPU, the grid-descriptor path and the GPU enumeration
    oracle (--extras)."""
    import ctypes
    out = {}
    hbm, _ = peaks()
    sim_alpha = _simdev_alpha(kc)
    w = kc.ModelWeights(device="simdev-v1", alpha=sim_alpha, covered=[a != 0 for a in sim_alpha])
    stream = torch.cuda.current_stream(dev).cuda_stream

    side = args.side
    total = side ** 3
    progs = [kc.load_program(v) for v in VARIANTS]
    # ---- config 4 from a grid descriptor: the same 1e9
    # (variant, size) points, bindings generated in registers -- 8 B/point out
    preds = torch.empty(total, dtype=torch.float64, device=dev)
    grids = [kc.Grid.for_program(p, {"n": (UNIT, UNIT, side), "m": (UNIT, UNIT, side), "l": (UNIT, UNIT, side)})
             for p in progs]
    gstructs = [g.c_struct() for g in grids]

    def c4g():
        for p, g in zip(progs, gstructs):
            kc.api.check(kc.api.lib().kcg_eval_predict_grid(p.handle, ctypes.byref(g), 0, total, w.alpha_array(),
                                                            preds.data_ptr(), None, 0, stream))
    sec = _timed(torch, c4g, reps=5)
    out["config4_grid_descriptor"] = {
        "points": total * len(progs), "ms": sec * 1e3, "points_per_s": total * len(progs) / sec,
        "bytes_per_point": 8, "hbm_frac": 8 * total * len(progs) / sec / 1e9 / hbm,
        "note": "kcg_eval_predict_grid per variant: lattice (n,m,l)=336*(u,v,w) decoded per thread "
                "(odometer), exact evaluate + predict, fp64 predictions streamed out"}
    del preds

    # ---- config 5 (single GPU): fused evaluate -> row -> Gram, 1e9 rows ----
    tiled = kc.load_program("matmul_tiled_g16x16")
    side5 = 1000
    rows = side5 ** 3
    idx = torch.arange(0, rows, dtype=torch.int64, device=dev)
    cols5 = {"n": ((idx // (side5 * side5) + 1) * 16).contiguous(),
             "m": (((idx // side5) % side5 + 1) * 16).contiguous(),
             "l": ((idx % side5 + 1) * 16).contiguous()}
    del idx
    T = kc.noiseless_time(sim_alpha, tiled, cols5)   # stored timings on the GPU
    st5 = kc.GramStats.zeros(len(tiled.props), dev)
    a5 = _colarr(tiled, cols5)

    def c5():
        st5.G.zero_(); st5.xt1.zero_(); st5.colmax.zero_()
        kc.api.check(kc.api.lib().kcg_gram_fused(tiled.handle, a5, T.data_ptr(), rows, st5.G.data_ptr(),
                                                 st5.xt1.data_ptr(), st5.colmax.data_ptr(), None, stream))
    sec = _timed(torch, c5, reps=3, warm=1)
    alpha, rank = kc.solve_gram(st5)
    obj = torch.zeros(1, dtype=torch.float64, device=dev)
    full = [0.0] * kc.schema_size()
    for j, k in enumerate(tiled.props):
        full[k] = alpha[j]
    sec_r = _timed(torch, lambda: kc.api.check(kc.api.lib().kcg_residual_fused(
        tiled.handle, a5, T.data_ptr(), rows, (ctypes.c_double * len(full))(*full), obj.data_ptr(), stream)),
        reps=1, warm=0)
    out["config5_fused_gram_1gpu"] = {
        "rows": rows, "ms": sec * 1e3, "rows_per_s": rows / sec,
        "hbm_frac": 32 * rows / sec / 1e9 / hbm, "rank": rank,
        "residual_pass_ms": sec_r * 1e3, "objective": float(obj.item()),
        "note": "matmul_tiled_g16x16 rows (n,m,l)=16*(u,v,w) u,v,w<=1000, T = noiseless_time on the GPU; "
                "9 columns of rank 2 (all flop/memory counts are multiples of n*m*l): min-norm solve"}
    del cols5, T

    # ---- GPU enumeration oracle vs the reference's CPU
    # enumerate_points on this host (single-threaded, as in the reference)
    ep = kc.load_enum_program("fd_stencil_g16x16")
    ne = 16384
    ep.enumerate_points({"n": 1024})  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    counts, pts = ep.enumerate_points({"n": ne})
    sec_e = time.perf_counter() - t0
    ref = None
    exe = ROOT / "oracle" / "_ref" / "kcref_bench"
    if exe.exists():
        try:
            r = subprocess.run([str(exe), "enumerate", "fd_stencil_g16x16", "512"], capture_output=True,
                               text=True, timeout=120)
            ref = json.loads(r.stdout)
        except Exception as e:  # noqa: BLE001
            ref = {"error": str(e)[:200]}
    out["enumerate_fd_stencil"] = {
        "n": ne, "visited_points": pts, "seconds": sec_e, "points_per_s": pts / sec_e,
        "equals_symbolic": counts == {kc.schema_keys()[k]: v for k, v in _sym_counts(kc, torch, dev, ne).items()},
        "cpu_reference_n512": ref,
        "note": "kcg_enumerate_points (statement walks + footprint bitmaps + host tally), wall clock incl. "
                "host compile and sync; CPU: reference enumerate_points (shim bigint), 1 thread"}
    return out


def _sym_counts(kc, torch, dev, n):
    p = kc.load_program("fd_stencil_g16x16")
    bb = kc.evaluate_properties(p, {"n": torch.tensor([n], dtype=torch.int64, device=dev)})
    torch.cuda.synchronize()
    return {k: bb.counts_int(j, 0) for j, k in enumerate(p.props) if bb.counts_int(j, 0)}


if __name__ == "__main__":
    main()
