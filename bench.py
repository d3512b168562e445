#!/usr/bin/env python3
"""ABCS hot-path benchmark (contract: one JSON line from rank 0).

Headline (BASELINE.json metric, workload = configs[1], "cfg2"): megapixels/s of
sense + reconstruct (DD-ABCS, B=16, fp32 DCTs, inverse-DCT reconstruction) over a
batch of 1024 synthetic 512x512 uint8 images per GPU, one step = the subrate
sweep {0.1, 0.3, 0.5} (3 x 1024 images). Inputs are resident in HBM (generated
on device) and larger than L2 (268 MB u8 per subrate + ~1.4 GB of outputs).
Secondary object "ida": cfg4 (64 x 512^2, BBV 0.3, 10 IDA iterations), image-
iterations/s. Multi-GPU: one process per GPU, each rank senses its own 1024
images (disjoint global image indices), no collective on the data path
("scaling": "weak"); timing is the max over ranks of CUDA-event time.

--impl reference runs the reference's own CPU implementation (oracle/_ref, the
unmodified reference library, else the C port) on the host cores on a bounded
sample of the same workload.
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

SUBRATES = ((1, 10), (3, 10), (1, 2))
CFG2 = dict(H=512, W=512, B=16, n=1024, ellipses=20, sigma=5.0, seed=2)
CFG4 = dict(H=512, W=512, B=16, n=64, ellipses=20, sigma=5.0, seed=4, num=3, den=10, iters=10)


def load_traffic():
    """DRAM bytes per image of the hot kernels from the committed ncu --set full capture summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's own start-up (NVML init, first query) stays out of the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 2.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- distributed plumbing
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" and not args.dry_run else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def shard(rank, per_rank):
    """Global image indices [first, first + per_rank) of this rank: each rank senses its own
    images of one global seeded dataset; no data moves between ranks."""
    return rank * per_rank, per_rank


def aggregate_rate(units_per_rank, world, seconds_max):
    """Whole-job throughput: the units all ranks processed / the slowest rank's time."""
    return world * units_per_rank / seconds_max


def max_over_ranks(v, world, device=None):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- CPU (reference) arm
def cpu_sample(checker, imgs, threads):
    """sense + reconstruct(idct) of every image at every subrate; returns (seconds, pixels)."""
    t0 = time.perf_counter()
    px = 0
    for num, den in SUBRATES:
        if hasattr(checker, "sense_reconstruct_batch"):
            checker.sense_reconstruct_batch(imgs, CFG2["B"], num, den, 2, method=0, iters=1, threads=threads)
        else:  # C port: per image, threaded
            from concurrent.futures import ThreadPoolExecutor

            def one(i):
                ms = checker.sense(imgs[i], CFG2["B"], num, den, 2)
                checker.decode(ms["rows"], ms["cols"], CFG2["B"], ms["counts"], ms["coeffs"])

            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(len(imgs))))
        px += imgs.shape[0] * imgs.shape[1] * imgs.shape[2]
    return time.perf_counter() - t0, px


CPU_TARGET_CORE_S = 40.0  # calibration overestimates per-image cost ~2x: lands at ~15-25 core-seconds


def calibrated_count(checker, imgs, threads, cap):
    """Images per CPU sample so one sample is ~CPU_TARGET_CORE_S core-seconds (a multiple of threads)."""
    n0 = min(len(imgs), threads)
    cpu_sample(checker, imgs[:n0], threads)  # warm-up (thread start, page-in)
    sec, _ = cpu_sample(checker, imgs[:n0], threads)
    per_img = sec * min(threads, n0) / n0  # core-seconds per image (all subrates)
    n = int(CPU_TARGET_CORE_S / max(per_img, 1e-6))
    n = max(threads, (n // threads) * threads)
    return min(n, cap)


def oracle_module():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as o
    return o


def sample_images(n, c=CFG2, first=0, video=False):
    """BASELINE inputs for the CPU arms from the oracle library's copy of the seeded generator
    (oracle/synth_inputs.c): the reference arm never loads the product library."""
    return oracle_module().synth_images(c["H"], c["W"], c["ellipses"], c["sigma"], c["seed"], first, n, video)


def get_checker():
    o = oracle_module()
    if o.Reference.available():
        return o.Reference(), "reference"
    return o.CPort(), "port"


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    checker, kind = get_checker()
    threads = host_cores()
    n = calibrated_count(checker, sample_images(threads), threads, cap=1024)
    imgs = sample_images(n)
    for _ in range(max(args.warmup - 1, 0)):
        cpu_sample(checker, imgs[: min(n, threads)], threads)
    times, px = [], 0
    for _ in range(args.steps):
        t, p_ = cpu_sample(checker, imgs, threads)
        times.append(t)
        px = p_
    sec = float(np.mean(times))
    value = px / sec / 1e6
    sample = f"{n} cfg2 images (512x512, seed {CFG2['seed']}) x subrates {{0.1,0.3,0.5}} per step"
    line = {
        "impl": "reference", "metric": "megapixels/s for ABCS sense+reconstruct", "value": round(value, 3),
        "unit": "MP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: DD-ABCS B=16 subrate sweep {0.1,0.3,0.5}, IDCT reconstruction, 512x512 u8",
                   "images_per_step": n, "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "MP/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


CPU_CONFIGS = [  # (key, H, W, B, num, den, algo(1 BBV, 2 DD), ellipses, sigma, seed, video, ida_iterations)
    ("cfg1", 256, 256, 16, 1, 4, 1, 20, 5.0, 1, False, 0),
    ("cfg3", 1080, 1920, 8, 1, 5, 1, 20, 5.0, 3, True, 0),
    ("cfg4", 512, 512, 16, 3, 10, 1, 20, 5.0, 4, False, 10),
    ("cfg5", 4096, 4096, 16, 1, 4, 2, 200, 8.0, 5, False, 5),
]


def cpu_config_baselines(threads):
    """The reference library (oracle/_ref) timed on this host beside every other BASELINE config:
    sense + decode_idct MP/s, and for cfg4/cfg5 the IDA loop (recon.cpp:225-257) in image-iterations/s.
    Each phase runs over `threads` images on `threads` host threads (the reference is reentrant);
    cfg1 is one image on one core, median of 5 (tools/abcs_main.cpp:42-52). cfg5's IDA runs one
    iteration per image and is extrapolated per iteration as t(Ida, 1) - t(Idct) (the warm-start
    init is one decode plus one forward, about one Idct reconstruct)."""
    o = oracle_module()
    if not o.Reference.available():
        return {"unavailable": "oracle/_ref not built"}
    res = {}
    for key, H, W, B, num, den, algo, ell, sig, seed, video, iters in CPU_CONFIGS:
        spec = dict(H=H, W=W, ellipses=ell, sigma=sig, seed=seed)
        if key == "cfg1":
            imgs = sample_images(1, spec)
            runs = sorted(sum(o.reference_bench_phases(imgs, B, num, den, algo, 0, 1, 1)) for _ in range(5))
            t = runs[2]
            res[key] = {"sense_decode_ms": round(t * 1e3, 3), "MP_s": round(H * W / t / 1e6, 3), "cores": 1,
                        "sample": "1 image, median of 5 (sense + decode_idct)"}
            continue
        n = threads * (4 if key in ("cfg3", "cfg4") else 1)
        imgs = sample_images(n, spec, video=video)
        ts, td = o.reference_bench_phases(imgs, B, num, den, algo, 0, 1, threads)
        row = {"MP_s": round(n * H * W / (ts + td) / 1e6, 3), "sense_s": round(ts, 3), "decode_s": round(td, 3),
               "cores": threads, "sample": f"{n} images (seed {seed}) over {threads} host threads"}
        if iters:
            it_run = iters if key == "cfg4" else 1
            _, ti = o.reference_bench_phases(imgs, B, num, den, algo, 5, it_run, threads)
            if key == "cfg4":
                row["ida_it_s"] = round(n * iters / ti, 2)
                row["ida_sample"] = f"{n} images x {iters} iterations incl. warm-start init"
            else:
                step = max(ti - td, 1e-9)
                row["ida_it_s"] = round(n / step, 3)
                row["ida_sample"] = (f"{n} images x 1 iteration; per-iteration time = t(Ida,1) - t(Idct) = "
                                     f"{step:.2f} s wall (extrapolated to {iters} iterations)")
        res[key] = row
    return res


# ---------------------------------------------------------------- GPU arm
def run_ours(args, world, rank, local):
    import torch
    import paper_2001_09632_b200 as p

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    ctx = p.Context.get(local)
    hbm, peak_src = peaks()
    n = CFG2["n"]
    spec = p.SynthSpec(CFG2["H"], CFG2["W"], CFG2["ellipses"], CFG2["sigma"], CFG2["seed"])
    first, n = shard(rank, n)
    imgs = p.synth_images(spec, first, n, device=local)  # disjoint global indices per rank
    cfgs = [p.SensingConfig(CFG2["B"], num, den, p.Algorithm.DD) for num, den in SUBRATES]
    plans = [p.sense_plan(c, CFG2["H"], CFG2["W"]) for c in cfgs]
    # outputs allocated once: payload/counts/offsets per subrate + decoded images
    fused = [p.sense_decode_batch(imgs, c, pl) for c, pl in zip(cfgs, plans)]
    batches = [f[0] for f in fused]
    outs = [f[1] for f in fused]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    nsub = len(SUBRATES)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nsub + 1)] for _ in range(args.steps)]

    def step_independent(evs):
        # one subrate at a time: sense (DD phase 1 + allocation + zigzag gather) and decode_idct,
        # fused over the payload
        for j, (c, pl, b) in enumerate(zip(cfgs, plans, batches)):
            if evs and j == 0:
                evs[0].record(stream)
            p.sense_decode_batch(imgs, c, pl, out=b, image_out=outs[j])
            if evs:
                evs[j + 1].record(stream)

    def step_sweep(evs):
        # the subrate sweep in one call: DD phase 1 of the 3 subrates from one forward transform
        # per block, then per subrate its own fixup, allocation, payload and decode (outputs
        # identical to step_independent: tests/test_gpu_parity.py::test_sense_decode_sweep_*)
        p.sense_decode_sweep(imgs, cfgs, outs=batches, image_outs=outs)  # (no per-step events: one call)

    step = step_independent if args.independent else step_sweep

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    barrier(world)
    launches0 = ctx.launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)  # the timed region: no per-kernel instrumentation inside it
    for k in range(args.steps):
        step(ev[k])
    end.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    # per-kernel CUDA events on the launching streams, from an instrumented repeat of the same steps
    ctx.kernel_timing(True)
    for k in range(args.steps):
        step(None)
    torch.cuda.synchronize()
    ktimes_conc = ctx.kernel_times()
    ctx.kernel_timing(False)
    # The timed region pipelines each batch over 3 streams, so concurrent kernels stretch each
    # other's event times. The per-kernel roofline therefore comes from a serialised pass of the
    # same steps (1 stream) right after it; kernel shares of that pass are the ncu-comparable ones.
    ctx.set_pipeline_streams(1)
    ctx.kernel_timing(True)
    ser0, ser1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ser0.record(stream)
    for k in range(args.steps):
        step(None)
    ser1.record(stream)
    torch.cuda.synchronize()
    ktimes = ctx.kernel_times()
    ctx.kernel_timing(False)
    ctx.set_pipeline_streams(3)
    ser_step_ms = ser0.elapsed_time(ser1) / args.steps
    clk = clocks.stop() if clocks else None
    # the per-subrate path (one sense_decode_batch per subrate), timed the same way: its
    # per-subrate phases give the pipeline roofline, and its rate is reported beside the sweep
    ev_ind = [[torch.cuda.Event(enable_timing=True) for _ in range(nsub + 1)] for _ in range(args.steps)]
    for _ in range(args.warmup):
        step_independent(None)
    torch.cuda.synchronize()
    barrier(world)
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    for k in range(args.steps):
        step_independent(ev_ind[k])
    i1.record(stream)
    torch.cuda.synchronize()
    ind_ms_max = max_over_ranks(i0.elapsed_time(i1), world, dev)
    barrier(world)
    sub_ms = [sum(ev_ind[k][j].elapsed_time(ev_ind[k][j + 1]) for k in range(args.steps)) / args.steps
              for j in range(nsub)]
    ms = start.elapsed_time(end)
    ms_max = max_over_ranks(ms, world, dev)
    ms_step = ms_max / args.steps
    px_step = nsub * n * CFG2["H"] * CFG2["W"]
    value = aggregate_rate(px_step * args.steps, world, ms_max / 1e3) / 1e6

    # per-kernel roofline from the library's CUDA events (launching streams) over the timed region:
    # algorithmic bytes per image of each kernel of the fused DD step
    N = CFG2["H"] * CFG2["W"]
    Ks = [pl.coeffs_per_image for pl in plans]
    nB = plans[0].n_blocks
    alg_bytes = {  # per step (all subrates)
        # u8 in (once per step for the sweep's single multi-plan pass), payload+counts/offsets, f32 out
        "sense16_gather_decode": (0 if args.independent else -(nsub - 1) * n * N)
        + sum(n * (N + 4 * K + 6 * nB + 4 * N) for K in Ks),
        "sense16_weights": nsub * n * (N + 4 * nB),                                    # u8 in, n_i out
        "sense16_weights_sweep": n * (N + nsub * 4 * nB),                              # u8 in once, n_i per subrate
        "alloc_cta": nsub * n * (4 * nB + 6 * nB),                                     # n_i in, counts+offsets out
    }
    kt = {k: v for k, v in ktimes.items()}
    dom = max(kt, key=lambda k: kt[k][1]) if kt else None
    roof = None
    if dom is not None:
        launches_k, total_ms, _ = kt[dom]
        per_step_ms = total_ms / args.steps
        lps = launches_k / args.steps
        bytes_step = alg_bytes.get(dom)
        ach = bytes_step / (per_step_ms / 1e3) / 1e9 if bytes_step else None
        traffic = None
        tr = load_traffic().get(dom)
        if tr and bytes_step:
            traffic = round(tr["dram_bytes_per_image"] * (nsub * n / lps))
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1) if ach else None, "peak": hbm,
                "peak_source": peak_src, "unit": "GB/s", "frac": round(ach / hbm, 4) if ach else None,
                "traffic": traffic, "algorithmic_bytes_per_launch": round(bytes_step / lps) if bytes_step else None,
                "avg_launch_ms": round(total_ms / launches_k, 4), "launches_per_step": lps,
                "share_of_step": round(per_step_ms / ser_step_ms, 4), "measured_on": "serialised pass (1 stream)",
                "traffic_source": tr.get("source") if tr else None}
    kernels = {k: {"launches_per_step": v[0] / args.steps, "ms_per_step": round(v[1] / args.steps, 4),
                   "share_of_step": round(v[1] / args.steps / ser_step_ms, 4),
                   "concurrent_ms_per_step": round(ktimes_conc.get(k, (0, 0.0, 0))[1] / args.steps, 4),
                   "achieved_gbs": (round(alg_bytes[k] / (v[1] / args.steps / 1e3) / 1e9, 1) if k in alg_bytes
                                    else None)} for k, v in kt.items()}
    per_j = []
    for j, K in enumerate(Ks):
        b_j = n * (N + 4 * K + 2 * nB) + n * (4 * K + 2 * nB + 4 * N)
        per_j.append(dict(subrate=f"{SUBRATES[j][0]}/{SUBRATES[j][1]}", K=K, ms=round(sub_ms[j], 4),
                          algorithmic_bytes=b_j, frac=round(b_j / (sub_ms[j] / 1e3) / 1e9 / hbm, 4)))
    pipe_ach = sum(x["algorithmic_bytes"] for x in per_j) / (sum(sub_ms) / 1e3) / 1e9

    # e2e through the C ABI with host buffers (pinned), H2D + kernels + D2H in the timed region
    import ctypes as C
    lib = p._lib.load()
    h_in = torch.empty((n, CFG2["H"], CFG2["W"]), dtype=torch.uint8, pin_memory=True)
    h_in.copy_(imgs.cpu())
    h_out = torch.empty((n, CFG2["H"], CFG2["W"]), dtype=torch.float32, pin_memory=True)
    # one output buffer per subrate: the step's decoded images all come back to the host
    h_outs = [h_out] + [torch.empty_like(h_out, pin_memory=True) for _ in plans[1:]]
    parr = (p._lib.SensePlanC * nsub)(*plans)
    oarr = (C.c_void_p * nsub)(*[t.data_ptr() for t in h_outs])
    e2e_times = []
    for it in range(1 + max(1, min(args.steps, 3))):
        barrier(world)
        t0 = time.perf_counter()
        if args.independent:
            for pl, ho in zip(plans, h_outs):
                st = lib.abcs_sense_decode_host(ctx.handle, C.byref(pl), h_in.data_ptr(), n, ho.data_ptr(),
                                                None, None, 64)
                if st != 0:
                    raise RuntimeError(p._lib.last_error())
        else:  # the sweep: each chunk of images uploaded once for the 3 subrates
            st = lib.abcs_sense_decode_sweep_host(ctx.handle, parr, nsub, h_in.data_ptr(), n, oarr, 64)
            if st != 0:
                raise RuntimeError(p._lib.last_error())
        dt = time.perf_counter() - t0
        if it > 0:
            e2e_times.append(dt)
    e2e_s = max_over_ranks(float(np.mean(e2e_times)), world, dev)
    e2e_value = aggregate_rate(px_step, world, e2e_s) / 1e6
    h2d = (len(SUBRATES) if args.independent else 1) * n * N
    d2h = len(SUBRATES) * n * N * 4

    # the reference bench's own step (abcs_main.cpp:226-258): sense + decode every image under
    # every subrate, then psnr/ssim per cell; only the cells (mse, psnr, ssim: f64) come back
    cells = [torch.empty((nsub, n), dtype=torch.float64, pin_memory=True) for _ in range(3)]
    cell_times = []
    for it in range(1 + max(1, min(args.steps, 3))):
        barrier(world)
        t0 = time.perf_counter()
        st = lib.abcs_bench_cells_host(ctx.handle, parr, nsub, h_in.data_ptr(), n, *[c.data_ptr() for c in cells], 64)
        if st != 0:
            raise RuntimeError(p._lib.last_error())
        dt = time.perf_counter() - t0
        if it > 0:
            cell_times.append(dt)
    cells_s = max_over_ranks(float(np.mean(cell_times)), world, dev)
    e2e_cells = {"value": round(aggregate_rate(px_step, world, cells_s) / 1e6, 1), "unit": "MP/s",
                 "h2d_bytes_per_step": n * N, "d2h_bytes_per_step": 3 * nsub * n * 8,
                 "api": "abcs_bench_cells_host (the reference bench step: mse/psnr/ssim cells back, pinned host images in)",
                 "mean_psnr_db": [round(float(x), 3) for x in cells[1].mean(dim=1)]}

    # secondary: cfg4 IDA (64 x 512^2, BBV 0.3, 10 iterations)
    ida = run_ida(p, torch, local, rank, hbm, world, dev)

    # the .abcs container of the subrate-0.3 batch, packed and unpacked on the device
    container = None
    if rank == 0:
        try:
            container = container_bench(p, torch, batches[1], hbm)
        except Exception as e:
            container = {"error": repr(e)[:200]}

    # batched quality metrics of the subrate-0.3 decode against its sources
    metrics = None
    if rank == 0:
        try:
            metrics = metrics_bench(p, torch, imgs, outs[1], hbm)
        except Exception as e:
            metrics = {"error": repr(e)[:200]}

    # the rest of the reconstruction family on the cfg4 batch
    family = None
    if rank == 0:
        try:
            family = family_bench(p, torch)
        except Exception as e:
            family = {"error": repr(e)[:200]}

    # THB / THI oracle decodes (fp64, bit-exact) on 64 of the cfg2 images at subrate 0.3
    oracles = None
    if rank == 0:
        try:
            oracles = {}
            sub = imgs[:64]
            for name, glob in (("thb", False), ("thi", True)):
                p.threshold_decode_batch(sub, cfgs[1], glob)
                torch.cuda.synchronize()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                p.threshold_decode_batch(sub, cfgs[1], glob)
                s1.record()
                torch.cuda.synchronize()
                ms_o = s0.elapsed_time(s1)
                oracles[name] = {"ms": round(ms_o, 3), "MP_s": round(64 * CFG2["H"] * CFG2["W"] / ms_o / 1e3, 1)}
            oracles["workload"] = "64 x 512^2, DD 3/10 budget, fp64 transforms (bit-exact oracle baselines)"
        except Exception as e:
            oracles = {"error": repr(e)[:200]}

    # the other BASELINE configs (parity-test workloads, not bench lines): device throughput and
    # algorithmic-bytes roofline fraction of sense+decode (and IDA) on this rank's GPU
    configs = None
    if rank == 0 and not args.no_config_sweep:
        try:
            configs = config_sweep(p, torch, hbm)
        except Exception as e:  # informative only; never fail the headline line
            configs = {"error": repr(e)[:200]}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        checker, kind = get_checker()
        threads = host_cores()
        ns = calibrated_count(checker, imgs[:threads].cpu().numpy(), threads, cap=imgs.shape[0])
        himgs = imgs[:ns].cpu().numpy()
        sec, pxs = cpu_sample(checker, himgs, threads)
        cpu = {"value": round(pxs / sec / 1e6, 3), "unit": "MP/s", "cores": threads, "kind": kind,
               "sample": f"{ns} of this rank's cfg2 images x subrates {{0.1,0.3,0.5}} "
                         f"({sec:.2f} s wall, ~{sec * threads:.0f} core-s)"}
        if kind == "reference":
            try:
                cpb = cpu_config_baselines(threads)
            except Exception as e:
                cpb = {"error": repr(e)[:200]}
            cpu["configs"] = cpb
            if isinstance(configs, dict):  # each config's device row gets the reference beside it
                for name, row in configs.items():
                    k = name.split()[0]
                    if isinstance(row, dict) and k in cpb:
                        row["cpu_reference"] = cpb[k]
            if isinstance(ida, dict) and "cfg4" in cpb and "ida_it_s" in cpb["cfg4"]:
                ida["cpu_reference"] = {"value": cpb["cfg4"]["ida_it_s"], "unit": "it/s", "cores": threads,
                                        "kind": "reference", "sample": cpb["cfg4"]["ida_sample"]}

    if rank == 0:
        line = {
            "metric": "megapixels/s for ABCS sense+reconstruct", "value": round(value, 1), "unit": "MP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp16 hi/lo operands, fp32 accumulate)", "data": "synthetic",
            "config": {"workload": "cfg2: 1024 x 512x512 u8 per GPU, DD-ABCS B=16, subrate sweep {0.1,0.3,0.5}, "
                                   "IDCT reconstruction (BASELINE configs[1])",
                       "global_batch": world * n, "l2": "inputs+outputs >> L2 (no flush needed)",
                       "parallelism": f"dp{world} (independent images, no collective)"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernels": kernels,
            "serialised_ms_per_step": round(ser_step_ms, 3),
            "step_api": ("one sense_decode_batch per subrate" if args.independent else
                         "sense_decode_sweep (abcs_sense_decode_sweep_batch): shared DD phase-1 transform"),
            "independent_subrates": {"what": "the same step as one sense_decode_batch call per subrate",
                                     "value": round(aggregate_rate(px_step * args.steps, world, ind_ms_max / 1e3)
                                                    / 1e6, 1), "unit": "MP/s",
                                     "ms_per_step": round(ind_ms_max / args.steps, 3)},
            "pipeline_roofline": {"what": "whole step vs its algorithmic bytes (SURVEY 8d), per subrate on the "
                                          "independent path",
                                  "achieved": round(pipe_ach, 1), "frac": round(pipe_ach / hbm, 4), "phases": per_j},
            "e2e": {"value": round(e2e_value, 1), "unit": "MP/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": ("abcs_sense_decode_host per subrate" if args.independent else
                            "abcs_sense_decode_sweep_host") + " (pinned host buffers)"},
            "e2e_bench_cells": e2e_cells,
            "ida": ida,
            "container": container,
            "metrics": metrics,
            "recon_family": family,
            "threshold_oracles": oracles,
            "configs": configs,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    return 0


def container_bench(p, torch, b, hbm):
    """write/read_measurement_set bytes for a 1024-image batch: pack (counts+payload -> containers) and
    unpack (+ validation); algorithmic bytes = bytes read + bytes written."""
    data = p.pack_containers(b)
    p.unpack_containers(data, b.plan)
    torch.cuda.synchronize()
    size = p.container_size(b.plan)
    nB, K = b.plan.n_blocks, b.plan.coeffs_per_image
    src = b.n * (2 * nB + 4 * K)
    dst = b.n * size

    def t(fn, reps=10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    ms_pack = t(lambda: p.pack_containers(b, out=data))
    # unpack: device time of its kernels (validate + unpack) from the ctx's CUDA events; the
    # Python wrapper's per-container status readback is host work outside the device path
    ctx = p.Context.get()
    ctx.kernel_timing(True)
    for _ in range(10):
        p.unpack_containers(data, b.plan)
    kt = ctx.kernel_times()
    ctx.kernel_timing(False)
    ms_unpack = sum(v[1] for k, v in kt.items() if k in ("container_validate", "container_unpack")) / 10
    return {"workload": f"{b.n} containers of cfg2 DD 3/10 ({size} B each)",
            "pack_ms": round(ms_pack, 4), "pack_gbs": round((src + dst) / ms_pack / 1e6, 1),
            "pack_frac": round((src + dst) / ms_pack / 1e6 / hbm, 4),
            "unpack_ms": round(ms_unpack, 4), "unpack_gbs": round((src + dst) / ms_unpack / 1e6, 1),
            "unpack_frac": round((src + dst) / ms_unpack / 1e6 / hbm, 4)}


def metrics_bench(p, torch, refs, dec, hbm):
    """mse+psnr and ssim (metrics.cpp:63-125) of 1024 decoded 512^2 images: algorithmic bytes
    = u8 reference + f32 image per pixel."""
    n = refs.shape[0]
    px = n * refs.shape[1] * refs.shape[2]

    def t(want, reps=3):
        p.quality_batch(refs, dec, want)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            p.quality_batch(refs, dec, want)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    ms_p, ms_s = t(("mse", "psnr")), t(("ssim",))
    return {"workload": f"{n} x 512^2 decoded (DD 3/10) vs sources",
            "mse_psnr_ms": round(ms_p, 4), "mse_psnr_frac": round(5 * px / ms_p / 1e6 / hbm, 4),
            "ssim_ms": round(ms_s, 4), "ssim_mp_s": round(px / ms_s / 1e3, 1),
            "ssim_note": "fp64 11x11 Gaussian statistics, taps in the reference's order with DFMA (FP64-bound)"}


def family_bench(p, torch):
    """image-iterations/s of ISTA, AMP, DAMP (dct_threshold, with the Monte-Carlo divergence) and IDA
    with the blur denoiser on cfg4's batch (64 x 512^2, BBV 0.3), 10 iterations each."""
    c = CFG4
    imgs = p.synth_images(p.SynthSpec(c["H"], c["W"], c["ellipses"], c["sigma"], c["seed"]), 0, c["n"])
    b = p.sense_batch(imgs, p.SensingConfig(c["B"], c["num"], c["den"], p.Algorithm.BBV))
    out = torch.empty((c["n"], c["H"], c["W"]), dtype=torch.float32, device=imgs.device)
    res = {}
    for name, rc in (("ista", p.ReconConfig(p.ReconMethod.Ista, 10, 2.0, p.DenoiserSpec(), 0.05)),
                     ("amp", p.ReconConfig(p.ReconMethod.Amp, 10, 2.0, p.DenoiserSpec(), 1.0)),
                     ("damp_dct", p.ReconConfig(p.ReconMethod.Damp, 10)),
                     ("ida_blur", p.ReconConfig(p.ReconMethod.Ida, 10, 2.0, p.DenoiserSpec("blur")))):
        p.recon_batch(b, rc, out=out, trace=False, check=False)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        p.recon_batch(b, rc, out=out, trace=False, check=False)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        res[name] = {"ms_per_batch": round(ms, 3), "it_s": round(c["n"] * 10 / ms * 1e3, 1)}
    return {"workload": "cfg4 batch: 64 x 512^2, BBV 0.3, 10 iterations", **res}


SWEEP = [  # (name, H, W, n, B, num, den, algorithm, ellipses, sigma, seed, video, ida_iterations)
    ("cfg1 1x256^2 B16 BBV0.25", 256, 256, 1, 16, 1, 4, "BBV", 20, 5.0, 1, False, 0),
    ("cfg3 256x1920x1080 B8 BBV0.2", 1080, 1920, 256, 8, 1, 5, "BBV", 20, 5.0, 3, True, 0),
    ("cfg4 64x512^2 B16 BBV0.3 + IDA10", 512, 512, 64, 16, 3, 10, "BBV", 20, 5.0, 4, False, 10),
    ("cfg5 16x4096^2 B16 DD0.25 + IDA5 (one GPU's shard of 128)", 4096, 4096, 16, 16, 1, 4, "DD", 200, 8.0, 5,
     False, 5),
]


def config_sweep(p, torch, hbm):
    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    out = {}
    for name, H, W, n, B, num, den, algo, ell, sig, seed, video, iters in SWEEP:
        imgs = p.synth_images(p.SynthSpec(H, W, ell, sig, seed, video=video), 0, n)
        cfg = p.SensingConfig(B, num, den, getattr(p.Algorithm, algo))
        plan = p.sense_plan(cfg, H, W)
        b, dec = p.sense_decode_batch(imgs, cfg, plan)
        ms = timed(lambda: p.sense_decode_batch(imgs, cfg, plan, out=b, image_out=dec))
        N, K, S, nB = H * W, plan.coeffs_per_image, plan.side_per_image, plan.n_blocks
        Nc = plan.rows * B * plan.cols * B
        alg = n * (N + 8 * K + 4 * nB + 4 * S + 4 * Nc)
        row = {"sense_decode_ms": round(ms, 4), "MP_s": round(n * N / ms / 1e3, 1),
               "hbm_frac": round(alg / (ms / 1e3) / 1e9 / hbm, 4)}
        if iters:
            rc = p.ReconConfig(p.ReconMethod.Ida, iterations=iters)
            ms_i = timed(lambda: p.ida_batch(b, rc, out=dec, trace=False, check=False), reps=3)
            alg_i = n * ((8 * Nc + 12 * K) * iters + 8 * K + 4 * Nc)
            row.update({"ida_ms": round(ms_i, 3), "ida_it_s": round(n * iters / ms_i * 1e3, 1),
                        "ida_hbm_frac": round(alg_i / (ms_i / 1e3) / 1e9 / hbm, 4)})
        out[name] = row
        del imgs, b, dec
        torch.cuda.empty_cache()
    return out


# fp32 pipe operations per pixel per IDA iteration as the kernel computes them (IDA):
# the denoiser's 8-point butterflies (36 operations each) with the row stage shared by the two tiles
# over a row segment and the inverse row stage applied once to the two tiles' summed columns:
# per 64x64 region 72 x 17 row DCTs + 289 tiles x (8 + 8) column transforms + 64 x 17 inverse row
# transforms = 249 k operations, 61 per pixel; the B = 16 block phase's 16-point butterflies
# (116 operations) forward and inverse over rows and columns = 29 per pixel. The reference's naive
# separable matrix form costs 394 FLOP per pixel.
IDA_FP32_OPS_PER_PX = 90
IDA_NAIVE_FLOP_PER_PX = 394


def ida_compute_view(pixels, avg_ms):
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz, src = float(json.load(f)["sm_max_mhz"]), "MEASURED_PEAKS.json sm_max_mhz"
    except (OSError, KeyError, ValueError):
        mhz, src = 1965.0, "B200 boost clock (fallback)"
    peak = 148 * 128 * mhz * 1e6 / 1e12  # fp32 lanes x clock: one FADD/FMUL/FFMA (FFMA2: two per 2 clk)
    ach = pixels * IDA_FP32_OPS_PER_PX / (avg_ms / 1e3) / 1e12
    return {"bound": "fp32 pipe (the kernel is latency/issue-bound below it)", "fp32_ops_per_px": IDA_FP32_OPS_PER_PX,
            "naive_flop_per_px_reference_form": IDA_NAIVE_FLOP_PER_PX,
            "achieved": round(ach, 2), "peak": round(peak, 2), "unit": "T fp32 op/s", "frac": round(ach / peak, 4),
            "peak_source": "148 SMs x 128 fp32 lanes x " + src}


def run_ida(p, torch, local, rank, hbm, world, dev):
    c = CFG4
    spec = p.SynthSpec(c["H"], c["W"], c["ellipses"], c["sigma"], c["seed"])
    first, cnt = shard(rank, c["n"])
    imgs = p.synth_images(spec, first, cnt, device=local)
    cfg = p.SensingConfig(c["B"], c["num"], c["den"], p.Algorithm.BBV)
    b = p.sense_batch(imgs, cfg)
    rc = p.ReconConfig(p.ReconMethod.Ida, iterations=c["iters"])
    out = torch.empty((c["n"], c["H"], c["W"]), dtype=torch.float32, device=dev)
    for _ in range(3):
        p.ida_batch(b, rc, out=out, trace=False, check=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    ctx = p.Context.get(local)
    s.record()  # the batch as a user runs it: init + 10 steps replayed as one CUDA graph
    for _ in range(reps):
        p.ida_batch(b, rc, out=out, trace=False, check=False)
    e.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(s.elapsed_time(e) / reps, world, dev)
    ctx.kernel_timing(True)  # per-kernel events on the launching stream (plain launches)
    for _ in range(reps):
        p.ida_batch(b, rc, out=out, trace=False, check=False)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.kernel_timing(False)
    N, K = c["H"] * c["W"], b.plan.coeffs_per_image
    per_iter = c["n"] * (8 * N + 12 * K)
    init = c["n"] * (8 * K + 4 * N)
    alg = per_iter * c["iters"] + init
    ach = alg / (ms / 1e3) / 1e9
    step_roof = None
    if "ida_step" in kt:  # the dominant kernel: one launch per iteration
        launches_k, total_ms, _ = kt["ida_step"]
        avg = total_ms / launches_k
        a_k = per_iter / (avg / 1e3) / 1e9
        tr = load_traffic().get("ida_step")
        step_roof = {"kernel": "ida_step (ida_mma_kernel<16>: fp32 FFMA2 denoiser + fp32 block phase)", "bound": "hbm",
                     "achieved": round(a_k, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(a_k / hbm, 4), "avg_launch_ms": round(avg, 4),
                     "algorithmic_bytes_per_launch": int(per_iter),
                     "traffic": round(tr["dram_bytes_per_image"] * c["n"]) if tr else None,
                     "share_of_batch": round(min(total_ms / reps / ms, 1.0), 4),
                     "compute_view": ida_compute_view(c["n"] * N, avg)}
    return {"metric": "IDA image-iterations/s (cfg4: 64 x 512^2, BBV 0.3, 10 it, dct_threshold)",
            "value": round(world * c["n"] * c["iters"] / (ms / 1e3), 1), "unit": "it/s",
            "mp_it_per_s": round(world * c["n"] * c["iters"] * N / (ms / 1e3) / 1e6, 1),
            "ms_per_batch": round(ms, 3),
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "algorithmic_bytes": int(alg)},
            "kernel_roofline": step_roof}


def spawn_ranks(args):
    """`bench.py --gpus N` without torchrun: one process per GPU on this node, RANK / LOCAL_RANK /
    WORLD_SIZE / MASTER_* set as torch.distributed.run would set them; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rcs = [pr.wait() for pr in procs]
    return max(rcs, key=abs)


def run_dry(args, world, rank):
    """--dry-run: the multi-rank plumbing without device work (CPU, gloo): each rank takes its shard
    of the global image indices, 'times' a stand-in step, and rank 0 prints the aggregate line."""
    import torch
    first, n = shard(rank, CFG2["n"])
    barrier(world)
    t0 = time.perf_counter()
    sample_images(1, dict(CFG2, H=64, W=64), first=first)  # a token of per-rank work on its own indices
    sec = max_over_ranks(time.perf_counter() - t0, world)
    firsts = [None] * world
    if world > 1:
        torch.distributed.all_gather_object(firsts, (first, n))
    else:
        firsts = [(first, n)]
    if rank == 0:
        px = len(SUBRATES) * n * CFG2["H"] * CFG2["W"]
        print(json.dumps({"metric": "megapixels/s for ABCS sense+reconstruct", "dry_run": True, "n_gpus": world,
                          "value": round(aggregate_rate(px, world, sec) / 1e6, 3), "unit": "MP/s",
                          "shards": firsts, "scaling": "weak"}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config-sweep", action="store_true", help="skip the cfg1/3/4/5 device sweep")
    ap.add_argument("--independent", action="store_true",
                    help="time one sense_decode_batch per subrate instead of the sweep call")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (no device work; gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return spawn_ranks(args)
    world, rank, local = dist_setup(args)
    try:
        if args.dry_run:
            return run_dry(args, world, rank)
        if args.impl == "reference":
            return run_reference(args, world, rank)
        return run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
