#!/usr/bin/env python
"""Benchmark: log-polar FBP of 2048^2 slices (BASELINE.json metric
"backprojected 2048^2 slices/sec at 1/2/4/8 B200; HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--slices S] [--scaling strong|weak] [--e2e-slices E]

One process per GPU (torchrun for N > 1).  A step is one pass of the FBP hot
path over the rank's resident slices.  Default workload: configs[3], the
2048-slice volume of 2048 angles x 2048 bins, sharded by slice index over the N
ranks (strong scaling: rank r takes the contiguous block bench.shard(2048, N, r),
seeds = global slice index); --scaling weak gives every rank S slices of its own.
There is no inter-GPU data exchange: torch.distributed carries only the barrier,
the max-over-ranks timing and the shard bookkeeping.  Inputs (>= 4 GB per rank
at N = 8) are far larger than L2, so no L2 flush is needed between steps.

--config 4 times the direct pixel-driven backprojector on the 64 config-2 slices.

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/fastbp_oracle.py: numpy/scipy restatement of fastbp) on the
host's cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "backprojected 2048^2 slices/sec at 1/2/4/8 B200; HBM GB/s vs peak"
try:
    MEASURED = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
except (OSError, ValueError):
    MEASURED = {}
# dram__bytes_read.sum + dram__bytes_write.sum per slice and kernel, from the committed ncu
# --set full capture named in profiles/traffic.json; used only when that capture was taken
# on the same kernel sources (sha256 of paper_1608_03589_b200/csrc), else reported as null
TRAFFIC_FILE = os.path.join(REPO, "profiles", "traffic.json")


def load_traffic(engine: str):
    """(per-slice DRAM bytes by kernel, provenance) of the committed capture for `engine`."""
    from paper_1608_03589_b200 import roofline
    try:
        t = json.load(open(TRAFFIC_FILE))[engine]
    except (OSError, ValueError, KeyError):
        return None, {"source": None, "note": "no committed capture"}
    here = roofline.kernel_source_digest()
    prov = {"source": t.get("capture"), "csrc_sha256": t.get("csrc_sha256"), "current_csrc_sha256": here}
    if t.get("csrc_sha256") != here:
        prov["note"] = "capture predates the current kernel sources: traffic not reported"
        return None, prov
    return t["per_slice"], prov


UNIT = "slices/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--slices", type=int, default=0, help="slices per rank per step (0 = config default)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="slices per internal pipeline chunk (0 = 256 for the power-of-two log-polar path (one stream), "
                         "16 for generic sizes and bst: the measured bests)")
    ap.add_argument("--e2e-slices", type=int, default=512)
    ap.add_argument("--e2e-chunk", type=int, default=4)
    ap.add_argument("--streams", type=int, default=0,
                    help="CUDA streams the device-resident chunks alternate on (0 = 1; 2 for the fused mixed-radix path; bst 1: "
                         "two BST chunks in flight halve the L2 its gridding gathers hit)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = min(cores, memory/2.5GB, 32)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--geometry", default="",
                    help="NTxNTHETA: the config's phantoms and output size at another sinogram shape, e.g. 3200x2048 "
                         "(the paper's LNLS datasets, PAPER.md:151-153)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's volume (2048 slices for config 3) is sharded by slice index "
                         "over the ranks; weak: every rank processes --slices (or the config's count) of its own")
    ap.add_argument("--engine", default="logpolar", choices=["logpolar", "bst"],
                    help="logpolar (the north-star path, default) or bst (fbp's default engine in the reference)")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# distributed plumbing (barrier + max over ranks; no data-path collective)
# ----------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo")
            self.pg = dist

    def cuda_index(self) -> int:
        """This rank's GPU: LOCAL_RANK, wrapped onto the visible devices.  On a box with fewer GPUs
        than local ranks (functional checks of the N > 1 path only) ranks share a device and the
        line says so in run.shared_device; such a run is not a scaling measurement."""
        import torch

        nd = torch.cuda.device_count()
        self.shared_device = nd < int(os.environ.get("LOCAL_WORLD_SIZE", str(self.world)))
        if self.shared_device:
            print(f"[bench] rank {self.rank}: {nd} visible GPU(s) for the local ranks: devices are shared "
                  "(functional check, not a scaling number)", file=sys.stderr)
        return self.local % max(nd, 1)

    def bind_numa(self, cuda_index: int) -> str:
        """N > 1: pin this rank's process to the host cores local to its GPU (the PCI device's
        local_cpulist in sysfs), so the pinned buffers of the e2e leg are allocated on the GPU's own
        socket and every rank's H2D / D2H stays off the inter-socket link.  Returns what was done."""
        if self.world <= 1 or getattr(self, "shared_device", False):
            return "not bound (one rank)" if self.world <= 1 else "not bound (ranks share a device)"
        try:
            import torch

            pr = torch.cuda.get_device_properties(cuda_index)
            dev = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            with open(f"/sys/bus/pci/devices/{dev}/local_cpulist") as f:
                spec = f.read().strip()
            cpus = set()
            for part in spec.split(","):
                if part:
                    lo, _, hi = part.partition("-")
                    cpus.update(range(int(lo), int(hi or lo) + 1))
            cpus &= os.sched_getaffinity(0)
            if cpus:
                os.sched_setaffinity(0, cpus)
                return f"{len(cpus)} cores local to GPU {dev} (sysfs local_cpulist)"
            return "not bound (no local cores in this process's set)"
        except Exception as e:  # no sysfs entry: leave the scheduler's placement
            return f"not bound ({type(e).__name__})"

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj) -> list:
        """Every rank's `obj`, in rank order (host-side bookkeeping only)."""
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def shard(total: int, world: int, rank: int) -> range:
    """Contiguous slice-index block of `rank`."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return range(lo, hi)


def rank_slices(total: int, world: int, rank: int, scaling: str) -> list[int]:
    """Global slice indices rank `rank` reconstructs (their per-slice seeds make the inputs).
    strong: the `total`-slice volume split into contiguous blocks; weak:
    `total` slices per rank, rank r taking [r total, (r + 1) total)."""
    if scaling == "strong":
        return list(shard(total, world, rank))
    return list(range(rank * total, (rank + 1) * total))


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, path: str | None):
        self.gpu, self.path, self.proc = gpu, path, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]
            if self.path:
                with open(self.path, "w") as f:
                    f.write(self.Q + "\n" + "\n".join(self.lines) + "\n")

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------
# CPU baseline (oracle port of the reference algorithm), one slice per worker
# ----------------------------------------------------------------------------
def _cpu_worker_many(jobs):
    """Generate every input first (untimed), then time each reconstruction."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import fastbp_oracle as O
    from oracle import phantoms

    inputs = [(c, phantoms.sinogram(phantoms.config_seed(cfg, idx), c["nt"], c["ntheta"], c["k"], c["amin"],
                                    c["amax"], c["noise"]).astype("float64"), eng)
              for cfg, c, idx, eng in jobs]
    times = []
    for c, g, eng in inputs:
        t = time.perf_counter()
        if eng == "bst":
            O.fbp_bst(g, c["n"]) if c["fbp"] else O.bst_backproject(g, c["n"])
        elif c["fbp"]:
            O.fbp_logpolar(g, c["n"])
        else:
            O.logpolar_backproject(g, c["n"])
        times.append(time.perf_counter() - t)
    return times


def cpu_workers(requested: int) -> int:
    if requested > 0:
        return requested
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    try:
        avail_gb = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) / 1e6
    except Exception:
        avail_gb = 16.0
    return max(1, min(ncpu, int(avail_gb / 2.5), 32))


def cpu_baseline(cfg: int, workers: int, slices_per_worker: int = 1, engine: str = "logpolar", c: dict | None = None):
    """Throughput of the oracle port on `workers` host cores: one process per core,
    all running concurrently, each reconstructing whole slices.  Only the
    reconstruction is timed (each worker generates its input first, untimed):
    throughput = slices / (longest per-worker reconstruction time)."""
    env = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}
    os.environ.update(env)
    if c is None:
        from oracle import phantoms
        c = phantoms.CONFIGS[cfg]
    jobs = [[(cfg, c, 1000 + w * slices_per_worker + i, engine) for i in range(slices_per_worker)]
            for w in range(workers)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        per = pool.map(_cpu_worker_many, jobs, chunksize=1)
    busy = max(sum(p) for p in per)
    flat = [t for p in per for t in p]
    return workers * slices_per_worker / busy, busy, flat


def cpu_model() -> str:
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------
def workload_name(config: int, c: dict) -> str:
    """The workload string both arms report (the driver pairs the lines on it)."""
    tag = f"config{config}" + (" phantoms" if c.get("geometry") else "")
    return f"{tag}: {'FBP' if c['fbp'] else 'BP'} {c['nt']} bins x {c['ntheta']} angles -> {c['n']}^2"


def workload_config(a, c: dict, world: int, geom: dict, chunk: int, nstreams: int) -> dict:
    """The line's `config`: identical in both arms for the same command line (the driver pairs the
    lines on it).  Everything here follows from the arguments, the world size and the plan geometry
    `geom` = {nrho, L, nphi}; what depends on the box (host binding, ranks sharing a device) is
    reported under `run` instead."""
    total = a.slices or c["slices"]
    ranks = [rank_slices(total, world, r, a.scaling) for r in range(world)]
    S = len(ranks[0])
    return {"workload": workload_name(a.config, c), "slices_total": sum(len(r) for r in ranks),
            "slices_per_rank": S, "rank_slice_ranges": [[r[0], r[-1] + 1] if r else [0, 0] for r in ranks],
            "chunk": min(chunk, S), "streams": nstreams,
            "parallelism": f"slice-shard x{world} ({a.scaling} scaling, no inter-GPU exchange)",
            "l2": f"no flush: {S * c['nt'] * c['ntheta'] * 4 / 1e9:.1f} GB of sinograms per rank per step "
                  f">> 126 MB L2",
            "nrho": int(geom["nrho"]), "L": int(geom["L"]), "nphi": int(geom["nphi"])}


def default_schedule(a, generic: bool, unfused: bool, bst: bool = False) -> tuple[int, int]:
    """(chunk, streams) of the device-resident leg.  Power-of-two log-polar path: ONE stream, chunks of
    256 slices (a 32.8 GB workspace; with K2p, r02n: chunk 128 / 256 / 512 -> 9576 / 9630 / 9649 slices/s).
    Measured at 2048^2 before K2p (B200, r02l): 1 stream x chunk 32 / 64 / 128 -> 8689 / 8820 / 8874
    slices/s, 2 streams x chunk 32 / 64 -> 8987 / 8937.  Two streams buy 1.3 % by overlapping kernel
    tails, but every launch then shares the SMs with the other stream's kernel, so the live per-launch
    durations the roofline is built from double (K3 0.155 of the HBM peak live against 0.242 alone) and
    the kernels' live shares of the step stop matching the serialised ncu launch list.  One stream
    keeps the timed region, the live roofline and the ncu evidence the same thing; `--streams 2
    --chunk 32` is the throughput-best schedule.  With K3's K-hat column held in TMEM per CTA, longer
    launches amortise each CTA's prologue and the launches' tails.  A generic-size plan whose inverse
    DFT + readout stay unfused (Bluestein lengths, odd nt: through an HBM log-polar image) also runs
    on one stream, like BST: two chunks in flight halve the L2 the readout's gathers hit (LNLS before
    its fused path: 3175 slices/s on one stream, 2373 on two); the fused mixed-radix path takes two
    streams (LNLS: 4800 vs 4596); generic plans take chunks of 16."""
    chunk = a.chunk if a.chunk > 0 else (16 if (bst or generic) else 256)
    nstreams = a.streams if a.streams > 0 else (1 if (bst or unfused or not generic) else 2)
    return chunk, nstreams


def bench_config(a) -> dict:
    """The config's workload, with --geometry NTxNTHETA overriding the sinogram shape."""
    from oracle import phantoms
    c = dict(phantoms.CONFIGS[a.config])
    if a.geometry:
        nt, nth = (int(v) for v in a.geometry.lower().split("x"))
        c.update(nt=nt, ntheta=nth, geometry=a.geometry)
    return c


def run_reference(a, d: Dist):
    """--impl reference: the reference algorithm on the host cores, rank 0 only."""
    if d.rank != 0:
        d.close()
        return
    from oracle import phantoms

    c = bench_config(a)
    # the plan geometry our arm reports in `config`, restated from the oracle's mesh rule (no GPU here)
    from oracle import fastbp_oracle as fo
    _, _, nr, _ = fo.lp_geometry(c["nt"], c["n"])
    nphi = 2 * c["ntheta"]
    geom = {"nrho": nr, "L": 1 << (2 * nr - 2).bit_length(), "nphi": nphi}
    pow2 = nphi & (nphi - 1) == 0 and 512 <= nphi <= 4096 and c["nt"] % 4 == 0
    generic, fused = not pow2, nphi in (6400, 1536, 2560, 4608, 3072, 5120)
    workers = cpu_workers(a.cpu_workers)
    vals = []
    for i in range(a.warmup + a.steps):
        v, busy, _ = cpu_baseline(a.config, workers, 1, c=c)
        if i >= a.warmup:
            vals.append((v, busy))
    v = sum(x for x, _ in vals) / len(vals)
    ms = sum(w for _, w in vals) / len(vals) * 1000.0
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded random-ellipse sinograms + 1% Gaussian noise)",
        "config": workload_config(a, c, a.gpus, geom, *default_schedule(a, generic, generic and not fused)),
        "run": {"slices_per_step": workers},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"{workers} slices per step, one per concurrent worker process, reconstruction "
                                   f"only (inputs generated untimed), oracle/fastbp_oracle.py (numpy/scipy "
                                   f"restatement of fastbp), CPU {cpu_model()}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    d.close()


def copy_ceiling(host_in, host_out, chunk: int, steps: int, d: Dist) -> float:
    """Slices/s that PCIe alone allows for the e2e traffic on this box: the same pinned
    buffers and chunking, H2D on one stream and D2H on another, no compute."""
    import torch
    E = host_in.shape[0]
    din = torch.empty((2, chunk) + tuple(host_in.shape[1:]), dtype=torch.float32, device="cuda")
    dout = torch.empty((2, chunk) + tuple(host_out.shape[1:]), dtype=torch.float32, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def once():
        for i, k in enumerate(range(0, E, chunk)):
            m = min(chunk, E - k)
            with torch.cuda.stream(s_in):
                din[i & 1, :m].copy_(host_in[k:k + m], non_blocking=True)
            with torch.cuda.stream(s_out):
                host_out[k:k + m].copy_(dout[i & 1, :m], non_blocking=True)
        torch.cuda.synchronize()

    once()
    d.barrier()
    t = time.perf_counter()
    for _ in range(steps):
        once()
    return d.sum(E * steps) / d.max(time.perf_counter() - t)


def run_ours(a, d: Dist):
    import numpy as np
    import torch

    import paper_1608_03589_b200 as p

    ci = d.cuda_index()
    torch.cuda.set_device(ci)
    dev = torch.device("cuda", ci)
    numa = d.bind_numa(ci)
    c = bench_config(a)
    nt, nth, n = c["nt"], c["ntheta"], c["n"]
    total = a.slices or c["slices"]
    spec = (0.0, 1.0) if c["fbp"] else None
    bst = a.engine == "bst"
    plan = p.BstPlan(nt, nth, p.BstOptions(n_out=n), spec) if bst else p.get_plan(nt, nth, n, None, None, spec)

    # ---- synthetic inputs, generated on the device (per-slice seeds = global slice index)
    global_ids = rank_slices(total, d.world, d.rank, a.scaling)
    S = len(global_ids)
    shards = d.gather([global_ids[0], global_ids[-1] + 1] if global_ids else [0, 0])
    sino = p.synth.config_batch(a.config, global_ids, dev, geometry=(nt, nth))
    out = torch.empty((S, n, n), dtype=torch.float32, device=dev)
    info = {} if bst else plan.info
    generic = bool(info.get("generic", 0))
    unfused = generic and not (info.get("phi_q", 0) > 0 and info.get("band_rows", 0) == 2)
    chunk, nstreams = default_schedule(a, generic, unfused, bst)
    chunk = min(chunk, S)
    # one workspace per stream: the plan is immutable, chunks on different streams overlap
    wss = [None if bst else torch.empty(plan.workspace_bytes(chunk), dtype=torch.uint8, device=dev)
           for _ in range(nstreams)]

    def run(x, o, ws):
        if bst:
            plan.execute(x, out=o, chunk=chunk)
        else:
            plan.execute(x, out=o, workspace=ws)
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    main = torch.cuda.current_stream(dev)

    def step():
        n_l = 0
        for st in streams:
            st.wait_stream(main)
        for i, k in enumerate(range(0, S, chunk)):
            with torch.cuda.stream(streams[i % nstreams]):
                run(sino[k:k + chunk], out[k:k + chunk], wss[i % nstreams])
            n_l += plan.last_launches
        for st in streams:
            main.wait_stream(st)
        return n_l

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    clk = ClockSampler(d.local, os.path.join(REPO, "gpurun_out", f"clocks_rank{d.rank}.csv"))
    d.barrier()
    torch.cuda.synchronize()
    stream = main
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    # CUDA events around every kernel launch, on its launching stream, during the timed steps
    # (lpbp_profile_*): the roofline's per-launch durations are measured live
    plan.profile(True)
    with clk:
        time.sleep(0.3)
        e0.record(stream)
        for _ in range(a.steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize()
    stages = plan.profile_read()
    plan.profile(False)
    d.barrier()
    # the same kernels once more in isolation (one stream, no overlap), for the per-stage split
    plan.profile(True)
    for k in range(0, S, chunk):
        run(sino[k:k + chunk], out[k:k + chunk], wss[0])
    torch.cuda.synchronize()
    iso = plan.profile_read()
    plan.profile(False)
    ms_total = e0.elapsed_time(e1)
    ms_max = d.max(ms_total)
    total_slices = d.sum(S * a.steps)
    value = total_slices / (ms_max / 1000.0)

    # ---- roofline of the dominant kernel (largest share of device time)
    info = plan.info
    ab = p.roofline.bst_algorithmic_bytes(plan) if bst else p.algorithmic_bytes(plan)
    dom = max(stages, key=lambda k: stages[k]["ms"])
    st = stages[dom]
    per_launch_ms = st["ms"] / max(1, st["launches"])
    slices_per_launch = st["slices"] / max(1, st["launches"])
    own_bytes_per_launch = ab[dom]["per_slice"] * slices_per_launch + ab[dom]["per_launch"]
    # the roofline's algorithmic bytes: SURVEY §8(d)'s figure of the stage this kernel computes (the
    # task's definition); this decomposition's own compulsory bytes are reported beside it
    sv = None if bst else p.roofline.survey_stage_bytes(plan).get(dom)
    bytes_per_launch = (sv["per_slice"] * slices_per_launch + sv["per_launch"]) if sv else own_bytes_per_launch
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    achieved = bytes_per_launch / (per_launch_ms / 1000.0) / 1e9
    flops = p.roofline.bst_nominal_flops(plan) if bst else p.roofline.nominal_flops(plan)
    fp_ach = flops.get(dom, 0.0) * slices_per_launch / (per_launch_ms / 1000.0) / 1e12
    fp_peak = p.roofline.fp32_peak_tflops(float(MEASURED.get("sm_max_mhz", 1965.0)))
    tr_table, tr_prov = load_traffic("bst" if bst else "logpolar")
    traffic = (tr_table or {}).get(dom)
    traffic = traffic * slices_per_launch if traffic else None
    pipe_bytes = sum(ab[k]["per_slice"] for k in ab if k in stages) + sum(
        ab[k]["per_launch"] * stages[k]["launches"] for k in stages) / max(1, S * a.steps)
    survey_bytes = None if bst else p.roofline.survey_bytes_per_slice(plan)
    share_live = st["ms"] / max(1e-9, sum(v["ms"] for v in stages.values()))
    iso_dom = iso.get(dom, {"ms": 0.0, "launches": 1, "slices": 1})
    iso_ms = iso_dom["ms"] / max(1, iso_dom["launches"])

    # ---- end to end through the public host API (pinned host in/out, H2D + D2H inside)
    E = min(a.e2e_slices, S)
    host_in = torch.empty((E, nt, nth), dtype=torch.float32, pin_memory=True)
    host_in.copy_(sino[:E])
    host_out = torch.empty((E, n, n), dtype=torch.float32, pin_memory=True)
    hin, hout = (host_in.numpy(), host_out.numpy()) if bst else (host_in, host_out)
    plan.execute_host(hin, hout, chunk=a.e2e_chunk)
    d.barrier()
    t = time.perf_counter()
    for _ in range(a.e2e_steps):
        plan.execute_host(hin, hout, chunk=a.e2e_chunk)
    e2e_s = d.max(time.perf_counter() - t)
    e2e_value = d.sum(E * a.e2e_steps) / e2e_s
    copy_value = copy_ceiling(host_in, host_out, a.e2e_chunk, a.e2e_steps, d)

    cpu = None
    if d.rank == 0 and a.gpus == 1 and not a.no_cpu_baseline:
        w = cpu_workers(a.cpu_workers)
        v, busy, per = cpu_baseline(a.config, w, 1, a.engine, c=c)
        cpu = {"value": v, "unit": UNIT, "cores": w, "kind": "port",
               "sample": f"{w} config-{a.config} slices, one per concurrent worker process (reconstruction only, "
                         f"slowest worker {busy:.1f} s, mean {np.mean(per):.2f} s/slice/core), "
                         f"oracle/fastbp_oracle.py ({'fbp_bst' if bst else 'fbp_logpolar'}), CPU {cpu_model()}"}

    slices_total = int(d.sum(S))  # a collective: every rank takes part
    assert slices_total == sum(hi - lo for lo, hi in shards), (slices_total, shards)
    if d.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": d.world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (device-generated seeded random-ellipse sinograms, K=50, 1% Gaussian noise)",
            "config": dict(workload_config(a, c, d.world, info if not bst else {"nrho": 0, "L": info["L"], "nphi": 0},
                                           chunk, nstreams),
                           **({"workload": workload_name(a.config, c) + " (BST engine)", "engine": "bst",
                               "big": info["big"], "m_need": info["m_need"]} if bst else {})),
            "run": dict({"rank_slice_ranges_gathered": shards},
                        **({"shared_device": True} if getattr(d, "shared_device", False) else {}),
                        **({"host_binding": numa} if d.world > 1 else {})),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": per_launch_ms,
                         "basis": (f"SURVEY 8(d) stage {sv['stage']}: {sv['per_slice'] / 1e6:.3f} MB per slice"
                                   + (f" + {sv['per_launch'] / 1e6:.1f} MB K-hat per launch" if sv["per_launch"] else "")
                                   + f", {slices_per_launch:.0f} slices per launch") if sv else "own decomposition",
                         "own_decomposition": {
                             "bytes_per_launch": own_bytes_per_launch,
                             "frac": own_bytes_per_launch / (per_launch_ms / 1000.0) / 1e9 / peak,
                             "note": "what this kernel itself must move: K3 reads the semi-polar row spectra "
                                     "(nh x ns complex) and interpolates the log-polar column on chip, so the "
                                     "log-polar image S3 would read never crosses HBM; `traffic` is to be "
                                     "compared with this figure"},
                         "timing": f"CUDA events on the launching stream around each of the {st['launches']} "
                                   f"launches inside the timed steps ({nstreams} streams overlap)",
                         "share_of_step_live": share_live,
                         "isolated_launch_ms": iso_ms,
                         "isolated_frac": bytes_per_launch / (iso_ms / 1000.0) / 1e9 / peak if iso_ms else None,
                         "traffic_provenance": tr_prov,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                         "fp32_pipe": {"achieved_tflops": fp_ach, "peak_tflops": fp_peak, "frac": fp_ach / fp_peak,
                                       "note": "nominal FFT flops (5 N log2 N) of the kernel / launch time vs "
                                               "148 SMs x 128 lanes x 2 x clock; FFT stages are FP32-pipe bound"}},
            "pipeline": {"stage_ms_per_slice_live": {k: v["ms"] / max(1, v["slices"]) for k, v in stages.items()},
                         "stage_ms_per_slice_isolated": {k: v["ms"] / max(1, v["slices"]) for k, v in iso.items()},
                         "algorithmic_bytes_per_slice": pipe_bytes,
                         "hbm_equiv_gbs": pipe_bytes * value / d.world / 1e9,
                         "hbm_equiv_frac": pipe_bytes * value / d.world / 1e9 / peak,
                         "survey_bytes_per_slice": survey_bytes,
                         "survey_hbm_equiv_frac": (survey_bytes * value / d.world / 1e9 / peak) if survey_bytes
                         else None,
                         "survey_basis": "SURVEY §8(d) stage decomposition (S1+S2+S3+S4, K-hat once per batch)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": E * nt * nth * 4,
                    "d2h_bytes_per_step": E * n * n * 4, "slices_per_step": E,
                    "api": "BstPlan.execute_host" if bst else "LogPolarPlan.execute_host",
                    "copy_ceiling": copy_value, "frac_of_copy_ceiling": e2e_value / copy_value,
                    "copy_ceiling_note": "same bytes, same chunking, H2D and D2H alone on two streams, no compute, "
                                         "all ranks at once (so at N > 1 it is the shared host-DRAM / PCIe ceiling)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    d.close()


def run_direct(a, d: Dist):
    """configs[4]: the direct pixel-driven backprojector (the accuracy cross-check),
    timed on the config-2 inputs (64 slices per rank) and compared with the log-polar
    path on the same slices."""
    import numpy as np
    import torch

    import paper_1608_03589_b200 as p

    ci = d.cuda_index()
    torch.cuda.set_device(ci)
    dev = torch.device("cuda", ci)
    c = p.synth.CONFIGS[4]
    S = a.slices or c["slices"]
    n, nt, nth = c["n"], c["nt"], c["ntheta"]
    ids = list(range(d.rank * S, (d.rank + 1) * S))
    x = p.synth.config_batch(4, ids, dev)
    out = torch.empty((S, n, n), dtype=torch.float32, device=dev)
    from ctypes import byref, c_size_t, c_void_p
    lib = p._native.lib()
    nbytes = c_size_t()
    p._native.check(lib.lpbp_naive_workspace_bytes(nt, nth, S, byref(nbytes)))
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        p._native.check(lib.lpbp_naive_backproject(c_void_p(x.data_ptr()), c_void_p(out.data_ptr()), nt, nth, n, S,
                                                   c_void_p(ws.data_ptr()), c_void_p(stream.cuda_stream)))
        return int(lib.lpbp_last_launch_count())

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(d.local, None)
    d.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with clk:
        time.sleep(0.2)
        e0.record(stream)
        for _ in range(a.steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = d.max(e0.elapsed_time(e1))
    nv = out
    lp = p.logpolar_backproject_batch(x, n)
    xs = -1.0 + (np.arange(n) + 0.5) * (2.0 / n)
    X, Y = np.meshgrid(xs, xs)
    disk = torch.from_numpy(np.hypot(X, Y) <= 1.0).to(dev)
    gap = ((lp - nv)[:, disk].double().norm() / nv[:, disk].double().norm()).item()
    full = ((lp - nv).double().norm() / nv.double().norm()).item()
    # e2e through the public API: host sinograms in, host images out (one slice group per call)
    E = min(S, 8)
    host_in = x[:E].cpu().pin_memory()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(max(1, a.steps // 2)):
        img = p.backproject_naive_batch(host_in.to(dev, non_blocking=True), n).cpu()
    e2e = E * max(1, a.steps // 2) / (time.perf_counter() - t)
    value = d.sum(S * a.steps) / (ms / 1e3)
    lerps = value * n * n * nth
    clock = clk.summary()
    mhz = clock["sm_mhz"] or float(MEASURED.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    per_clk_sm = lerps / d.world / (nsm * mhz * 1e6)
    if d.rank == 0:
        print(json.dumps({
            "metric": "direct (pixel-driven) backprojected 2048^2 slices/sec", "value": value, "unit": UNIT,
            "n_gpus": d.world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (config-2 seeds: the same 64 slices configs[4] names)",
            "config": {"workload": f"config4: direct BP {nt} bins x {nth} angles -> {n}^2", "slices_per_rank": S,
                       "l2": "no flush: 1.1 GB of sinograms per step >> 126 MB L2"},
            "ms_per_slice": ms / a.steps / S,
            "lerps_per_s": lerps,
            "roofline": {"bound": "shared-memory gathers",
                         "achieved_lerps_per_clk_sm": per_clk_sm, "peak_lerps_per_clk_sm": 16.0,
                         "frac": per_clk_sm / 16.0,
                         "note": "each lerp needs two 4-byte samples; shared memory serves 128 B/clk/SM, "
                                 "so 16 lerps/clk/SM bounds any gather-based direct backprojector",
                         "fp32_pipe": {"flops_per_lerp": 4, "achieved_tflops": lerps * 4 / d.world / 1e12,
                                       "peak_tflops": p.roofline.fp32_peak_tflops(mhz),
                                       "frac": lerps * 4 / d.world / 1e12 / p.roofline.fp32_peak_tflops(mhz)}},
            "lp_vs_direct_rel_l2": {"unit_disk": gap, "full_image": full, "slices": S},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": E * nt * nth * 4,
                    "d2h_bytes_per_step": E * n * n * 4, "api": "backproject_naive_batch"},
            "gpu_launches": launches, "clocks": clock}), flush=True)
    d.close()


def main():
    a = parse()
    d = Dist()
    if a.impl == "reference":
        run_reference(a, d)
    elif a.config == 4:
        run_direct(a, d)
    else:
        run_ours(a, d)


if __name__ == "__main__":
    main()
