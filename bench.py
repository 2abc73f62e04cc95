#!/usr/bin/env python
"""bench.py -- ROCP streaming throughput on B200 (BASELINE.json configs[1]).

Workload (configs[1]): 3-way fp64 tensor 1000 x 1000 x 1000, CP rank R = 20,
factors iid N(0,1), Gaussian noise at SNR 20 dB, randomized CP-ALS init on the
first 100 slices (reference defaults tol 1e-4, <= 100 sweeps), then the
remaining 900 slices streamed in batches of 25 (36 batches), S = 600 samples
per mode.  One "step" = one full pass of the online update over the 900
streamed slices from the post-init state (RocpStream::consume x 36,
reference rocp.cpp:144-160), with a fresh sampling seed every step.

Reported (one JSON line on rank 0):
  value    time slices/s with the tensor resident in HBM (device-timed with
           CUDA events over K steps; max over ranks for N > 1)
  e2e      the same metric through the reference-facing host-slab call
           (rocp_stream_consume_range_host): every step starts from the 900
           slices in host memory (a rocp_host_alloc buffer), moves the
           sampled fibres to the device and reads the model back
  roofline the window gather kernel (sampled-fibre gather, north-star item 1):
           algorithmic sector bytes per launch / its average
           CUDA-event launch time in the timed region, vs MEASURED_PEAKS.json.
           In a step it runs overlapped on a few SMs beside the chain (`sms`);
           `standalone` is the same launch on every SM, timed after the region
  cpu_baseline  the CPU oracle port (single thread) on a bounded sample of the
           same stream
--impl reference times the CPU port of the reference path on all host threads.
"""
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

METRIC = "ROCP time-slices/sec and sampled-gather HBM GB/s vs B200 peak"
# BASELINE.json configs (C1..C5); the default bench line is configs[1].
CONFIGS = {
    "c1": dict(name="configs[0]", dims=[200, 200, 500], rank=10, t_init=50, batch=10, snr_db=20.0,
               tol=1e-6, max_iters=20, family="normal"),
    "c2": dict(name="configs[1]", dims=[1000, 1000, 1000], rank=20, t_init=100, batch=25, snr_db=20.0,
               tol=1e-4, max_iters=100, family="normal"),
    "c3": dict(name="configs[2]", dims=[200, 200, 200, 200], rank=10, t_init=20, batch=10, snr_db=30.0,
               tol=1e-4, max_iters=100, family="uniform"),
    "c4": dict(name="configs[3]", dims=[4000, 4000, 500], rank=50, t_init=50, batch=50, snr_db=20.0,
               tol=1e-4, max_iters=100, family="normal"),
    "c5": dict(name="configs[4]", dims=[60, 60, 60, 60, 300], rank=16, t_init=10, batch=10, snr_db=10.0,
               tol=1e-4, max_iters=100, family="congruent"),
}
CFG = CONFIGS["c2"]


def make_factors(dims, R, family, g):
    """Seeded factors of the config's family: iid N(0,1), iid U(0,1), or pairwise
    column congruence 0.9 (G L^T, L = chol(0.9 11^T + 0.1 I))."""
    if family == "uniform":
        return [np.asfortranarray(g.random((d, R))) for d in dims]
    if family == "congruent":
        L = np.linalg.cholesky(np.full((R, R), 0.9) + 0.1 * np.eye(R))
        return [np.asfortranarray(g.standard_normal((d, R)) @ L.T) for d in dims]
    return [np.asfortranarray(g.standard_normal((d, R))) for d in dims]


def workload_text(cfg):
    d = cfg["dims"]
    nb = (d[-1] - cfg["t_init"]) // cfg["batch"]
    return (f"{cfg['name']}: {'x'.join(map(str, d))} fp64, R={cfg['rank']}, init {cfg['t_init']} slices "
            f"(cprand tol {cfg['tol']:g}, <= {cfg['max_iters']} sweeps), stream {nb * cfg['batch']} slices in "
            f"{nb} batches of {cfg['batch']}, S={auto_s(cfg['rank'])}")


def sector_bytes_per_batch(dims, S, B):
    """8*S*I1 + 32*S*(B + sum_{2<=n<N} I_n) (mode-1 fibres 32-B aligned,
    every other gathered element its own 32-B sector)."""
    return 8 * S * dims[0] + 32 * S * (B + sum(dims[1:-1]))


def useful_bytes_per_batch(dims, S, B):
    return 8 * S * (B + sum(dims[:-1]))


def auto_s(R):
    return max(R, int(np.ceil(10.0 * R * np.log(R))))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        time.sleep(0.15)
        self.lines = []
        if self.proc:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for k, n in enumerate(names):
                if len(f) > 2 + k and f[2 + k].lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        # one GPU per rank; more ranks than GPUs only in the functional check below (replicas share)
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        # ROCP_BENCH_BACKEND=gloo: exercise the multi-rank plumbing (barrier, max over ranks)
        # where NCCL cannot run, e.g. two replica ranks sharing one GPU in a functional check
        dist.init_process_group(os.environ.get("ROCP_BENCH_BACKEND", "nccl"))
        return world, rank, local, dist, torch
    return world, rank, local, None, None


def max_over_ranks(v, dist, torch):
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# --------------------------------------------------------------------------- CPU port
def cpu_sample_stream(model_head, best_kr, R, S, t_init, head, slabs, B, budget_s, threads=1):
    """Times the oracle port's consume (rocp.cpp:144-160) on host slabs:
    `threads` independent streams (ROCP_THREADS semantics, reference
    bench.cpp:113-119), each repeating the sample until budget_s elapses."""
    from oracle import oracle as orc

    temporal0 = np.zeros((t_init, R), order="F")
    counts = [0] * threads

    def worker(k):
        st = orc.Stream(list(model_head) + [temporal0], t_init, best_kr, S)
        t_end = time.perf_counter() + budget_s
        bid = 1
        while time.perf_counter() < t_end:
            for x in slabs:
                st.consume(x, B, 1234 + k, bid)
                bid += 1
                counts[k] += B
                if st.t_len > t_init + 100000:
                    break
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(k,)) for k in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    return sum(counts) / wall, sum(counts), wall


def reference_arm(args):
    """--impl reference: the CPU port of the reference path on all host threads."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    CFG = CONFIGS[args.config]
    dims, R, B = CFG["dims"], CFG["rank"], CFG["batch"]
    S = auto_s(R)
    head = dims[:-1]
    g = np.random.default_rng(0)
    from oracle import oracle as orc
    A = make_factors(head, R, CFG["family"], g)
    nslab = 4 if int(np.prod(head)) * B <= 50_000_000 else 2
    slabs = []
    for k in range(nslab):  # [[A_1 .. A_{N-1}, a_t]] + noise at the config's SNR (gen_synthetic semantics)
        a_t = make_factors([B], R, CFG["family"], g)[0]
        x = orc.reconstruct(A + [a_t], head + [B])
        e = g.standard_normal(x.size)
        x += np.linalg.norm(x) * 10 ** (-CFG["snr_db"] / 20) / np.linalg.norm(e) * e
        slabs.append(np.ascontiguousarray(x))
    kr = []
    for n in range(1, len(dims)):
        _, dec = orc.draw_samples(head + [CFG["t_init"]], n, S, 7, 0, 0)
        temporal = np.asfortranarray(g.standard_normal((CFG["t_init"], R)))
        kr.append(orc.sampled_khatri_rao(dec, orc.factors_excluding(A + [temporal], n)))
    threads = os.cpu_count() or 1
    per_step = []
    for _ in range(args.warmup):
        cpu_sample_stream(A, kr, R, S, CFG["t_init"], head, slabs[:1], B, 0.0, threads=1)
    budget = float(os.environ.get("ROCP_REF_STEP_SECONDS", "8"))
    for _ in range(args.steps):
        v, n, wall = cpu_sample_stream(A, kr, R, S, CFG["t_init"], head, slabs, B, budget, threads)
        per_step.append((v, n, wall))
    value = sum(n for _, n, _ in per_step) / sum(w for _, _, w in per_step)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "time-slices/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * statistics.mean(w for _, _, w in per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_text(CFG),
                   "sample": f"{nslab} synthetic batches of {B} slices repeated for {budget:.0f} s per step "
                             f"on each of {threads} threads (independent streams, ROCP_THREADS semantics)"},
        "cpu_baseline": {"value": value, "unit": "time-slices/s", "cores": threads, "kind": "port",
                         "sample": f"oracle port of RocpStream::consume on {nslab} x {B}-slice slabs, "
                                   f"{threads} threads x {budget:.0f} s per step"},
        "e2e": {"value": value, "unit": "time-slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_buildable": False,
        "note": "reference needs Eigen3/doctest/CLI11 (absent); timed path is the plain-C++ oracle port",
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="BASELINE.json config (c2 = configs[1], the headline workload)")
    ap.add_argument("--sharded", action="store_true",
                    help="one stream sharded along mode 1 across the N GPUs (NCCL exchange; strong "
                         "scaling, north star for configs[3]/[4]) instead of N independent replicas")
    ap.add_argument("--virtual-shards", type=int, default=8)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)

    import paper_2007_10798_b200 as rocp

    world, rank, local, dist, torch = dist_setup()
    CFG = CONFIGS[args.config]
    dims, R, t_init, B = CFG["dims"], CFG["rank"], CFG["t_init"], CFG["batch"]
    head = dims[:-1]
    S = auto_s(R)
    T = dims[-1]
    nb = (T - t_init) // B
    slices_per_step = nb * B

    sharded = args.sharded
    if sharded and world > 1:  # NCCL bootstrap id from rank 0 over the torch process group
        box = [rocp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        dev = rocp.Device(local, world, rank, box[0])
    else:
        dev = rocp.Device(local)
    # ---- data: [[A1 .. AN]] + noise at the config's SNR, generated on the device
    # (replicas: a different tensor per rank; sharded: the same tensor on every rank)
    dseed = 0 if sharded else rank
    g = np.random.default_rng(1000 + dseed)
    truth = make_factors(dims, R, CFG["family"], g)
    X = dev.tensor(dims)
    X.generate(truth, snr_db=CFG["snr_db"], noise_seed=2000 + dseed)
    # ---- init: randomized CP-ALS on the first t_init slices (cprand.cpp:12-69)
    init0 = [np.asfortranarray(g.standard_normal((d, R))) for d in head + [t_init]]
    dev.synchronize()
    t0 = time.perf_counter()
    init = rocp.cprand_decompose(dev, X.slab(0, t_init), R, init0, seed=3000 + dseed,
                                 tol=CFG["tol"], max_iters=CFG["max_iters"])
    init_seconds = time.perf_counter() - t0
    stream = rocp.RocpStream(dev, init, S, t_capacity=T + 8)
    XS = X
    if sharded:  # this rank keeps rows [r0, r1) of mode 1
        r0, r1 = stream.shard(args.virtual_shards)
        XS = X.rows(r0, r1)
        X._free()
        X = None
    stream.checkpoint()

    def step(seed):
        stream.restore()
        stream.consume_range(XS, t_init, B, nb, seed, 1)

    for w in range(args.warmup):
        step(9000 + w)
    dev.synchronize()
    # ---- timed region (device events, barrier + sync both sides)
    stream.time_gather(True)
    barrier(dist)
    dev.synchronize()
    l0 = dev.kernel_launches
    with ClockSampler(local) as clk:
        dev.timer_record(0)
        for k in range(args.steps):
            step(10000 + k)
        dev.timer_record(1)
        ms = dev.timer_elapsed_ms(0, 1)
    dev.synchronize()
    barrier(dist)
    launches = dev.kernel_launches - l0
    gather_ms = stream.gather_times()
    chain_ms = stream.chain_times()
    stream.time_gather(False)
    ms_max = max_over_ranks(ms, dist, torch)
    value = (1 if sharded else world) * args.steps * slices_per_step / (ms_max / 1000.0)
    fit_model = stream.model()

    # ---- roofline of the window gather: live, in the timed steps (where it may run
    # overlapped on a few SMs beside the chain), and the same kernel alone on every SM
    # (event-timed after the timed region, same window shape, fresh seeds)
    peak, peak_src = measured_peaks()
    sector_per_launch = nb * sector_bytes_per_batch(dims, S, B)
    useful_per_launch = nb * useful_bytes_per_batch(dims, S, B)
    g_avg_ms = statistics.mean(gather_ms) if gather_ms else None
    achieved = sector_per_launch / (g_avg_ms / 1000.0) / 1e9 if g_avg_ms else None
    gather_sms = stream.last_gather_sms if not sharded else 0
    standalone = None
    if not sharded:
        sa = [stream.gather_window(XS, t_init, B, nb, 50000 + k, 1, 0) for k in range(4)][1:]
        sa_ms = statistics.mean(sa)
        standalone = {"kernel": "k_gather_warps on all SMs (nothing else running)", "avg_launch_ms": sa_ms,
                      "achieved": sector_per_launch / (sa_ms / 1000.0) / 1e9,
                      "frac": sector_per_launch / (sa_ms / 1000.0) / 1e9 / peak, "launches": len(sa)}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gather_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- secondary roofline: the persistent chain (K3-K6), latency-bound by design
    # (SURVEY.md 8d): algorithmic fp64 flops per launch (contraction 2 S R (B + sum I)
    # + Gram S R (R+1) per stage, per batch) over its CUDA-event launch time, against
    # the fp64 CUDA-core peak derived from the SM count and max clock (not in
    # MEASURED_PEAKS.json): SMs x 64 FMA/clk x 2 x clock.
    chain_roof = None
    if chain_ms:
        flops = nb * (2 * S * R * (B + sum(head)) + len(dims) * S * R * (R + 1))
        c_avg = statistics.mean(chain_ms)
        fp64_peak = 148 * 64 * 2 * 1.965e9 / 1e12
        chain_roof = {"kernel": "k_chain (persistent factor-dependent chain, one launch per window)",
                      "bound": "latency (dependent Gauss-Seidel chain; fp64 pipe as the compute ceiling)",
                      "achieved": flops / (c_avg / 1000.0) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                      "frac": flops / (c_avg / 1000.0) / 1e12 / fp64_peak,
                      "peak_source": "derived: 148 SMs x 64 fp64 FMA/clk x 2 x 1.965 GHz",
                      "algorithmic_flops_per_launch": flops, "avg_launch_ms": c_avg,
                      "share_of_step": sum(chain_ms) / ms, "launches": len(chain_ms)}

    # ---- e2e through the host-slab call: the caller's slabs stay in (pinned) host memory;
    # only the sampled fibres cross PCIe (host gather), the model is read back every step
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0 and not sharded:
        slice_ = int(np.prod(head))
        hbuf = rocp.HostBuffer(slices_per_step * slice_)  # pinned, 2 MB pages (rocp_host_alloc)
        host = hbuf.array
        X.slab(t_init, slices_per_step).download(out=host)
        # replicas share the host: each rank's gather pool takes its share of the cores
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        host_threads = max(1, (os.cpu_count() or 1) // max(1, local_world))
        stream.restore()  # warm the host-slab path once
        stream.consume_range_host(host, B, nb, 777, 1, threads=host_threads)
        dev.synchronize()
        e2e_ms = []
        for k in range(args.e2e_steps):
            stream.restore()
            dev.timer_record(2)
            stream.consume_range_host(host, B, nb, 20000 + k, 1, threads=host_threads)
            out = stream.model()  # device -> host read of the step's result
            dev.timer_record(3)
            e2e_ms.append(dev.timer_elapsed_ms(2, 3))
        e2e_ms_max = max_over_ranks(max(e2e_ms), dist, torch)
        xs_elems = nb * sum(((I + 31) // 32) * 32 * S for I in [B] + head)  # row-tiled X_s per window
        e2e = {"value": world * slices_per_step / ((statistics.mean(e2e_ms) if world == 1 else e2e_ms_max) / 1000.0),
               "unit": "time-slices/s",
               "h2d_bytes_per_step": int(xs_elems * 8),
               "d2h_bytes_per_step": int(sum(m.size for m in out) * 8 + nb * len(dims) * S * 8),
               "steps": args.e2e_steps, "ms_per_step": statistics.mean(e2e_ms), "host_threads_per_rank": host_threads,
               "path": "rocp_stream_consume_range_host: device draw -> host threads gather the strided "
                       "sampled fibres, the GPU reads the mode-1 fibres in place (zero-copy) -> H2D of "
                       "X_s per batch on a copy stream -> persistent chain per batch"}

    # ---- CPU baseline (rank 0, bounded sample)
    cpu = None
    if rank == 0 and not args.no_cpu and not sharded:
        slice_ = int(np.prod(head))
        xs = XS.slab(t_init, 4 * B).download() if not sharded else None
        slabs = [np.ascontiguousarray(xs[k * B * slice_:(k + 1) * B * slice_]) for k in range(4)]
        v, n, wall = cpu_sample_stream(init.model[:-1], init.best_sampled_kr, R, S, t_init, head, slabs, B,
                                       args.cpu_seconds, threads=1)
        cpu = {"value": v, "unit": "time-slices/s", "cores": 1, "kind": "port",
               "sample": f"oracle port of RocpStream::consume, 1 thread, first 4 streamed batches of "
                         f"{CFG['name']} repeated ({n} slices in {wall:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "time-slices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": f"synthetic (seeded {CFG['family']} factors, {CFG['snr_db']:g} dB Gaussian noise, "
                    f"generated on device)",
            "config": {"workload": workload_text(CFG),
                       "step": f"one full streaming pass ({nb} x RocpStream::consume) from the post-init state",
                       "l2": f"inputs larger than L2 ({8 * int(np.prod(dims)) / 1e9:.1f} GB tensor); "
                             f"fresh sampling seed every step",
                       "parallelism": (f"one stream sharded along mode 1 over {world} GPU(s), "
                                       f"{args.virtual_shards} virtual shards, NCCL all-gather of partials"
                                       if sharded else
                                       f"{world} independent stream replica(s), one per GPU (no collective)")},
            "entries_per_s": value * int(np.prod(head)),
            "init_seconds": init_seconds, "init_sweeps": init.iterations, "init_fitness": init.best_fitness,
            "gpu_launches": launches,
            "roofline": {"kernel": ("k_gather_warps (window sampled-fibre gather, TMA boxes), overlapped on "
                                    f"{gather_sms} SMs beside k_chain" if gather_sms else
                                    "k_gather (window sampled-fibre gather, every SM, before the chain)"),
                         "bound": "hbm", "sms": gather_sms or 148,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": sector_per_launch,
                         "useful_bytes_per_launch": useful_per_launch,
                         "avg_launch_ms": g_avg_ms, "launches": len(gather_ms),
                         "share_of_step": (sum(gather_ms) / ms) if gather_ms else None,
                         "note": ("in the step the gather runs on a few SMs concurrently with the chain "
                                  "(off the critical path); standalone = the same launch on every SM"
                                  if gather_sms else "serial gather before the chain"),
                         "standalone": standalone},
            "roofline_chain": chain_roof,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
