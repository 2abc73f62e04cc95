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
  e2e_per_batch  the reference's own call pattern: RocpStream::consume once per
           batch (rocp_stream_consume_host) on ordinary heap memory
  configs  device values of every BASELINE config (C1..C5) in the same run
--impl reference times the CPU port of the reference path (the oracle; the
reference itself needs Eigen3, absent here and on the GPU box) on all host
threads, on the SAME bytes: both arms build the tensor with synth_host() from
the same seed, run the same cprand init (bitwise identical on both sides) and
stream the same post-init batches with the same counter-RNG keys.
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


def synth_host(cfg, seed, threads=None):
    """[[A_1 .. A_N]] + Gaussian noise at the config's SNR (gen_synthetic semantics,
    synthetic.cpp:8-31: |noise| scaled after the draw so the SIR is exact), built on
    the host in a fixed chunking (deterministic for any thread count).  Returns the
    flat tensor (first index fastest), float64."""
    dims, R = cfg["dims"], cfg["rank"]
    g = np.random.default_rng(1000 + seed)
    truth = make_factors(dims, R, cfg["family"], g)
    kr = truth[-1]  # rows of modes 2..N, mode 2 fastest: kr[j] = prod_n A_n[i_n]
    for A in reversed(truth[1:-1]):
        kr = (kr[:, None, :] * A[None, :, :]).reshape(-1, R)
    n = int(np.prod(dims))
    x = np.empty(n)
    xm = x.reshape(kr.shape[0], dims[0])  # X_(1) column-major == (KR A_1^T) row-major
    step = max(1, kr.shape[0] // 64)
    for r0 in range(0, kr.shape[0], step):
        np.matmul(kr[r0:r0 + step], truth[0].T, out=xm[r0:r0 + step])
    del kr
    nchunk = 64
    bounds = [n * k // nchunk for k in range(nchunk + 1)]
    seeds = np.random.SeedSequence(5000 + seed).spawn(nchunk)
    sig2 = np.zeros(nchunk)
    e2 = np.zeros(nchunk)

    def pass1(k):
        lo, hi = bounds[k], bounds[k + 1]
        sig2[k] = float(np.dot(x[lo:hi], x[lo:hi]))
        e = np.random.Generator(np.random.PCG64(seeds[k])).standard_normal(hi - lo)
        e2[k] = float(np.dot(e, e))

    def run(fn):
        ths = threads or min(32, os.cpu_count() or 1)
        idx = list(range(nchunk))
        lock = threading.Lock()

        def worker():
            while True:
                with lock:
                    if not idx:
                        return
                    k = idx.pop(0)
                fn(k)
        ts = [threading.Thread(target=worker) for _ in range(ths)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    run(pass1)
    scale = np.sqrt(sig2.sum()) * 10.0 ** (-cfg["snr_db"] / 20.0) / np.sqrt(e2.sum())

    def pass2(k):  # the same noise chunks again, added at the exact-SIR scale
        lo, hi = bounds[k], bounds[k + 1]
        e = np.random.Generator(np.random.PCG64(seeds[k])).standard_normal(hi - lo)
        x[lo:hi] += scale * e
    run(pass2)
    return x


def init_factors(cfg, seed):
    """cprand's initial model (random_model's role), seeded; both arms use it."""
    g = np.random.default_rng(4000 + seed)
    dims = cfg["dims"][:-1] + [cfg["t_init"]]
    return [np.asfortranarray(g.standard_normal((d, cfg["rank"]))) for d in dims]


def config_dict(cfg, sharded=False, world=1, virtual_shards=8):
    """The `config` key both arms print (same workload, same step definition)."""
    d = cfg["dims"]
    nb = (d[-1] - cfg["t_init"]) // cfg["batch"]
    return {"workload": workload_text(cfg),
            "step": f"one full streaming pass ({nb} x RocpStream::consume) from the post-init state",
            "data_seed": 0, "stream_seeds": "10000 + step",
            "l2": f"inputs larger than L2 ({8 * int(np.prod(d)) / 1e9:.1f} GB tensor); fresh sampling seed every step",
            "parallelism": (f"one stream sharded along mode 1 over {world} GPU(s), {virtual_shards} virtual "
                            f"shards, exchange over peer memory" if sharded else
                            f"{world} independent stream replica(s), one per GPU (no collective)")}


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


def cpu_passes(init, cfg, x, seeds, threads):
    """Times full post-init stream passes of the oracle port (RocpStream::consume,
    rocp.cpp:144-160) on the host tensor x: `threads` independent streams (ROCP_THREADS
    semantics, reference bench.cpp:113-119), thread t replaying pass seeds[t::threads]
    from the post-init state.  Returns (slices, wall seconds)."""
    from oracle import oracle as orc

    dims, B, t_init = cfg["dims"], cfg["batch"], cfg["t_init"]
    nb = (dims[-1] - t_init) // B
    S = auto_s(cfg["rank"])
    slice_ = int(np.prod(dims[:-1]))
    counts = [0] * threads

    def worker(t):
        for seed in seeds[t::threads]:
            st = orc.Stream(init.model, t_init, init.best_sampled_kr, S, regularized=init.regularized)
            for b in range(nb):
                t0 = t_init + b * B
                st.consume(x[t0 * slice_:(t0 + B) * slice_], B, seed, b + 1)
            counts[t] += nb * B
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(t,)) for t in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return sum(counts), time.perf_counter() - t0


def reference_arm(args):
    """--impl reference: the CPU port of the reference path (oracle; Eigen3 is absent, so
    the reference itself cannot be built) on all host threads, same config and bytes."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    CFG = CONFIGS[args.config]
    dims, R, B, t_init = CFG["dims"], CFG["rank"], CFG["batch"], CFG["t_init"]
    nb = (dims[-1] - t_init) // B
    x = synth_host(CFG, 0)
    slice_ = int(np.prod(dims[:-1]))
    t0 = time.perf_counter()
    init = orc.cprand_decompose(x[:t_init * slice_], dims[:-1] + [t_init], R, init_factors(CFG, 0), seed=3000,
                                tol=CFG["tol"], max_iters=CFG["max_iters"])
    init_seconds = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    cpu_passes(init, CFG, x, [9000], 1)  # warm the port once
    for w in range(args.warmup - 1):
        cpu_passes(init, CFG, x, [9001 + w], 1)
    per_step = []
    for k in range(args.steps):  # step k: every thread streams the post-init batches with key 10000 + k
        n, wall = cpu_passes(init, CFG, x, [10000 + k] * threads, threads)
        per_step.append((n, wall))
    value = sum(n for n, _ in per_step) / sum(w for _, w in per_step)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "time-slices/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * statistics.mean(w for _, w in per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded {CFG['family']} factors, {CFG['snr_db']:g} dB Gaussian noise, built on the "
                f"host by synth_host: the same bytes as the GPU arm)",
        "config": config_dict(CFG),
        "same_config": True,
        "init_seconds": init_seconds, "init_sweeps": init.iterations, "init_fitness": init.best_fitness,
        "cpu_baseline": {"value": value, "unit": "time-slices/s", "cores": threads, "kind": "port",
                         "sample": f"oracle port of RocpStream::consume: per step {threads} threads each stream "
                                   f"the {nb} post-init batches ({nb * B} slices) from the cprand init"},
        "e2e": {"value": value, "unit": "time-slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_buildable": False,
        "note": "the reference needs Eigen3/doctest/CLI11 (absent here and on the GPU box); the timed path is "
                "the plain-C++ oracle port, pinned to the reference's own test vectors",
    }
    print(json.dumps(line), flush=True)


def gather_traffic(cfg_key, gather_sms):
    """ncu DRAM bytes (read + write) per launch of the window gather for this config,
    from profiles/ncu_gather_traffic.json (one capture per config); None when no
    capture matches the config and the split the step used."""
    prof = os.path.join(ROOT, "profiles", "ncu_gather_traffic.json")
    if not os.path.exists(prof):
        return None, None
    try:
        d = json.load(open(prof))
    except Exception:
        return None, None
    e = d.get("configs", {}).get(cfg_key)
    if not e or int(e.get("gather_sms", -1)) != int(gather_sms):
        return None, None
    return e.get("dram_bytes_per_launch"), e.get("source")


def device_config_run(rocp, dev, cfg, steps, warmup):
    """One BASELINE config on this device (device-generated data): cprand init, then
    `steps` timed full streaming passes (same step definition as the headline)."""
    dims, R, t_init, B = cfg["dims"], cfg["rank"], cfg["t_init"], cfg["batch"]
    nb = (dims[-1] - t_init) // B
    g = np.random.default_rng(1000)
    X = dev.tensor(dims)
    X.generate(make_factors(dims, R, cfg["family"], g), snr_db=cfg["snr_db"], noise_seed=2000)
    dev.synchronize()
    t0 = time.perf_counter()
    init = rocp.cprand_decompose(dev, X.slab(0, t_init), R, init_factors(cfg, 0), seed=3000, tol=cfg["tol"],
                                 max_iters=cfg["max_iters"])
    init_s = time.perf_counter() - t0
    st = rocp.RocpStream(dev, init, auto_s(R), t_capacity=dims[-1] + 8)
    st.checkpoint()
    for w in range(warmup):
        st.restore()
        st.consume_range(X, t_init, B, nb, 9000 + w, 1)
    dev.synchronize()
    dev.timer_record(6)
    for k in range(steps):
        st.restore()
        st.consume_range(X, t_init, B, nb, 10000 + k, 1)
    dev.timer_record(7)
    ms = dev.timer_elapsed_ms(6, 7)
    out = {"workload": workload_text(cfg), "value": steps * nb * B / (ms / 1000.0), "unit": "time-slices/s",
           "entries_per_s": steps * nb * B / (ms / 1000.0) * int(np.prod(dims[:-1])),
           "ms_per_step": ms / steps, "steps": steps, "init_seconds": init_s, "init_sweeps": init.iterations,
           "init_fitness": init.best_fitness, "gather_sms": st.last_gather_sms,
           "data": "device-generated (same semantics)"}
    st._free()
    X._free()
    dev.synchronize()
    return out


def multi_stream_run(rocp, cfg, K, steps, warmup, num_sms=148, chain_sms=0):
    """K independent streams of one config sharing the GPU, one handle (CUDA stream, scratch,
    tensor) each -- the reference's trial-level parallelism (bench.cpp:190-213, ROCP_THREADS; what
    the reference arm times on the host cores).  Every handle's persistent chain takes
    num_sms // K blocks (rocp_set_chain_sms), so the K cooperative chains are co-resident; the
    window gathers run serially per stream (several handles on one GPU) and overlap the other
    streams' chains.  Timed on the host around device synchronisations AND with CUDA events per
    handle; the slower of the two is reported."""
    dims, R, t_init, B = cfg["dims"], cfg["rank"], cfg["t_init"], cfg["batch"]
    nb = (dims[-1] - t_init) // B
    sms = chain_sms if chain_sms else max(16, num_sms // K)
    devs, Xs, sts = [], [], []
    for i in range(K):
        d = rocp.Device(0)
        d.set_chain_sms(sms)
        g = np.random.default_rng(1000 + i)
        X = d.tensor(dims)
        X.generate(make_factors(dims, R, cfg["family"], g), snr_db=cfg["snr_db"], noise_seed=2000 + i)
        init = rocp.cprand_decompose(d, X.slab(0, t_init), R, init_factors(cfg, i), seed=3000 + i, tol=cfg["tol"],
                                     max_iters=cfg["max_iters"])
        st = rocp.RocpStream(d, init, auto_s(R), t_capacity=dims[-1] + 8)
        st.checkpoint()
        devs.append(d)
        Xs.append(X)
        sts.append(st)
    for w in range(warmup):
        for i in range(K):
            sts[i].restore()
            sts[i].consume_range(Xs[i], t_init, B, nb, 9000 + w, 1)
    for d in devs:
        d.synchronize()
    t0 = time.perf_counter()
    for d in devs:
        d.timer_record(6)
    for k in range(steps):
        for i in range(K):
            sts[i].restore()
            sts[i].consume_range(Xs[i], t_init, B, nb, 10000 + k, 1)
    for d in devs:
        d.timer_record(7)
    for d in devs:
        d.synchronize()
    wall_ms = 1000.0 * (time.perf_counter() - t0)
    ev_ms = max(d.timer_elapsed_ms(6, 7) for d in devs)
    ms = max(wall_ms, ev_ms)
    out = {"streams": K, "chain_sms_per_stream": sms, "value": K * steps * nb * B / (ms / 1000.0),
           "unit": "time-slices/s", "steps": steps, "ms_per_round": ms / steps, "wall_ms": wall_ms,
           "event_ms_max": ev_ms,
           "note": "aggregate of K independent streams on one GPU (one handle each); the slower of host wall "
                   "time around device synchronisations and the per-handle CUDA-event time"}
    for st in sts:
        st._free()
    for X in Xs:
        X._free()
    for d in devs:
        d.synchronize()
        d.close()
    return out


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--device-data", action="store_true", help="generate the tensor on the device")
    ap.add_argument("--no-configs", action="store_true", help="skip the all-config device sweep")
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
    # ---- data: [[A1 .. AN]] + noise at the config's SNR.  Replicas: a different tensor
    # per rank; sharded: the same tensor on every rank.  Built on the host (synth_host,
    # the reference arm builds the same bytes) unless it is too large for a quick host
    # build (configs[3], 64 GB: generated on the device, same semantics).
    dseed = 0 if sharded else rank
    host_data = (not args.device_data) and int(np.prod(dims)) <= 4_500_000_000
    x_host = None
    if host_data:
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        x_host = synth_host(CFG, dseed, threads=max(1, (os.cpu_count() or 1) // max(1, local_world)))
        X = dev.tensor(dims, x_host)
    else:
        g = np.random.default_rng(1000 + dseed)
        X = dev.tensor(dims)
        X.generate(make_factors(dims, R, CFG["family"], g), snr_db=CFG["snr_db"], noise_seed=2000 + dseed)
    # ---- init: randomized CP-ALS on the first t_init slices (cprand.cpp:12-69)
    dev.synchronize()
    t0 = time.perf_counter()
    init = rocp.cprand_decompose(dev, X.slab(0, t_init), R, init_factors(CFG, dseed), seed=3000 + dseed,
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

    dev.decision_stats(reset=True)
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
    dec_stats = dev.decision_stats(reset=True)
    gather_ms = stream.gather_times()
    chain_ms = stream.chain_times()
    stream.time_gather(False)
    ms_max = max_over_ranks(ms, dist, torch)
    value = (1 if sharded else world) * args.steps * slices_per_step / (ms_max / 1000.0)

    # ---- roofline of the window gather: live, in the timed steps (where it may run
    # overlapped on a few SMs beside the chain), and the same kernel alone on every SM
    # (event-timed after the timed region, same window shape, fresh seeds)
    peak, peak_src = measured_peaks()
    sector_per_launch = nb * sector_bytes_per_batch(dims, S, B)
    useful_per_launch = nb * useful_bytes_per_batch(dims, S, B)
    strided_per_launch = nb * S * (B + sum(head[1:]))  # isolated 8-byte elements (own DRAM page each)
    g_avg_ms = statistics.mean(gather_ms) if gather_ms else None
    achieved = sector_per_launch / (g_avg_ms / 1000.0) / 1e9 if g_avg_ms else None
    gather_sms = stream.last_gather_sms if not sharded else 0
    standalone = None
    probe = None
    if not sharded:
        sa = [stream.gather_window(XS, t_init, B, nb, 50000 + k, 1, 0) for k in range(4)][1:]
        sa_ms = statistics.mean(sa)
        # the device's isolated random-read ceiling over the same tensor (k_probe_random_reads)
        rate, probe_ms = dev.probe_random_reads(XS, 1 << 26)
        probe = {"kernel": "k_probe_random_reads (8-byte loads at hashed offsets of the tensor, every SM)",
                 "reads_per_s": rate, "ms": probe_ms}
        standalone = {"kernel": "k_gather_warps on all SMs (nothing else running)", "avg_launch_ms": sa_ms,
                      "achieved": sector_per_launch / (sa_ms / 1000.0) / 1e9,
                      "frac": sector_per_launch / (sa_ms / 1000.0) / 1e9 / peak, "launches": len(sa),
                      "strided_elements_per_s": strided_per_launch / (sa_ms / 1000.0),
                      "access_rate": strided_per_launch / (sa_ms / 1000.0) / rate}
    traffic, traffic_src = gather_traffic(args.config, gather_sms)

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
        chain_name = ("k_flow (dataflow chain, no grid barriers)" if R <= 32 and os.environ.get("ROCP_CHAIN") != "barrier"
                      else "k_chain (grid-barrier chain" + (", streamed fp64-MMA pair items)" if R > 32 else ")"))
        chain_roof = {"kernel": chain_name + ": the persistent factor-dependent chain, one launch per window",
                      "bound": "latency (dependent Gauss-Seidel chain; fp64 pipe as the compute ceiling)",
                      "achieved": flops / (c_avg / 1000.0) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                      "frac": flops / (c_avg / 1000.0) / 1e12 / fp64_peak,
                      "peak_source": "derived: 148 SMs x 64 fp64 FMA/clk x 2 x 1.965 GHz",
                      "algorithmic_flops_per_launch": flops, "avg_launch_ms": c_avg,
                      "share_of_step": sum(chain_ms) / ms, "launches": len(chain_ms)}

    # ---- e2e through the host-slab call: the caller's slabs stay in (pinned) host memory;
    # only the sampled fibres cross PCIe (host gather), the model is read back every step
    e2e = e2e_pb = None
    slice_ = int(np.prod(head))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    host_threads = max(1, (os.cpu_count() or 1) // max(1, local_world))
    if not args.no_e2e and args.e2e_steps > 0 and not sharded:
        hbuf = rocp.HostBuffer(slices_per_step * slice_)  # pinned, 2 MB pages (rocp_host_alloc)
        host = hbuf.array
        if x_host is not None:
            np.copyto(host, x_host[t_init * slice_:(t_init + nb * B) * slice_])
        else:
            X.slab(t_init, slices_per_step).download(out=host)
        stream.restore()  # warm the host-slab path once
        stream.consume_range_host(host, B, nb, 777, 1, threads=host_threads)
        dev.synchronize()
        e2e_ms = []
        for k in range(args.e2e_steps):
            stream.restore()
            dev.timer_record(2)
            stream.consume_range_host(host, B, nb, 10000 + k, 1, threads=host_threads)
            out = stream.model()  # device -> host read of the step's result
            dev.timer_record(3)
            e2e_ms.append(dev.timer_elapsed_ms(2, 3))
        e2e_ms_max = max_over_ranks(max(e2e_ms), dist, torch)
        xs_elems = nb * sum(((I + 31) // 32) * 32 * S for I in [B] + head)  # row-tiled X_s per window
        e2e = {"value": world * slices_per_step / ((statistics.mean(e2e_ms) if world == 1 else e2e_ms_max) / 1000.0),
               "unit": "time-slices/s",
               "h2d_bytes_per_step": int(xs_elems * 8),
               "d2h_bytes_per_step": int(sum(m.size for m in out) * 8 + nb * len(dims) * S * 8),
               "steps": args.e2e_steps, "ms_per_step": statistics.mean(e2e_ms),
               "ms_min": min(e2e_ms), "ms_max": max(e2e_ms), "host_threads_per_rank": host_threads,
               "path": "rocp_stream_consume_range_host on a rocp_host_alloc range: host draw -> host threads "
                       "gather the strided sampled fibres, the GPU reads the mode-1 fibres in place (zero-copy) "
                       "-> H2D of X_s per batch on a copy stream -> persistent chain per batch"}
        hbuf.free()
        # RocpStream::consume once per batch on ordinary (pageable) memory: the reference's call
        # pattern (rocp.cpp:144-160, bench.cpp:50-59), rocp_stream_consume_host per batch
        src = x_host if x_host is not None else None
        if src is None:
            src = X.slab(t_init, slices_per_step).download()
            base = 0
        else:
            base = t_init * slice_
        slabs = [src[base + b * B * slice_: base + (b + 1) * B * slice_] for b in range(nb)]
        for rep in range(2):  # warm
            stream.restore()
            for b in range(nb):
                stream.consume(slabs[b], 777 + rep, b + 1)
        dev.synchronize()
        pb_ms = []
        for k in range(args.e2e_steps):
            stream.restore()
            dev.timer_record(4)
            for b in range(nb):
                stream.consume(slabs[b], 10000 + k, b + 1)
            out = stream.model()
            dev.timer_record(5)
            pb_ms.append(dev.timer_elapsed_ms(4, 5))
        e2e_pb = {"value": slices_per_step / (statistics.mean(pb_ms) / 1000.0), "unit": "time-slices/s",
                  "steps": args.e2e_steps, "ms_per_step": statistics.mean(pb_ms), "ms_per_batch":
                  statistics.mean(pb_ms) / nb, "host_threads_per_rank": host_threads,
                  "path": f"RocpStream::consume per batch ({nb} calls of rocp_stream_consume_host on pageable "
                          f"numpy slabs of {B} slices), model read back after the pass"}

    # ---- CPU baseline (rank 0, bounded sample): the oracle port, 1 thread, full post-init passes
    # over the same bytes from the same (bitwise identical) init
    cpu = None
    if rank == 0 and not args.no_cpu and not sharded:
        src = x_host if x_host is not None else X.download()
        seeds, n_sl, wall = [], 0, 0.0
        while wall < args.cpu_seconds and len(seeds) < 1000:
            n, w = cpu_passes(init, CFG, src, [10000 + len(seeds)], 1)
            seeds.append(0)
            n_sl += n
            wall += w
        cpu = {"value": n_sl / wall, "unit": "time-slices/s", "cores": 1, "kind": "port",
               "sample": f"oracle port of RocpStream::consume, 1 thread: {len(seeds)} full post-init passes "
                         f"({nb} batches of {B}) of {CFG['name']} from the same init ({n_sl} slices in {wall:.1f} s)"}

    # ---- every BASELINE config on this device (device-generated data), same metric
    configs_line = None
    if rank == 0 and world == 1 and not sharded and not args.no_configs:
        configs_line = {}
        for key in sorted(CONFIGS):
            if key == args.config:
                configs_line[key] = {"value": value, "ms_per_step": ms_max / args.steps,
                                     "init_seconds": init_seconds, "gather_sms": gather_sms}
                continue
            configs_line[key] = device_config_run(rocp, dev, CONFIGS[key], steps=3, warmup=3)

    # ---- K independent streams sharing this GPU (the reference arm's shape: independent streams
    # on all host threads), a secondary key beside the single-stream headline
    multi = None
    if rank == 0 and world == 1 and not sharded and not args.no_configs and int(np.prod(dims)) * 8 <= 9e9:
        multi = multi_stream_run(rocp, CFG, 4, steps=5, warmup=3, chain_sms=30)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "time-slices/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": (f"synthetic (seeded {CFG['family']} factors, {CFG['snr_db']:g} dB Gaussian noise, built on "
                     f"the host by synth_host and uploaded: the bytes the reference arm streams)" if host_data else
                     f"synthetic (seeded {CFG['family']} factors, {CFG['snr_db']:g} dB Gaussian noise, generated "
                     f"on the device)"),
            "config": config_dict(CFG, sharded, world, args.virtual_shards),
            "entries_per_s": value * int(np.prod(head)),
            "init_seconds": init_seconds, "init_sweeps": init.iterations, "init_fitness": init.best_fitness,
            "gpu_launches": launches,
            "gram_decisions": {"counts": dec_stats, "keys": ["no_reg", "reg", "exact_eigen", "tier2_used"],
                               "note": "solve_gram regularisation decisions since init (DESIGN.md 3.4)"},
            "roofline": {"kernel": ("k_gather_warps (window sampled-fibre gather, TMA boxes), overlapped on "
                                    f"{gather_sms} SMs beside the persistent chain" if gather_sms else
                                    "k_gather (window sampled-fibre gather, every SM, before the chain)"),
                         "bound": "hbm", "sms": gather_sms or 148,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                         "strided_elements_per_launch": strided_per_launch,
                         "random_read_ceiling": probe,
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
            "e2e_per_batch": e2e_pb,
            "cpu_baseline": cpu,
            "configs": configs_line,
            "multi_stream": multi,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
