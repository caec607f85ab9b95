"""Benchmark: threshold-RHG edges/s on B200 (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX] [--impl ours|reference]

A "step" is one full stats-only generation (generator.hpp:219-291) of the
workload: host layout, device sampler, cell index, every edge kernel, the
counter all-reduce (N > 1) and the counters back on the host.

Workloads (BASELINE.json configs, SURVEY 8(d) chunk counts P):
  N = 1: cfg2 (configs[1], n=2^24, d=64, gamma=2.2, seed=7, P=64) -- the 1-B200 config.
  N > 1: cfg3 (configs[2], n=2^26, d=256, gamma=3, seed=11, P=512) -- strong scaling;
         --config cfg4 is the weak-scaling line (n = 2^28 N, P = 4096 N, d=4, seed=13).
  With N > 1 and no WORLD_SIZE in the environment, bench.py re-launches itself under
  torchrun with N ranks (one per GPU; fewer visible GPUs is an error).  Each rank owns
  engines [r P/N, (r+1) P/N), regenerates its halo from the seeds, and every step ends
  with ONE device-side ncclAllReduce(uint64) of the (edges, fingerprint, comps) counters
  inside the library (rhg_attach_comm), on the timed stream.

value = whole-graph edges per step x K / (max over ranks of the summed per-step device
time: CUDA events on the library's stream).  e2e = the same metric through the public
API call (host layout + table upload + kernels + all-reduce + counter readback), host
wall clock, max over ranks.  --impl reference times the reference's own CPU generator
(oracle/_ref, the unmodified reference headers compiled in place) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges/sec (device-timed, max over ranks) at 1/2/4/8 B200; % of FP64 roofline"
UNIT = "edges/s"

# name: (n, avg degree, gamma, seed, chunks, weak) -- weak: n and P scale with the GPU count
CONFIGS = {
    "cfg1": (1 << 20, 16.0, 3.0, 1, 8, False),
    "cfg2": (1 << 24, 64.0, 2.2, 7, 64, False),
    "cfg3": (1 << 26, 256.0, 3.0, 11, 512, False),
    "cfg4": (1 << 28, 4.0, 3.0, 13, 4096, True),
    "cfg5": (1 << 30, 16.0, 2.6, 17, 2048, False),
}
GOLDEN_NAME = {"cfg1": "cfg1", "cfg2": "cfg2", "cfg3": "cfg3", "cfg5": "cfg5"}


def workload(name, world):
    n, d, g, seed, P, weak = CONFIGS[name]
    if weak:
        n, P = n * world, P * world
    return n, d, g, seed, P, weak


def golden_row(name, n, P):
    """The reference's (edges, fingerprint, comps) for this workload, from the goldens the
    reference produced (tests/golden/stats.json, make_golden.py)."""
    try:
        rows = json.load(open(os.path.join(ROOT, "tests", "golden", "stats.json")))
    except (OSError, ValueError):
        return None
    for s in rows:
        if s["n"] == n and s["P"] == P and s["name"].startswith(name):
            return s
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def kernel_profile():
    """Pipe / L1 / issue utilisation of the slab join from the committed ncu summary."""
    for p in (os.path.join(ROOT, "profiles", "r02", "ncu_kernels_cfg2.json"),
              os.path.join(ROOT, "profiles", "r01", "ncu_kernels_cfg2_latest.json")):
        try:
            rows = [k for k in json.load(open(p)) if "slab_kernel" in k.get("kernel", "")]
        except (OSError, ValueError):
            continue
        if not rows:
            continue
        keys = {"fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "fp32_fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
                "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active"}
        out = {"source": os.path.relpath(p, ROOT) + " (ncu --set full, the slab launches of a step)"}
        for name, key in keys.items():
            vals = []
            for r in rows:
                try:
                    vals.append(float(str(r.get(key, "")).split()[0]))
                except (ValueError, IndexError):
                    pass
            out[name] = round(sum(vals) / len(vals), 1) if vals else None
        out["bound"] = ("latency/issue: the FP32 pre-filter replaced the FP64 predicate for 99.9% of the pairs "
                        "(exact FP64 recheck near the threshold), so the FP64 pipe is not the limit")
        return out
    return None


def traffic_from_profile():
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary."""
    for p in (os.path.join(ROOT, "profiles", "r02", "roofline_traffic.json"),
              os.path.join(ROOT, "profiles", "roofline_traffic.json")):
        try:
            return json.load(open(p))
        except (OSError, ValueError):
            continue
    return None


def cpu_reference_run(n, d, g, seed, P, threads=0):
    """The reference's generate_stats on the host cores (oracle/_ref)."""
    from oracle.refbind import Ref
    ref = Ref()
    alpha = ref.alpha_from_gamma(g)
    C = ref.radial_const_from_avg_degree(d, alpha)
    t = time.perf_counter()
    st = ref.generate_stats(n, alpha, C, seed, P, threads)
    return st, time.perf_counter() - t


def workload_config(name, wl, world):
    n, d, g, seed, P, weak = wl
    return {"workload": f"{name}: threshold RHG n={n}, avg degree {d:g}, gamma {g}, seed {seed}, chunks P={P}"
                        + (f" (weak scaling: 2^28 points and 4096 chunks per GPU)" if weak else ""),
            "n": n, "avg_degree": d, "gamma": g, "seed": seed, "chunks": P, "parallelism": f"chunk-shard x{world}",
            "l2": "inputs larger than L2: every step regenerates the full point set (~64 B/point in HBM)"}


def parity_block(name, wl, result, cpu_result=None):
    n, P = wl[0], wl[4]
    g = golden_row(name, n, P)
    out = {}
    if g is not None:
        want = {"edges": g["edges"], "fingerprint": g["fingerprint"], "comps": g["comps"]}
        out["golden"] = {"source": f"tests/golden/stats.json row {g['name']} (the reference run by make_golden.py)",
                         "expected": want, "equal": all(result[k] == want[k] for k in want)}
    if cpu_result is not None:
        out["cpu_baseline_equal"] = all(result[k] == cpu_result[k] for k in ("edges", "fingerprint", "comps"))
    out["equal"] = all(v["equal"] if isinstance(v, dict) else v for v in out.values()) if out else None
    return out


def run_reference(args, name, wl, world, rank):
    if rank != 0:
        return 0
    n, d, g, seed, P, _ = wl
    cores = os.cpu_count() or 1
    budget_s = float(os.environ.get("RHG_REF_BUDGET_S", "150"))
    st, wall = cpu_reference_run(n, d, g, seed, P)  # warm-up (page cache, thread pool); one is enough on a CPU
    secs, steps_run = [], 0
    t_start = time.perf_counter()
    for _ in range(args.steps):
        st, wall = cpu_reference_run(n, d, g, seed, P)
        secs.append(st["seconds"])
        steps_run += 1
        if time.perf_counter() - t_start + st["seconds"] > budget_s:
            break
    v = st["edges"] * len(secs) / sum(secs)
    result = {"edges": st["edges"], "fingerprint": st["fingerprint"], "comps": st["comps"]}
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
            "scaling": "weak" if wl[5] else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded model sampler)", "config": workload_config(name, wl, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "cpu": cpu_model(), "kind": "reference",
                             "sample": f"full {name} graph per step (RunStats.seconds), GenOptions.workers = "
                                       f"hardware_concurrency; {steps_run} of {args.steps} steps timed "
                                       f"(budget {budget_s:.0f} s), median {statistics.median(secs):.3f} s"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "result": result, "parity": parity_block(name, wl, result)}
    print(json.dumps(line), flush=True)
    return 0


# SURVEY 8(d) per-point figures (the cost at small average degree is per point): HBM bytes per
# sampled point that the pipeline's passes must move (DESIGN 8): radius uniforms 8 + radius
# attributes 40 + beta 8 (sampler), beta cells 28 + rank / scatter 128 + lambda cells 12 (sort
# phase), slab staging 32 + own-window (beta, hw) 16 (sparse engine)
DESIGN_BYTES_PER_POINT = 8 + 40 + 8 + 28 + 128 + 12 + 32 + 16


def per_point_block(params, rank, world, step_ms, sample_ms):
    import paper_1710_07565_b200 as rhg
    pts = rhg.shard_extent(params, rank, world).sampled_points
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        pass
    gbs = pts * DESIGN_BYTES_PER_POINT / (step_ms * 1e-3) / 1e9 if step_ms > 0 else 0.0
    return {"points_sampled_per_rank": pts,
            "points_per_s": pts / (step_ms * 1e-3) if step_ms > 0 else 0.0,
            "sampler_points_per_s": pts / (sample_ms * 1e-3) if sample_ms > 0 else 0.0,
            "design_hbm_bytes_per_point": DESIGN_BYTES_PER_POINT,
            "design_hbm_GBps": gbs,
            "hbm_peak_GBps": peak, "hbm_frac": gbs / peak if peak else None,
            "note": "rank 0's shard; sampler rate over the main stream's sampler phase (chains + radius side)"}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """--gpus N without torchrun: re-launch under torchrun, one rank per GPU."""
    one_gpu = os.environ.get("RHG_BENCH_ONE_GPU") == "1"
    if args.impl == "ours" and not one_gpu:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr,
                  flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: cfg2 at --gpus 1, cfg3 (strong scaling) at --gpus > 1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        return 2
    name = args.config or ("cfg2" if world == 1 else "cfg3")
    wl = workload(name, world)
    if args.impl == "reference":
        return run_reference(args, name, wl, world, rank)

    import torch
    import torch.distributed as dist
    import paper_1710_07565_b200 as rhg

    # RHG_BENCH_ONE_GPU=1: functional check of the N-rank path on a 1-GPU box (every rank on
    # cuda:0; NCCL cannot put two ranks on one GPU, so the counters go through gloo in Python);
    # its timings are not scaling numbers
    one_gpu = os.environ.get("RHG_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            # the library's own communicator: rank 0's NCCL id, broadcast over the torch group
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(rhg.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            rhg.attach_comm(world, rank, bytes(uid.cpu().numpy().tobytes()), device=local)
    n, d, g, seed, P, weak = wl
    params = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    opts = rhg.GenOptions(device=local, rank=rank, world=world)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_1710_07565_b200.distributed import ShardResult, reduce_shards

    def step():
        st = rhg.generate_stats(params, opts)
        if world > 1 and one_gpu:  # the per-step counter reduction (gloo stands in for the device collective)
            gr = reduce_shards(ShardResult(st.total.edges, st.total.fingerprint, st.total.comps), device="cpu")
            st.total.edges, st.total.fingerprint, st.total.comps = gr.edges, gr.fingerprint, gr.comps
        return st

    for _ in range(args.warmup):
        step()
    barrier()
    dev_ms, wall_s, launches, h2d, d2h, edges_ms, pairs_ms, stream_comps = 0.0, 0.0, 0, 0, 0, 0.0, 0.0, 0
    sample_ms = 0.0
    with Clocks(local) as clk:
        for _ in range(args.steps):
            t = time.perf_counter()
            st = step()
            wall_s += time.perf_counter() - t
            dev_ms += st.device_ms
            edges_ms += st.edges_ms
            sample_ms += st.sample_ms
            pairs_ms += st.pairs_ms
            stream_comps += st.stream_comps
            launches += st.kernel_launches
            h2d += st.h2d_bytes
            d2h += st.d2h_bytes
    barrier()
    edges, fp, comps = st.total.edges, st.total.fingerprint, st.total.comps  # whole graph (reduced every step)
    # the sparse engine alone (untimed, after the timed region): the edge phase on one stream, so its
    # kernels do not share the SMs with the dense engine / global unit / tail as in the timed steps
    iso_ms, iso_tests = 0.0, 0
    if rank == 0 and world == 1:
        saved = {k: os.environ.get(k) for k in ("RHG_CONCURRENT_ENGINES", "RHG_SIDE_SMALL")}
        os.environ["RHG_CONCURRENT_ENGINES"], os.environ["RHG_SIDE_SMALL"] = "0", "0"
        try:
            for _ in range(3):
                si = step()
                iso_ms += si.pairs_ms
                iso_tests += si.stream_comps
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    tm = torch.tensor([dev_ms, wall_s, edges_ms], dtype=torch.float64, device="cpu" if one_gpu else "cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    dev_ms, wall_s, edges_ms = float(tm[0]), float(tm[1]), float(tm[2])
    value = edges * args.steps / (dev_ms * 1e-3)
    e2e = edges * args.steps / wall_s
    if rank == 0:
        ops, lat, _ = rhg.fp64_peak(local)
        # algorithmic FP64-pipe work = 8 per reference predicate test
        # (5 DMUL + 2 DADD + 1 DSETP).  Dominant kernel: the slab join (sparse
        # engine) - its own tests (stream_comps, this rank) over its own launch time
        # (CUDA events around the launch on the library stream).
        achieved = 8.0 * stream_comps / (pairs_ms * 1e-3) / 1e12 if pairs_ms > 0 else 0.0
        peak = ops / 1e12
        tr = traffic_from_profile()
        result = {"edges": edges, "fingerprint": fp, "comps": comps}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
                "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded model sampler)",
                "config": workload_config(name, wl, world),
                "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                        "d2h_bytes_per_step": d2h // args.steps},
                "gpu_launches": launches,
                "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak,
                             "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                             "kernel": "sparse engine: slab_kernel (+ its small tail_kernel, on its own stream: its "
                                       "own duration added), CUDA events around the launches; in the timed steps the "
                                       "dense engine runs beside it on the same SMs (see 'isolated')",
                             "kernel_ms": pairs_ms / args.steps,
                             "kernel_tests_per_launch": stream_comps / args.steps,
                             "peak_source": "measured live: non-FMA DMUL+DADD rate (rhg_fp64_peak)",
                             "work": "8 FP64-pipe ops per reference predicate test (SURVEY 8(d)) x the kernel's tests",
                             "dmul_latency_cycles": lat, "kernel_profile": kernel_profile(),
                             "isolated": ({"kernel_ms": iso_ms / 3, "achieved": 8.0 * iso_tests / (iso_ms * 1e-3) / 1e12,
                                           "frac": 8.0 * iso_tests / (iso_ms * 1e-3) / ops,
                                           "note": "3 untimed steps after the timed region with the edge phase on one "
                                                   "stream (RHG_CONCURRENT_ENGINES=0, RHG_SIDE_SMALL=0)"}
                                          if iso_ms > 0 else None)},
                "fp64_roofline_frac_edge_phase": (8.0 * comps * args.steps / (edges_ms * 1e-3)) / ops / world,
                "fp64_roofline_frac_whole_step": (8.0 * comps * args.steps / (dev_ms * 1e-3)) / ops / world,
                "per_point": per_point_block(params, rank, world, dev_ms / args.steps, sample_ms / args.steps),
                "clocks": clk.summary(),
                "collective": ("one ncclAllReduce(uint64, 9 counters) per step inside the timed region"
                               if world > 1 and not one_gpu else
                               "gloo all-reduce per step (RHG_BENCH_ONE_GPU functional mode)" if world > 1 else None),
                "result": dict(result, W_ops_per_edge=8.0 * comps / max(edges, 1))}
        cpu_res = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                runs = [cpu_reference_run(n, d, g, seed, P) for _ in range(3)]
                secs = sorted(r[0]["seconds"] for r in runs)
                stc = runs[0][0]
                cpu_res = {"edges": stc["edges"], "fingerprint": stc["fingerprint"], "comps": stc["comps"]}
                line["cpu_baseline"] = {"value": stc["edges"] / secs[1], "unit": UNIT,
                                        "cores": os.cpu_count() or 1, "cpu": cpu_model(), "kind": "reference",
                                        "sample": f"full {name} generate_stats (oracle/_ref, all host threads), "
                                                  f"median of 3 runs: {secs[1]:.3f} s ({', '.join(f'{x:.3f}' for x in secs)})",
                                        "result": cpu_res}
            except Exception as e:  # noqa: BLE001 - report, do not fail the bench
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
        line["parity"] = parity_block(name, wl, result, cpu_res)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
