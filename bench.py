#!/usr/bin/env python
"""bench.py -- 3LC state-change compression throughput on B200.

One step = one pass of the whole hot path over
one synthetic state-change tensor: tlc_compress (accumulate + global max, quantize +
residual, quartic encode, zero-run encode) followed by tlc_decompress (ZRE expand,
quartic decode, dequantize), through the C ABI of include/tlc.h.

Workload at N=1 (BASELINE.json configs[2], the config the metric's "% HBM peak" is
quoted on -- north_star: ">= 64M-element tensors"): one 268,435,456-element fp32
tensor, s = 1.75, N(0,1) state changes with the error-accumulation buffer carried
across steps (steady state), zero-run encoding on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tlc|reference]

For N > 1 (torchrun, one rank per GPU, NCCL) each rank runs the same workload on its
own tensor (weak scaling); timing is the max over ranks.  `--impl reference` times
the CPU oracle (oracle/, the deliberately slow reference) on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+decompress fp32 GB/s per B200 (% HBM peak); bits/value; 8-GPU xchg"
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["tlc", "reference"], default="tlc")
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--s", type=float, default=1.75)
    ap.add_argument("--no-zre", action="store_true")
    ap.add_argument("--inputs", type=int, default=2, help="rotating state-change tensors")
    ap.add_argument("--cpu-steps", type=int, default=2, help="timed oracle round trips at the config size")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: seconds the timed oracle steps may take before they shrink to a sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the ResNet-110 (configs[1]) side measurement")
    ap.add_argument("--no-r50", action="store_true",
                    help="N > 1: skip the ResNet-50 exchange (the other model of configs[4])")
    ap.add_argument("--mode", choices=["auto", "codec", "exchange"], default="auto",
                    help="auto: codec step at N=1, parameter-server exchange step at N>1")
    ap.add_argument("--model", default="bert-large", help="tensor list of the exchange workload")
    ap.add_argument("--xs", type=float, default=1.9, help="s of the exchange workload (configs[4])")
    ap.add_argument("--no-xchg-w1", action="store_true", help="skip the N=1 exchange side measurement")
    ap.add_argument("--xchg", choices=["p2p", "nccl", "nccl-exact"], default="p2p",
                    help="exchange transport: peer-memory kernels over NVLink, NCCL send/recv of capacity "
                         "regions, or NCCL with a sizes all-gather and exact payload bytes")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the C3 families / s grid / 2^20..2^30 size sweep side measurement")
    ap.add_argument("--no-codecs", action="store_true",
                    help="skip the compared-design codecs side measurement (Stoch 3-value + QE, 8-bit int)")
    return ap.parse_args()


def workload_name(n, s, zre):
    return (f"C3: single {n:,}-element fp32 state-change tensor, s={s}, gauss-steady "
            f"(N(0,1) per step, error buffer carried){'' if zre else ', ZRE off'}")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def load_traffic(kernel, n):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    ncu --set full capture (profiles/ncu_traffic.json), if one exists for this n."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(kernel)
        if e and int(e.get("n", -1)) == n:
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while running."""

    def __init__(self, device, period: float = 0.005):
        self.period = period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            import torch

            uuid = str(torch.cuda.get_device_properties(device).uuid)
            self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        for k, bit in names.items():
            if r & bit and k != "gpu_idle":
                self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self.nv:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle legs
def host_info():
    """Host CPU of the box the oracle runs on: logical CPUs usable here and the model."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cores": cores, "cpu_model": model}


def oracle_config(n: int, s: float, zre: bool, omp: bool, steps: int, warmup: int = 1, budget_s: float = None):
    """Time the CPU oracle (oracle/tlc_oracle.c as it stands) on compress + decompress round
    trips of the workload itself: an n-element N(0,1) fp32 state change, two rotating
    inputs, the error buffer carried (steady state).  omp=True: the -fopenmp build of the
    same source (element-wise loops on every host core, zero-run coding serial).  If a
    time budget is given and a warm-up round trip shows the steps would exceed it, the
    timed steps run on a leading sample of the tensor instead (stated in `sample`)."""
    import numpy as np

    import oracle as O
    import synth

    O.use_openmp(omp)
    try:
        ts = [synth.gaussian(n, 3, k) for k in range(2)]
        buf = np.zeros(n, np.float32)
        t_w = []
        for k in range(max(1, warmup)):                      # untimed; page-faults the buffers
            t0 = time.perf_counter()
            c = O.compress(ts[k % 2], buf, s, zre)
            O.decompress(c.payload, zre, c.M, n)
            t_w.append(time.perf_counter() - t0)
        m = n
        if budget_s is not None and t_w[-1] * steps > budget_s:
            m = max(1 << 16, int(n * budget_s / (t_w[-1] * steps)) // 1024 * 1024)
            ts = [x[:m].copy() for x in ts]
            buf = buf[:m].copy()
        tc = td = 0.0
        for k in range(steps):
            t0 = time.perf_counter()
            c = O.compress(ts[k % 2], buf, s, zre)
            t1 = time.perf_counter()
            st, out = O.decompress(c.payload, zre, c.M, m)
            td += time.perf_counter() - t1
            tc += t1 - t0
            assert c.status == 0 and st == 0
    finally:
        O.use_openmp(False)
    h = host_info()
    threads = h["cores"] if omp else 1
    el = tc + td
    return {"value": 4.0 * m * steps / el / 1e9, "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": (f"{steps} compress+decompress round trips of the {n:,}-element workload tensor"
                       if m == n else f"{steps} round trips of the leading {m:,} of the {n:,} elements "
                                      f"(budget {budget_s:.0f} s)") +
                      f" (N(0,1), s={s}, error buffer carried), "
                      + (f"-fopenmp build on {threads} threads (element-wise loops; ZRE serial)" if omp
                         else "plain build, 1 thread") + f", {el:.1f} s",
            "same_config": m == n, "n_timed": m, "seconds": el, "steps": steps,
            "compress_GBps": 4.0 * m * steps / tc / 1e9, "decompress_GBps": 4.0 * m * steps / td / 1e9,
            "cpu_model": h["cpu_model"], "host_cores": h["cores"], "bits_per_value": 8.0 * c.payload_len / m}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    zre = not args.no_zre
    r = oracle_config(args.n, args.s, zre, omp=True, steps=max(1, args.steps), warmup=max(1, args.warmup),
                      budget_s=args.ref_budget)
    ms = 1000.0 * r["seconds"] / max(1, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: N(0,1) fp32 state changes (numpy PCG64), error buffer carried",
        "config": {"workload": workload_name(args.n, args.s, zre) + ("" if r["same_config"] else
                   f"; each step a bounded {r['n_timed']:,}-element sample on the host"), "n": args.n, "s": args.s},
        "bits_per_value": r["bits_per_value"],
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                           "compress_GBps", "decompress_GBps", "same_config")},
        "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ C2: ResNet-110 set
def measure_resnet110(T, dev, s, steps=200, warmup=10):
    """BASELINE configs[1]: the 110 per-layer ResNet-110 gradient tensors (1,719,856 values),
    compress + decompress through the batched launches, captured in one CUDA graph."""
    import torch

    import synth

    sizes = synth.RESNET110_SIZES
    mus = synth.layer_means(sizes, 2, 110)
    tsets = [[torch.from_numpy(synth.layer_gradient(n, mus[k], 2, 0, k, step)).to(dev)
              for k, n in enumerate(sizes)] for step in range(2)]
    outs = [torch.empty(n, dtype=torch.float32, device=dev) for n in sizes]
    ctx = T.TensorSet(sizes, dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        for k in range(warmup):                     # error feedback reaches steady state
            ctx.compress(tsets[k % 2], s, True, stream)
            ctx.decompress(outs, T.TLC_MODE_OVERWRITE, stream)
    torch.cuda.synchronize(dev)
    cb = [ctx.compress_batch(tsets[k]) for k in range(2)]
    db = ctx.decompress_batch(outs)
    torch.cuda.synchronize(dev)
    graphs = []
    for k in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            ctx.compress(tsets[k], s, True, stream, batch=cb[k])
            ctx.decompress(outs, T.TLC_MODE_OVERWRITE, stream, batch=db)
        graphs.append(g)
    torch.cuda.synchronize(dev)
    # warm: back-to-back replays (the whole working set, ~30 MB, stays in the 126 MB L2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(steps):
            graphs[k % 2].replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_warm = e0.elapsed_time(e1) / steps
    # cold: L2 flushed (a 512 MiB write) before every step, each step timed on its own
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for k in range(steps):
            flush.fill_(k & 0xff)
            evs[k][0].record(stream)
            graphs[k % 2].replay()
            evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    # per-kernel device times of the same step (outside the graph, library CUDA events)
    T.tlc_prof_collect()
    T.tlc_prof_enable(True)
    with torch.cuda.stream(stream):
        for k in range(20):
            flush.fill_(k & 0xff)
            ctx.compress(tsets[k % 2], s, True, stream, batch=cb[k % 2])
            ctx.decompress(outs, T.TLC_MODE_OVERWRITE, stream, batch=db)
    torch.cuda.synchronize(dev)
    T.tlc_prof_enable(False)
    prof = T.tlc_prof_collect()
    kern = {k: round(t / c * 1e3, 2) for k, (c, t) in prof.items()}
    kern_launches = {k: c for k, (c, t) in prof.items()}
    del flush
    N = sum(sizes)
    Z = sum(h["payload_len"] for h in ctx.headers())
    return {"workload": "C2: ResNet-110 gradient set, 110 tensors, 1,719,856 values, one tlc_batch "
                        "(small-table kernels: K6g compress (clusters of 4) + K7 decompress, one launch each) in a CUDA "
                        "graph, error feedback carried", "s": s,
            "value": 4.0 * N / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "l2": "flushed (512 MiB write) before every timed step",
            "warm": {"value": 4.0 * N / (ms_warm / 1e3) / 1e9, "ms_per_step": ms_warm,
                     "l2": "back-to-back replays, working set L2-resident"},
            "bits_per_value": 8.0 * Z / N, "kernel_launches_per_step": sum(kern_launches.values()) // 20,
            "kernel_us_cold": kern}


# ------------------------------------------------------------------ C3 families / s grid / size sweep
C3_ALG = {  # algorithmic HBM bytes per launch of the codec kernels
    "k1_absmax": lambda n, P, Z: 8.0 * n,
    "k2_quant_qe": lambda n, P, Z: 12.0 * n + P,
    "k3_zre": lambda n, P, Z: float(P + Z),
    "k4_zre_scan": lambda n, P, Z: float(Z),
    "k5_expand_dequant": lambda n, P, Z: 4.0 * n + Z,
}


def measure_c3_sweep(T, dev, configs, steps=10, warmup=8, flush_below=1 << 27):
    """SURVEY 8(d) C3 side measurements next to the headline: the four input families at
    the headline size (zeros, dense and runs with a fresh error buffer every step; gauss
    carried to steady state), the s grid, and the 2^20..2^30 size sweep.  A step is one
    tlc_compress + tlc_decompress timed with its own CUDA-event pair on the launching
    stream; per-kernel device times come from a second, profiled pass (library events).
    Tensors of n < 2^27 fit the 126 MB L2 with their error buffer and output, so the L2 is
    flushed (512 MiB write) before each of their steps, outside the events."""
    import torch

    import synth

    peak, _ = load_peaks()
    stream = torch.cuda.current_stream(dev)
    flush = None
    res = []
    for label, fam, n, s in configs:
        ts = [synth.family_torch(fam, n, s, dev, 3, k) for k in range(2 if fam == "gauss" else 1)]
        err = torch.zeros(n, dtype=torch.float32, device=dev)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        payload = torch.empty(T.tlc_max_payload_bytes(n), dtype=torch.uint8, device=dev)
        hdr = T.new_header(dev)
        ws_c = torch.empty(T.tlc_compress_workspace_bytes(n), dtype=torch.uint8, device=dev)
        ws_d = torch.empty(T.tlc_decompress_workspace_bytes(n), dtype=torch.uint8, device=dev)
        fresh = fam != "gauss"
        cold = n < flush_below
        if cold and flush is None:
            flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

        def step(k):
            T.tlc_compress(ts[k % len(ts)], err, s, True, payload, hdr, ws_c, stream)
            T.tlc_decompress(payload, hdr, n, out, T.TLC_MODE_OVERWRITE, ws_d, stream)

        def prep(k):
            if fresh:
                err.zero_()
            if cold:
                flush.fill_(k & 0xff)

        for k in range(warmup):
            prep(k)
            step(k)
        torch.cuda.synchronize(dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            prep(k)
            evs[k][0].record(stream)
            step(k)
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        ms = sorted(a.elapsed_time(b) for a, b in evs)
        ms_med = ms[len(ms) // 2]
        T.tlc_prof_collect()
        T.tlc_prof_enable(True)
        for k in range(steps):
            prep(k)
            step(k)
        T.tlc_prof_enable(False)
        prof = T.tlc_prof_collect()
        h = T.parse_header(hdr)
        P, Z = (n + 4) // 5, h["payload_len"]
        kern = {}
        for name, (cnt, tot) in prof.items():
            avg = tot / max(cnt, 1)
            b = C3_ALG[name](n, P, Z) if name in C3_ALG else None
            kern[name] = {"avg_ms": round(avg, 5), "alg_GBps": round(b / (avg / 1e3) / 1e9, 1) if b else None}
        k2 = kern.get("k2_quant_qe", {}).get("alg_GBps")
        res.append({"label": label, "family": fam, "n": n, "s": s, "status": h["status"],
                    "error_buffer": "fresh (zeroed before every step)" if fresh else "carried (steady state)",
                    "l2": "flushed before every step" if cold else "inputs larger than L2",
                    "value": 4.0 * n / (ms_med / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms_med,
                    "ms_min": ms[0], "ms_max": ms[-1], "bits_per_value": 8.0 * Z / n,
                    "step_alg_frac": (24.0 * n + 2 * P + 3 * Z) / (ms_med / 1e3) / 1e9 / peak,
                    "k2_frac": (k2 / peak) if k2 else None, "kernels": kern})
        del ts, err, out, payload, ws_c, ws_d
        torch.cuda.empty_cache()
    return {"what": "C3 side measurements (SURVEY 8(d)): families at the headline size, s grid, size sweep; "
                    "value = fp32-input GB/s (median step), step_alg_frac = (24n + 2P + 3Z) bytes per step / "
                    "step time / measured HBM peak, k2_frac = K2's (12n + P) / its time / peak",
            "steps": steps, "warmup": warmup, "runs": res}


def c3_sweep_configs(n_head, s_head):
    cfg = [(f"family {f}", f, n_head, s_head) for f in ("zeros", "dense", "runs")]
    cfg += [(f"gauss s={sv}", "gauss", n_head, sv) for sv in (1.0, 1.5, 1.9)]
    cfg += [(f"gauss n=2^{e}", "gauss", 1 << e, s_head) for e in (20, 22, 24, 26, 30)]
    return cfg


# ------------------------------------------------------------------ exchange step (row e)
NVLINK_GBS = 770.0   # measured peer copy per direction per GPU (B200_PROFILING.md)


def measure_codecs(T, dev, ts, steps=20, warmup=3):
    """Side measurement: the paper's compared designs that share the 3LC
    kernels, on the same n-element N(0,1) tensors as the headline: "Stoch 3-value + QE"
    (QE only as in the paper, and with ZRE) and "8-bit int".  A step
    is one compress + decompress; value = fp32-input GB/s.  Per-kernel device times come from
    the library's CUDA events on the launching stream (a second, profiled pass)."""
    import torch

    n = ts[0].numel()
    P = (n + 4) // 5
    stream = torch.cuda.current_stream(dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    payload = torch.empty(T.tlc_max_payload_bytes(n), dtype=torch.uint8, device=dev)
    hdr = T.new_header(dev)
    ws_c = torch.empty(T.tlc_compress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    ws_d = torch.empty(T.tlc_decompress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    codes = torch.empty(n, dtype=torch.int8, device=dev)
    ws_8 = torch.empty(T.tlc_int8_workspace_bytes(n), dtype=torch.uint8, device=dev)

    def stoch_step(k, zre):
        T.tlc_stoch_compress(ts[k % len(ts)], 7, k, zre, payload, hdr, ws_c, stream)
        T.tlc_decompress(payload, hdr, n, out, T.TLC_MODE_OVERWRITE, ws_d, stream)

    def int8_step(k):
        T.tlc_int8_compress(ts[k % len(ts)], codes, hdr, ws_8, stream)
        T.tlc_int8_decompress(codes, hdr, n, out, T.TLC_MODE_OVERWRITE, stream)

    def timed(fn):
        for k in range(warmup):
            fn(k)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(steps):
            fn(k)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        T.tlc_prof_collect()
        T.tlc_prof_enable(True)
        for k in range(steps):
            fn(k)
        T.tlc_prof_enable(False)
        prof = T.tlc_prof_collect()
        h = T.parse_header(hdr)
        return ms, {k: v[1] / max(v[0], 1) for k, v in prof.items()}, h

    peak, _ = load_peaks()
    res = []
    for zre in (False, True):
        ms, kern, h = timed(lambda k: stoch_step(k, zre))
        Z = h["payload_len"]
        alg = {"k1_absmax": 4.0 * n, "k2s_stoch_qe": 4.0 * n + P, "k3_zre": float(P + Z) if zre else 0.0,
               "k4_zre_scan": float(Z), "k5_expand_dequant": 4.0 * n + Z}
        dom = "k2s_stoch_qe"
        ach = alg[dom] / (kern[dom] / 1e3) / 1e9
        res.append({"design": "Stoch 3-value + QE" + (" + ZRE" if zre else ""), "cite": "P:629-632, R22",
                    "value": 4.0 * n / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                    "bits_per_value": 8.0 * Z / n, "status": h["status"],
                    "kernel_ms": {k: round(v, 5) for k, v in kern.items()},
                    "roofline": {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                 "frac": ach / peak, "alg_bytes_formula": "4n + ceil(n/5)",
                                 "limiter": "instruction issue, not HBM: Philox4x32-10 (20 IMAD.WIDE + 20 LOP3 "
                                            "per 4 values) + the exact-comparison digit, ~36 thread-instr per "
                                            "value at ~60 % issue busy (ncu, profiles/r01_ncu_summary.md)"}})
    ms, kern, h = timed(int8_step)
    alg = {"k1_absmax": 4.0 * n, "kq8_int8_quant": 5.0 * n, "kd8_int8_dequant": 5.0 * n}
    doms = {k: alg[k] / (kern[k] / 1e3) / 1e9 for k in ("kq8_int8_quant", "kd8_int8_dequant")}
    res.append({"design": "8-bit int", "cite": "P:624-627, R23", "value": 4.0 * n / (ms / 1e3) / 1e9,
                "unit": "GB/s", "ms_per_step": ms, "bits_per_value": 8.0, "status": h["status"],
                "kernel_ms": {k: round(v, 5) for k, v in kern.items()},
                "roofline": {"kernel": "kq8_int8_quant", "bound": "hbm", "achieved": doms["kq8_int8_quant"],
                             "peak": peak, "unit": "GB/s", "frac": doms["kq8_int8_quant"] / peak,
                             "alg_bytes_formula": "5n (read t, write codes)",
                             "dequant_achieved": doms["kd8_int8_dequant"]}})
    return {"workload": f"n = {n:,} N(0,1) fp32 (same tensors as the headline), compress + decompress per step",
            "steps": steps, "designs": res}


def measure_exchange(T, dev, world, rank, model, s, steps, warmup, dist=None, p2p=True, e2e_steps=0, exact=False):
    """BASELINE configs[4]: the model's ndim>=2 gradient tensors exchanged through
    the parameter-server push/pull (tlc_exchange_push + tlc_exchange_pull, delta =
    mean) on `world` ranks; every rank holds its own full state change (weak
    scaling).  Returns the rank-local timings; the caller takes the max over ranks."""
    import torch

    import synth

    sizes = synth.MODELS[model]
    N = sum(sizes)
    grads = [synth.model_step_torch(model, k, rank, dev) for k in range(2)]
    outs = [torch.zeros(n, dtype=torch.float32, device=dev) for n in sizes]
    comm = T.Comm(rank, world, dev)
    x = T.Exchange(comm, sizes, p2p=p2p, exact=exact)
    stream = torch.cuda.current_stream(dev)

    def step(k):
        x.push(grads[k % 2], s, True, stream)
        x.pull(outs, s, True, stream)

    for k in range(max(3, warmup)):
        step(k)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    T.tlc_prof_collect()
    T.tlc_prof_enable(True)
    l0 = T.tlc_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(steps):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    T.tlc_prof_enable(False)
    launches = T.tlc_launch_count() - l0
    prof = T.tlc_prof_collect()
    ms = e0.elapsed_time(e1) / steps
    status = x.status(stream)
    wire = sum(x.traffic())
    kern_ms = sum(tot for (_, tot) in prof.values()) / steps

    e2e = None
    if e2e_steps:
        # End to end through the same public calls: every step copies its gradient set
        # (N fp32 values) from pinned host memory, runs push + pull and reads the
        # exchange status back to pinned host memory (the step's result; the model
        # update stays in HBM).  H2D on its own stream, double-buffered, so step k+1's
        # copy overlaps step k's exchange.
        gflat = [torch.empty(N, dtype=torch.float32, device=dev) for _ in range(2)]
        gv = [list(torch.split(g, sizes)) for g in gflat]
        hin = torch.empty(N, dtype=torch.float32, pin_memory=True)
        hin.copy_(torch.cat(grads[0]).cpu())
        hst = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        h2d = torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]

        def e2e_step(k):
            b = k % 2
            h2d.wait_event(ev_done[b])
            with torch.cuda.stream(h2d):
                gflat[b].copy_(hin, non_blocking=True)
            ev_in[b].record(h2d)
            stream.wait_event(ev_in[b])
            x.push(gv[b], s, True, stream)
            x.pull(outs, s, True, stream)
            x.status_async(hst[b:b + 1], stream)
            ev_done[b].record(stream)

        for b in range(2):
            ev_done[b].record(stream)
        for k in range(2):
            e2e_step(k)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for b in range(2):
            ev_done[b].record(stream)
        for k in range(e2e_steps):
            e2e_step(k)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        e2e = {"ms": f0.elapsed_time(f1) / e2e_steps, "h2d": 4 * N, "d2h": 4, "steps": e2e_steps,
               "status": int(hst.max())}
    x.close()
    comm.close()
    plan = T.tlc_plan(sizes, world)
    # K2's algorithmic bytes per step on this rank: 12 n_c + ceil(n_c / 5) per compressed
    # context (read t, err; write err, quartic bytes) -- every context in the push, the
    # contexts this rank owns in the pull (the owner re-compresses the model delta)
    k2_push = sum(12 * (hi - lo) + (hi - lo + 4) // 5 for (_, lo, hi, _) in plan)
    k2_pull = sum(12 * (hi - lo) + (hi - lo + 4) // 5 for (_, lo, hi, ow) in plan if ow == rank)
    # the step's streaming bytes on this rank, a lower bound (payload terms and the apply's
    # skip-zero read-modify-writes left out): push K1 + K2 over every context (8n + 12n + P),
    # K5m's 4 n_own of means, the pull's K1 + K2 over the owned contexts
    n_own = sum(hi - lo for (_, lo, hi, ow) in plan if ow == rank)
    step_bytes = 8 * N + k2_push + 4 * n_own + 8 * n_own + k2_pull
    keyed = n_own > 0 and "k1_absmax" in prof and prof["k1_absmax"][0] / steps < 1.5
    if keyed:
        # the pull compress's K1 folded into K5m (one K1 launch per step): K5m reads the pull
        # error buffer (4 n_own) instead of K1 reading mean and error buffer (8 n_own)
        step_bytes = 8 * N + k2_push + 4 * n_own + 4 * n_own + k2_pull
    if "k12_absmax_quant" in prof:
        # K12 reads t and err from HBM once (its quantize items hit L2): no K1 terms
        step_bytes = k2_push + 4 * n_own + k2_pull
    return {"ms": ms, "kernel_ms": kern_ms, "launches": launches, "wire": wire, "N": N, "status": status,
            "contexts": len(plan), "e2e": e2e, "k2_alg_bytes_per_step": k2_push + k2_pull,
            "step_alg_bytes": step_bytes,
            "kernels": {k: {"launches_per_step": c / steps, "ms_per_step": t / steps} for k, (c, t) in prof.items()}}


def measure_exchange_graph(T, dev, world, rank, model, s, steps, warmup, dist=None):
    """configs[3]: the ResNet-110 (latency-bound) PS push + pull, peer-memory transport,
    captured once as a CUDA graph and replayed (working set L2-resident: 6.9 MB of
    state changes per rank).  Returns this rank's ms per step."""
    import torch

    import synth

    sizes = synth.MODELS[model]
    grads = synth.model_step_torch(model, 0, rank, dev)
    outs = [torch.zeros(n, dtype=torch.float32, device=dev) for n in sizes]
    comm = T.Comm(rank, world, dev)
    x = T.Exchange(comm, sizes, p2p=True)
    for _ in range(max(3, warmup)):
        x.push(grads, s)
        x.pull(outs, s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        x.push(grads, s)
        x.pull(outs, s)
    for _ in range(max(3, warmup)):
        g.replay()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    status = x.status()
    del g
    x.close()
    comm.close()
    return ms, sum(sizes), status


def measure_allreduce(dev, world, rank, model, steps, warmup, dist, graph=False):
    """The paper's baseline, "32-bit float": the same per-rank gradient set
    averaged uncompressed -- one ncclAllReduce (sum) of the flat fp32 set, then / W --
    timed like the exchange (events on the stream, max over ranks).  graph=True captures
    the step in a CUDA graph (the ResNet-110 case, as its exchange is)."""
    import torch

    import synth

    sizes = synth.MODELS[model]
    flat = torch.cat(synth.model_step_torch(model, 0, rank, dev))
    stream = torch.cuda.current_stream(dev)

    def step():
        dist.all_reduce(flat)
        flat.div_(world)

    for _ in range(max(3, warmup)):
        step()
    g = None
    if graph:
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        g.replay() if g is not None else step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del g, flat
    torch.cuda.empty_cache()
    return float(t.item()), sum(sizes)


def run_exchange_leg(args, T, dev, world, rank, dist, e2e_steps=None):
    import torch

    r = measure_exchange(T, dev, world, rank, args.model, args.xs, args.steps, args.warmup,
                         dist if world > 1 else None, p2p=args.xchg == "p2p", exact=args.xchg == "nccl-exact",
                         e2e_steps=e2e_steps if e2e_steps is not None else (0 if args.no_e2e else args.e2e_steps))
    ms = r["ms"]
    ems = r["e2e"]["ms"] if r["e2e"] else None
    if world > 1:
        t = torch.tensor([ms, ems or 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        ems = float(t[1].item()) if r["e2e"] else None
    value = world * 4.0 * r["N"] / (ms / 1e3) / 1e9
    if r["e2e"]:
        r["e2e"]["value"] = world * 4.0 * r["N"] / (ems / 1e3) / 1e9
        r["e2e"]["ms"] = ems
    return r, ms, value


def exchange_roofline(r, step_ms=None):
    """roofline object of the exchange step's dominant kernel (K2 over the segment table,
    push + pull launches) on this rank: algorithmic bytes per step / its device time per step;
    step_frac: the step's streaming bytes (a lower bound) / step time / peak."""
    dom = "k12_absmax_quant" if "k12_absmax_quant" in r["kernels"] else "k2_quant_qe"
    k = r["kernels"].get(dom)
    if not k or not k["ms_per_step"]:
        return None
    fused = dom == "k12_absmax_quant"
    peak, peak_src = load_peaks()
    achieved = r["k2_alg_bytes_per_step"] / (k["ms_per_step"] / 1e3) / 1e9
    sf = (r["step_alg_bytes"] / ((step_ms or r["ms"]) / 1e3) / 1e9 / peak) if r.get("step_alg_bytes") else None
    return {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "step_frac": sf, "step_alg_bytes": r.get("step_alg_bytes"),
            "step_alg_bytes_formula": ("sum(12 n_c + ceil(n_c/5)) (push K12: t, err read once) + 4 n_own (K5m "
                                       "means) + sum_own(12 n_c + ceil(n_c/5)) (pull K12)" if fused else
                                       "8N + sum(12 n_c + ceil(n_c/5)) (push K1, K2) + 4 n_own (K5m means) + "
                                       "8 n_own (pull K1; 4 n_own when K5m folds the pull's keys, reading the "
                                       "pull error buffer) + sum_own(12 n_c + ceil(n_c/5)) (pull K2)") +
                                      "; payload bytes and the apply's skip-zero read-modify-writes omitted "
                                      "(lower bound); rank 0",
            "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
            "launches_per_step": k["launches_per_step"],
            "alg_bytes_per_launch": r["k2_alg_bytes_per_step"] / k["launches_per_step"],
            "alg_bytes_formula": "sum over compressed contexts of 12 n_c + ceil(n_c/5): all contexts (push) "
                                 "+ the contexts this rank owns (pull), per step; rank 0" +
                                 ("; K12 = K1 and K2 fused, t and err read from HBM once" if fused else "")}


# ------------------------------------------------------------------ the GPU leg
def run_tlc(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1802_07389_b200 as T
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    mode = args.mode if args.mode != "auto" else ("codec" if world == 1 else "exchange")
    if mode == "exchange":
        return run_exchange_main(args, T, dev, world, rank, dist)

    n, s, zre = args.n, float(args.s), not args.no_zre
    # Inputs: seeded host generator (same module the oracle tests use), copied once
    # to HBM before any timing; each rank draws its own stream.
    ts = [torch.from_numpy(synth.gaussian(n, 3, 1000 * rank + k)).to(dev) for k in range(args.inputs)]
    err = torch.zeros(n, dtype=torch.float32, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    payload = torch.empty(T.tlc_max_payload_bytes(n), dtype=torch.uint8, device=dev)
    hdr = T.new_header(dev)
    ws_c = torch.empty(T.tlc_compress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    ws_d = torch.empty(T.tlc_decompress_workspace_bytes(n), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(k):
        T.tlc_compress(ts[k % len(ts)], err, s, zre, payload, hdr, ws_c, stream)
        T.tlc_decompress(payload, hdr, n, out, T.TLC_MODE_OVERWRITE, ws_d, stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    for k in range(max(3, args.warmup)):
        step(k)
    barrier()
    h = T.parse_header(hdr)
    if h["status"] != 0:
        raise RuntimeError(f"compress status {h}")

    # ---------------- timed region (device events on the launching stream)
    K = args.steps
    clocks = ClockSampler(dev)
    launches0 = T.tlc_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clocks.start()
    e0.record(stream)
    for k in range(K):
        step(k)
    e1.record(stream)
    barrier()
    clocks.stop()
    gpu_launches = T.tlc_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    h = T.parse_header(hdr)
    Z = h["payload_len"]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * 4.0 * n * K / (ms / 1e3) / 1e9

    # ---------------- the same K steps again with a CUDA-event pair around every library
    # kernel launch on its stream (per-kernel durations for the roofline; the events
    # break the programmatic-dependent-launch overlap, so this pass is a bit slower)
    T.tlc_prof_collect()
    T.tlc_prof_enable(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    p0.record(stream)
    for k in range(K):
        step(k)
    p1.record(stream)
    barrier()
    T.tlc_prof_enable(False)
    prof = T.tlc_prof_collect()
    ms_prof = p0.elapsed_time(p1)

    # ---------------- roofline of the dominant kernel (K2) and the per-kernel table
    peak, peak_src = load_peaks()
    P = (n + 4) // 5
    alg = {  # algorithmic HBM bytes per launch
        "k1_absmax": 8.0 * n,                 # read t, err
        "k2_quant_qe": 12.0 * n + P,          # read t, err; write err, quartic bytes
        "k3_zre": float(P + Z) if zre else 0.0,   # read quartic bytes, write payload
        "k4_zre_scan": float(Z),              # read payload
        "k5_expand_dequant": 4.0 * n + Z,     # read payload, write out
    }
    kernels = {}
    for name, (cnt, tot) in prof.items():
        avg = tot / max(cnt, 1)
        b = alg.get(name)
        kernels[name] = {"launches_per_step": cnt / K, "avg_ms": avg,
                         "alg_bytes": b, "alg_GBps": (b / (avg / 1e3) / 1e9) if b else None,
                         "share_of_step": (tot / K) / (ms_prof / K) if ms_prof else None}
    dom = "k2_quant_qe"
    dk = kernels.get(dom, {})
    achieved = dk.get("alg_GBps")
    roofline = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": load_traffic(dom, n),
                "peak_source": peak_src,
                "alg_bytes_per_launch": alg[dom], "alg_bytes_formula": "12n + ceil(n/5) (read t, err; write err, quartic bytes)"}
    step_bytes = sum(alg.values())
    hbm_frac_step = step_bytes / (ms / K / 1e3) / 1e9 / peak

    # ---------------- end to end through the same C-ABI calls, host buffers
    e2e = None
    if not args.no_e2e:
        th = torch.empty(n, dtype=torch.float32, pin_memory=True)
        th.copy_(ts[0].cpu())
        ohb = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        tdb = [torch.empty_like(ts[0]) for _ in range(2)]
        outb = [out, torch.empty_like(out)]
        E = max(1, args.e2e_steps)
        # Step k: H2D of its input (copy stream 1), compress + decompress (the
        # codec stream), D2H of its output (copy stream 2).  Double buffers let
        # step k+1's H2D and step k's D2H run concurrently (full-duplex PCIe)
        # while every step still moves its whole input in and its output out.
        h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        for b in range(2):
            ev_done[b].record(stream)
            ev_out[b].record(stream)

        def e2e_step(k):
            b = k % 2
            h2d.wait_event(ev_done[b])                 # tdb[b] no longer read by step k-2
            with torch.cuda.stream(h2d):
                tdb[b].copy_(th, non_blocking=True)
            ev_in[b].record(h2d)
            stream.wait_event(ev_in[b])
            stream.wait_event(ev_out[b])               # outb[b] drained by step k-2's D2H
            T.tlc_compress(tdb[b], err, s, zre, payload, hdr, ws_c, stream)
            T.tlc_decompress(payload, hdr, n, outb[b], T.TLC_MODE_OVERWRITE, ws_d, stream)
            ev_done[b].record(stream)
            d2h.wait_event(ev_done[b])
            with torch.cuda.stream(d2h):
                ohb[b].copy_(outb[b], non_blocking=True)
            ev_out[b].record(d2h)

        for k in range(2):
            e2e_step(k)
        stream.wait_event(ev_out[0])
        stream.wait_event(ev_out[1])
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for b in range(2):                             # the timed steps start after f0
            ev_done[b].record(stream)
            ev_out[b].record(stream)
        for k in range(E):
            e2e_step(k)
        stream.wait_event(ev_out[0])
        stream.wait_event(ev_out[1])
        f1.record(stream)
        barrier()
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * 4.0 * n * E / (ems / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n, "steps": E,
               "ms_per_step": ems / E,
               "what": "per step: pinned host t -> HBM, tlc_compress, tlc_decompress, HBM -> pinned host out; "
                       "H2D, codec and D2H on three streams, double-buffered across steps"}

    xw1 = None
    if world == 1 and not args.no_xchg_w1:
        r, xms, xval = run_exchange_leg(args, T, dev, 1, 0, None, e2e_steps=0)
        xw1 = {"workload": f"configs[4]: {args.model} gradient exchange (push+pull) at s={args.xs}, W=1",
               "value": xval, "unit": "GB/s", "ms_per_step": xms, "kernel_ms_per_step": r["kernel_ms"],
               "roofline": exchange_roofline(r), "status": r["status"]}

    codecs = None
    if rank == 0 and world == 1 and not args.no_codecs:
        codecs = measure_codecs(T, dev, ts)

    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        del ts, err, out, payload, ws_c, ws_d
        torch.cuda.empty_cache()
        sweep = measure_c3_sweep(T, dev, c3_sweep_configs(n, s))

    c2 = None
    if rank == 0 and not args.no_c2:
        c2 = [measure_resnet110(T, dev, sv) for sv in (1.0, 1.75, 1.9)]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle at the config size, compress and decompress timed separately: the
        # -fopenmp build on every host core (the baseline), and the plain build on one
        r = oracle_config(n, s, zre, omp=True, steps=args.cpu_steps, budget_s=60.0)
        r1 = oracle_config(n, s, zre, omp=False, steps=1, warmup=1, budget_s=30.0)
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "host_cores",
                                 "compress_GBps", "decompress_GBps", "same_config")}
        cpu["single_thread"] = {k: r1[k] for k in ("value", "sample", "compress_GBps", "decompress_GBps",
                                                    "same_config")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": max(3, args.warmup), "ms_per_step": ms / K, "ms_per_step_profiled_pass": ms_prof / K,
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: N(0,1) fp32 state changes (numpy PCG64, synth/), "
                    f"{args.inputs} rotating tensors per rank, error buffer carried across steps",
            "config": {"workload": workload_name(n, s, zre), "n": n, "s": s, "use_zre": zre,
                       "family": "gauss-steady",
                       "l2": "inputs larger than L2 (t, err, out 1 GiB each vs 126 MB L2); no flush",
                       "parallelism": "replicas" if world > 1 else "single"},
            "bits_per_value": 8.0 * Z / n,
            "compression_ratio": 4.0 * n / Z if Z else None,
            "hbm_frac_step": hbm_frac_step,
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "c2_resnet110": c2,
            "xchg_w1": xw1,
            "next3_codecs": codecs,
            "c3_sweep": sweep,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_exchange_main(args, T, dev, world, rank, dist):
    """N > 1: the parameter-server exchange step of configs[4] (weak scaling)."""
    import torch

    clocks = ClockSampler(dev)
    clocks.start()
    r, ms, value = run_exchange_leg(args, T, dev, world, rank, dist)
    clocks.stop()
    ar_ms, _ = measure_allreduce(dev, world, rank, args.model, args.steps, args.warmup, dist)
    c4, ar4_ms = [], None
    if not args.no_c2:
        ar4_ms, _ = measure_allreduce(dev, world, rank, "resnet110", max(args.steps, 50), args.warmup, dist,
                                      graph=True)
        for s4 in (1.0, 1.75, 1.9):
            ms4, n4, st4 = measure_exchange_graph(T, dev, world, rank, "resnet110", s4, max(args.steps, 50),
                                                  args.warmup, dist)
            t = torch.tensor([ms4], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms4 = float(t.item())
            c4.append({"s": s4, "ms_per_step": ms4, "value": world * 4.0 * n4 / (ms4 / 1e3) / 1e9, "unit": "GB/s",
                       "status": st4, "allreduce_fp32_ms_per_step": ar4_ms,
                       "speedup_vs_allreduce": ar4_ms / ms4})
    r50 = None
    if not args.no_r50 and args.model != "resnet50":
        # configs[4]'s other model: ResNet-50's gradient set (161 tensors, ~25.6 M values per rank)
        rr = measure_exchange(T, dev, world, rank, "resnet50", args.xs, args.steps, args.warmup, dist,
                              p2p=args.xchg == "p2p", exact=args.xchg == "nccl-exact", e2e_steps=0)
        t = torch.tensor([rr["ms"]], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms50 = float(t.item())
        ar50, _ = measure_allreduce(dev, world, rank, "resnet50", args.steps, args.warmup, dist)
        r50 = {"workload": f"configs[4]: ResNet-50 gradient exchange (push + pull at s={args.xs}, "
                           f"{rr['N']:,} values per rank, {rr['contexts']} contexts), same transport",
               "ms_per_step": ms50, "value": world * 4.0 * rr["N"] / (ms50 / 1e3) / 1e9, "unit": "GB/s",
               "status": rr["status"], "allreduce_fp32_ms_per_step": ar50, "speedup_vs_allreduce": ar50 / ms50,
               "kernels_rank0": rr["kernels"]}
    if rank == 0:
        pct_nvlink = r["wire"] / 2 / (ms / 1e3) / 1e9 / NVLINK_GBS   # per direction
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic: {args.model} ndim>=2 gradient shapes, g = mu_l + N(0,1) per layer "
                    "(torch Philox on device, synth/), 2 rotating steps per rank",
            "config": {"workload": f"configs[4]: {args.model} gradient exchange, parameter-server push "
                                   f"(compress, owners' fused aggregate of the W payloads / W) + shared pull "
                                   f"(owner compresses once, every rank applies) at s={args.xs}, "
                                   f"{r['N']:,} values per rank; transport: "
                                   + ("kernels read peers' payloads over NVLink (CUDA IPC), flag barriers"
                                      if args.xchg == "p2p" else
                                      "NCCL sizes all-gather + grouped send/recv of exact payload bytes"
                                      if args.xchg == "nccl-exact" else
                                      "NCCL grouped send/recv of capacity regions"),
                       "n_per_rank": r["N"], "s": args.xs, "contexts": r["contexts"],
                       "l2": "inputs larger than L2 (1.34 GB of state changes per rank); no flush",
                       "parallelism": f"ps{world} (sharded parameter server, {args.xchg})"},
            "value_definition": "world x 4 x values-per-rank / step time (effective fp32 GB/s exchanged)",
            "wire_bytes_per_rank_per_step": r["wire"],
            "wire_definition": "bytes rank 0 received from other ranks per step (push + pull)",
            "nvlink_frac": pct_nvlink,
            "allreduce_fp32": {"what": "the paper's '32-bit float' baseline (P:621-622) on the same tensors: "
                                       "ncclAllReduce(sum) of the flat fp32 gradient set + /W, events, max over ranks",
                               "ms_per_step": ar_ms, "value": world * 4.0 * r["N"] / (ar_ms / 1e3) / 1e9,
                               "unit": "GB/s"},
            "speedup_vs_allreduce": ar_ms / ms,
            "roofline": exchange_roofline(r, ms),
            "kernel_ms_per_step_rank0": r["kernel_ms"],
            "kernels_rank0": r["kernels"],
            "gpu_launches": r["launches"],
            "exchange_status": r["status"],
            "resnet50": r50,
            "c4_resnet110": ({"workload": "configs[3]: ResNet-110 gradient set (110 tensors, 1,719,856 values per "
                                          "rank) PS push + pull, peer-memory transport, one CUDA graph per step, "
                                          "max over ranks; working set L2-resident",
                              "runs": c4} if c4 else None),
            "e2e": ({"value": r["e2e"]["value"], "unit": "GB/s", "h2d_bytes_per_step": r["e2e"]["h2d"],
                     "d2h_bytes_per_step": r["e2e"]["d2h"], "steps": r["e2e"]["steps"], "ms_per_step": r["e2e"]["ms"],
                     "status": r["e2e"]["status"],
                     "what": "per step and rank: pinned host gradient set -> HBM (own stream, double-buffered), "
                             "tlc_exchange_push + tlc_exchange_pull, exchange status -> pinned host"}
                    if r["e2e"] else None),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_tlc(args)


if __name__ == "__main__":
    sys.exit(main())
