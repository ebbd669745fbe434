#!/usr/bin/env python
"""Benchmark of the DMS front end (vertex order, lower-star gradient, critical
simplices, D0, D_{d-1}) on one B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

A step is one pass of the whole hot path over the
configured synthetic field, which is resident in HBM before the timed region.  Under
torchrun every rank runs an independent replica (its own seed): the path does not
shard, so scaling is weak and there is no
data-path collective; the timing is the max over ranks.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "M vertices/s (gradient + D0 + D_{d-1}, 1 B200) and % of HBM roofline"
UNIT = "M vertices/s"

CONFIG_DESC = {
    "c1": "3D 32^3 float32 iid U[0,1)",
    "c2": "3D 128^3 float32 sum of 32 Gaussians + 1e-3 noise",
    "c3": "3D 256^3 float32 iid U[0,1)",
    "c4": "3D 512^3 float32 5-octave value noise (period 64, gain 0.5) + N(0,1e-2)",
    "c5a": "2D 8192^2 float32 fBm H=0.7 (spectral)",
    "c5b": "1D 2^27 float32 random walk",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def algorithmic_bytes(N, ndim, ncrit, npairs):
    """B_min = N (4 read f + 4 write rank + G_w) + 8 sum|C_k| + 32 pairs,
    G_w = 8 / 2 / 0.25 B per vertex (3D / 2D / 1D reference gradient layout)."""
    gw = {3: 8.0, 2: 2.0, 1: 0.25}[ndim]
    e2e = N * (4 + 4 + gw) + 8 * sum(ncrit) + 32 * npairs
    grad_kernel = N * (4 + gw) + 8 * sum(ncrit)
    return e2e, grad_kernel


def host_cpu_info():
    """lscpu model name, physical cores and logical CPUs of the host the oracle runs on."""
    info = {"logical_cpus": os.cpu_count() or 1}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        cps, sk = kv.get("Core(s) per socket"), kv.get("Socket(s)")
        if cps and sk and cps.isdigit() and sk.isdigit():
            info["physical_cores"] = int(cps) * int(sk)
    except Exception:
        pass
    return info


ORACLE_STAGES = ("nan_scan_fstar", "gradient", "critical_sort", "d0", "dtop", "d1_and_generators")


def oracle_timed(crop, nthreads, want_d1=False):
    """One timed oracle pass over `crop`: the vertex order (orc_ranks) and the
    rest of the front end (orc_run: gradient, C_k, D0, D_{d-1}), per stage in ms.  With
    want_d1 (3D) the oracle also runs D1 + generators (Alg. 3, Sec. 9): reported as its
    own stage and NOT included in the returned front-end time."""
    import oracle

    t0 = time.perf_counter()
    oracle.ranks(crop)
    t_order = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    r = oracle.run(crop, nthreads=nthreads, want_pairs=False, want_d1=want_d1)
    t_run = (time.perf_counter() - t0) * 1e3
    stages = {"order": round(t_order, 2)}
    stages.update({k: round(float(v), 2) for k, v in zip(ORACLE_STAGES, r.ms[:6])})
    if not want_d1:
        stages.pop("d1_and_generators", None)
    else:
        t_run -= float(r.ms[5])
        stages["d1_pairs"] = int(len(r.d1))
    return t_order + t_run, stages


def cpu_oracle_sample(f_full, budget_s=24.0):
    """The oracle (as it stands, never tuned) on a bounded crop of the same field, on the
    host cores, 1 thread and all cores; each setting is one pass of the
    whole front end including the vertex order, with per-stage times.  The crop grows
    until the all-core pass takes >= 1/4 of the budget (the 1-thread pass then fits)."""
    import numpy as np

    cores = os.cpu_count() or 1
    d = f_full.ndim
    side = {3: 32, 2: 256, 1: 1 << 16}[d]
    while True:
        crop = np.ascontiguousarray(f_full[tuple(slice(0, min(side, s)) for s in f_full.shape)])
        t_all, st_all = oracle_timed(crop, cores, want_d1=(d == 3))
        grown = tuple(min(int(side * (1.26 if d == 3 else (1.41 if d == 2 else 2))), s) for s in f_full.shape)
        if t_all >= budget_s * 250 or grown == tuple(min(side, s) for s in f_full.shape):
            break
        side = max(grown)
    t_one, st_one = oracle_timed(crop, 1, want_d1=(d == 3))
    n = crop.size
    return {"value": round(n / (t_all / 1e3) / 1e6, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "one pass of the full front end (order, gradient, C_k, D0, D_{d-1}) on the crop %s of "
                      "the same field, all %d host threads; per-stage ms below" % (
                          "x".join(str(x) for x in crop.shape), cores),
            "one_thread": {"value": round(n / (t_one / 1e3) / 1e6, 4), "unit": UNIT, "stages_ms": st_one},
            "all_cores": {"value": round(n / (t_all / 1e3) / 1e6, 4), "unit": UNIT, "threads": cores,
                          "stages_ms": st_all},
            "host": host_cpu_info(),
            "note": "the oracle fans out only the per-vertex gradient over threads (the paper's "
                    "parallel structure, P:1121-1124); order, C_k sort and the union-finds are sequential. "
                    "3D: stages_ms.d1_and_generators is the oracle's sequential Alg. 3 + Sec. 9 generators on "
                    "the same crop (not in value)"}


def max_over_ranks(value, dist):
    """The timing rule for N > 1: every rank times its own replica, the job time is the
    maximum over ranks (all_reduce MAX; NCCL on the GPU box, gloo in the CPU test)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(n_vertices_per_rank, world, steps, ms_total):
    """whole-job throughput: vertices processed by all ranks / the (max) job time"""
    return world * n_vertices_per_rank * steps / (ms_total / 1e3) / 1e6


def make_field(cfg, seed):
    from synth import fields

    return fields.make(cfg, seed=seed)


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle, as it stands, timed on the host cores.  Each
    step is one full front-end pass (order + gradient + C_k + D0 + D_{d-1}) on a fixed
    crop of this config's field (a bounded sample: the whole c4 field takes the oracle
    ~9 min on 8 cores, tests/golden/fullsize_c4.json)."""
    if rank != 0:
        return
    import numpy as np

    f = make_field(args.config, 0)
    side = {3: 96, 2: 1024, 1: 1 << 20}[f.ndim]
    crop = np.ascontiguousarray(f[tuple(slice(0, min(side, s)) for s in f.shape)])
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_timed(crop, cores)
    dt, per = 0.0, {}
    for _ in range(args.steps):
        t, st = oracle_timed(crop, cores)
        dt += t / 1e3
        for k, v in st.items():
            per[k] = per.get(k, 0.0) + v / args.steps
    value = crop.size * args.steps / dt / 1e6
    sample = "crop %s of the %s field, full front end (order, gradient, C_k, D0, D_{d-1}), %d threads" % (
        "x".join(str(x) for x in crop.shape), args.config, cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 in, integer arithmetic (oracle)", "data": "synthetic",
        "config": {"workload": args.config, "desc": CONFIG_DESC[args.config], "N": int(f.size)},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "stages_ms_per_step": {k: round(v, 2) for k, v in per.items()}, "host": host_cpu_info()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="dms", choices=["dms", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-d1", action="store_true", help="skip the D1 / generator timing (3D)")
    ap.add_argument("--complex", default="freudenthal", choices=["freudenthal", "5tet"],
                    help="5tet: the paper's five-tetrahedra cut of the 3D configs (SURVEY 8(f) #4; no D1, "
                         "no cpu_baseline leg)")
    args = ap.parse_args()
    if args.complex == "5tet":
        args.no_d1 = True
        args.no_cpu_baseline = True

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch

    import paper_2206_13932_b200 as dms

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    f_host = make_field(args.config, seed=rank)
    N = f_host.size
    ndim = f_host.ndim
    f_dev = torch.from_numpy(f_host).cuda()
    stream = torch.cuda.current_stream()
    if args.complex == "5tet" and ndim != 3:
        raise SystemExit("--complex 5tet needs a 3D config")
    ctx = dms.DMS(f_dev, stream, complex=args.complex)
    rank_buf = torch.empty(N, dtype=torch.int32, device="cuda")
    grad_buf = torch.empty(dms.dms_gradient_bytes(ctx.ctx), dtype=torch.uint8, device="cuda")

    def step():
        ctx.run_all(rank_buf, grad_buf)
        # the step's results are complete once the diagram calls return (they sync)
        dms.dms_diagram0(ctx.ctx)
        dms.dms_diagram_top(ctx.ctx)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count()
    dms.dms_set_timing(ctx.ctx, True)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    stages = dms.dms_stage_ms(ctx.ctx)
    dms.dms_set_timing(ctx.ctx, False)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()

    ms_total = max_over_ranks(ms_total, dist)
    ms_step = ms_total / args.steps
    value = job_value(N, world, args.steps, ms_total)

    counts, _ = dms.dms_critical(ctx.ctx)
    ncrit = counts[: ndim + 1]
    _, nd0 = dms.dms_diagram0(ctx.ctx)
    _, ndt = dms.dms_diagram_top(ctx.ctx)
    bmin_e2e, bmin_grad = algorithmic_bytes(N, ndim, ncrit, nd0 + ndt)
    peak, peak_kind = load_peaks()
    g_ms = stages["gradient_kernel"] / max(1, stages["gradient_launches"])
    g_ach = bmin_grad / (g_ms / 1e3) / 1e9
    kernel_name = {3: "k_gradient_pool<3,8,1,true> (closed-form lower-star gradient + critical records)",
                   2: "k_gradient_lut2 (2D lower-star gradient by table lookup + critical records)",
                   1: "k_gradient1 (1D lower-star gradient + critical records)"}[ndim]
    if args.complex == "5tet":
        kernel_name = "k_gradient_t5 (ProcessLowerStars on the five-tetrahedra stars + critical records)"
    # roofline: the dominant kernel's ALGORITHMIC bytes per launch
    # (N (4 + G_w) + 8 sum|C_k|) over its average launch time (CUDA events on the
    # library's stream, inside the timed region) against the measured HBM peak
    roofline = {"kernel": kernel_name, "bound": "hbm", "achieved": round(g_ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(g_ach / peak, 4), "traffic": None, "peak_kind": peak_kind,
                "ms_per_launch": round(g_ms, 4), "algorithmic_bytes_per_launch": int(bmin_grad)}
    # per-stage and end-to-end fractions of the HBM roofline (SURVEY 8(d) per-stage minima:
    # a1 8 B/v; a2+a3 (4 + G_w) B/v + 8 sum|C_k|; a4-a8 32 B per output pair)
    def frac(nbytes, ms):
        return round(nbytes / (ms / 1e3) / 1e9 / peak, 5) if ms and ms > 0 else None

    st_ms = {k: v / args.steps for k, v in stages.items() if k != "gradient_launches"}
    roofline["stages"] = {
        "a1_order": frac(8.0 * N, st_ms.get("order")),
        "a2_a3_gradient_critical": frac(bmin_grad, st_ms.get("gradient", 0) + st_ms.get("critical", 0)),
        "a4_a8_diagrams": frac(32.0 * (nd0 + ndt), max(st_ms.get("d0", 0), st_ms.get("dtop", 0))),
        "end_to_end": frac(bmin_e2e, ms_step),
        "end_to_end_of_8TBps": round(bmin_e2e / (ms_step / 1e3) / 8e12, 5),
        "note": "order runs beside the gradient on a second stream and D0 beside D_{d-1}: stage times overlap",
    }
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tr = None
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                tr = json.load(fh).get(args.config)
        except Exception:
            tr = None
    if tr and args.complex == "5tet":
        tr = None  # the ncu traffic figures are the Freudenthal kernel's
    if tr:
        roofline["traffic"] = tr["bytes_per_launch"]
        roofline["traffic_source"] = tr.get("source")
        if tr.get("warp_inst_per_launch"):
            # the kernel is bound by integer issue (ncu: ALU pipe busy, DRAM a few %): its
            # issue rate, warp instructions per launch (ncu, fixed for the input) over the
            # live launch time against 1 warp instruction / cycle / SMSP x 148 SMs x 4 SMSPs
            # at the sampled SM clock
            issue_peak = 148 * 4 * (clk.get("sm_mhz") or 1965.0) * 1e6
            ach = tr["warp_inst_per_launch"] / (g_ms / 1e3)
            roofline["issue"] = {
                "bound": "alu", "achieved": round(ach / 1e9, 1), "peak": round(issue_peak / 1e9, 1),
                "unit": "G warp-inst/s", "frac": round(ach / issue_peak, 3),
                "warp_inst_per_launch": tr["warp_inst_per_launch"],
                "peak_kind": "derived: 148 SMs x 4 SMSPs x 1 warp-instruction/cycle x sampled SM clock",
                "lane_efficiency": tr.get("lane_efficiency"), "alu_pipe_pct_ncu": tr.get("alu_pipe_pct")}

    # end to end through the public API: pinned host input -> device, run, diagrams back
    e2e = None
    if not args.no_e2e:
        f_pin = torch.from_numpy(f_host).pin_memory()
        h2d = f_pin.numel() * 4

        # pinned destinations for the diagrams (grown on demand, outside the timed steps)
        pin_out = [torch.empty(0, dtype=torch.uint8).pin_memory() for _ in range(2)]

        def e2e_step():
            # the public host-input call: the upload overlaps the gradient slab by slab
            ctx.run_all_host(f_pin, rank_buf, grad_buf)
            a = ctx.diagram0(out=pin_out[0])
            b = ctx.diagram_top(out=pin_out[1])
            return a.nbytes + b.nbytes

        ctx.run_all(rank_buf, grad_buf)
        for k, fn in enumerate((dms.dms_diagram0, dms.dms_diagram_top)):
            need = fn(ctx.ctx)[1] * dms.PAIR_DTYPE.itemsize  # same field every step
            pin_out[k] = torch.empty(need + (1 << 20), dtype=torch.uint8).pin_memory()
        d2h = e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            d2h = e2e_step()
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = max_over_ranks(t0.elapsed_time(t1), dist)
        e2e = {"value": round(job_value(N, world, args.steps, ms_e2e), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(ms_e2e / args.steps, 3)}

    # D1 (Alg. 3 PairCriticalSimplices + the Sec. 9 generators, 3D only):
    # timed after the front end, by the library's stage events (the diagrams it consumes
    # are recomputed by run_all each step but not counted)
    d1 = None
    if ndim == 3 and not args.no_d1:
        def d1_step():
            ctx.run_all(rank_buf, grad_buf)
            dms.dms_diagram1(ctx.ctx)
            dms.dms_generators(ctx.ctx)

        d1_step()
        torch.cuda.synchronize()
        dms.dms_set_timing(ctx.ctx, True)
        for _ in range(args.steps):
            d1_step()
        st = dms.dms_stage_ms(ctx.ctx)
        dms.dms_set_timing(ctx.ctx, False)
        _, n1 = dms.dms_diagram1(ctx.ctx)
        po, _, _ = dms.dms_generators(ctx.ctx)
        off = np.empty(n1 + 1, dtype=np.int64)
        ctx._copy(off.ctypes.data, po, off.nbytes)
        rr = np.zeros(2, dtype=np.int32)
        import ctypes as _ct
        L = dms.lib()
        L.dms_internal_d1_rounds.argtypes = [_ct.c_void_p, _ct.c_void_p]
        ntaint = int(L.dms_internal_d1_rounds(ctx.ctx, rr.ctypes.data))
        ms_p, ms_g = st["d1"] / args.steps, st["generators"] / args.steps
        d1 = {"pairs": int(n1), "generator_edges": int(off[-1]), "rounds": [int(rr[0]), int(rr[1])],
              "rerun_for_generators": ntaint,
              "ms_pairs": round(ms_p, 4), "ms_generators": round(ms_g, 4),
              "mvertices_per_s_pairs": round(N / ms_p / 1e3, 1) if ms_p > 0 else None,
              "mpairs_per_s": round(n1 / ms_p / 1e3, 2) if ms_p > 0 else None,
              "output_bytes": int(32 * n1 + 8 * (n1 + 1) + 8 * int(off[-1])),
              "note": "latency-bound propagation rounds (host reads the active count per round); "
                      "ms include the round-trip gaps; pairs = |C1| - |D0| = |C2| - |D2|"}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_oracle_sample(f_host)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 in, integer arithmetic (ordered uint32 keys)", "data": "synthetic",
            "config": {"workload": args.config, "desc": CONFIG_DESC[args.config], "N": N, "complex": args.complex,
                       "l2": "input (%d MB) larger than L2; no flush" % (N * 4 >> 20),
                       "parallelism": "replicas" if world > 1 else "single"},
            "stages_ms_per_step": {k: round(v / args.steps, 4) for k, v in stages.items() if k != "gradient_launches"},
            # per stage as throughput: N / t_stage; stages on the concurrent
            # streams overlap, so these do not add up to the step
            "stages_mvertices_per_s": {k: round(N / (v / args.steps) / 1e3, 1) for k, v in stages.items()
                                       if k in ("order", "gradient", "critical", "d0", "dtop") and v > 0},
            "counts": {"critical": ncrit, "d0_pairs": nd0, "dtop_pairs": ndt},
            "roofline": roofline,
            "d1": d1,
            "cpu_baseline": cpu_base,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
