#!/usr/bin/env python
"""bench.py -- RL iterations/s of the B200 light-field Richardson-Lucy hot path (AutoDeconJ, arXiv 2208.11422).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...      (depth/phase sharding over NCCL)
    torchrun --nproc-per-node N ... bench.py --config c5 ...   (time-lapse: frame replicas, frame-batched RL)

A step is one RL iteration = every row of SURVEY §8(a) a2..a9 (forward projection, ratio, backward
projection, multiplicative update, z max-projection, fp64 DCT entropy, stop-rule bookkeeping with the
argmax snapshot), on the BASELINE config the metric is quoted on (c3: Nnum=15, 1005x1005, 51 planes).
Timing: W untimed iterations, then exactly K iterations inside one lfm_rl_iterate call, bracketed by
barrier + cudaDeviceSynchronize, measured with CUDA events on the launching stream, max over ranks.
The dominant kernel's duration comes from the library's per-stage CUDA events over the same timed region.
Inputs are larger than L2: every projection streams the 58.9 GB transfer matrices (L2 = 126 MB).
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

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, lf_like, plane_support, poisson  # noqa: E402

METRIC = "RL iterations/s (Nnum=15 LFM, 1/2/4/8 B200) and % of HBM roofline"
UNIT = "iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-calls", type=int, default=2, help="timed lfm_deconvolve_host calls (after one untimed "
                    "warm-up call that allocates the staging buffers)")
    ap.add_argument("--cpu-rows", type=int, default=256, help="rows of the oracle's bounded CPU sample (~10-30 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flags", type=int, default=0, help="lfm_plan_create flags (2 = direct path)")
    ap.add_argument("--frames", type=int, default=32, help="c5: frames per GPU per lockstep batch (8/16/32 with the default "
                    "LFM_PLAN_FRAMES plan; 2/4/8/16 with --flags 4)")
    return ap.parse_args()


def workload_desc(cfg):
    ks = sorted({plane_support(cfg, z) for z in range(cfg.nz)})
    return (f"{cfg.name}: Nnum={cfg.nnum}, {cfg.height}x{cfg.width} image, {cfg.nz} depth planes, "
            f"Gaussian-parallax PSF K_max={cfg.k_max} (per-plane support {ks[0]}..{ks[-1]}), "
            f"{cfg.phantom} phantom + Poisson noise, auto-stop policy (max 50)")


# ------------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks line")
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if "Active" == r[4 + i]})
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------------------------------------
# CPU baseline: the oracle, as it stands, on a bounded sample of the same workload
# ------------------------------------------------------------------------------------------------
def oracle_iteration_seconds(cfg, h64, x64, y64, rows):
    """Times the oracle's forward projection on `rows` output rows and its backward projection on the
    same rows of every plane (the two terms of one RL iteration), plus the full-size elementwise RL
    update and metric, and extrapolates to one full iteration.  The oracle scans the PSF's per-plane
    support once per call (a fixed cost a full-size call pays once, not once per row): it is timed on its own
    (a forward call over zero rows scans every plane) and kept out of the per-row extrapolation."""
    from oracle import lfm_oracle as O
    H = cfg.height
    r0 = max(0, H // 2 - rows // 2)
    r1 = min(H, r0 + rows)
    t0 = time.perf_counter()
    O.forward_project(x64, h64, rows=(r0, r0))
    t_scan = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.forward_project(x64, h64, rows=(r0, r1))
    t_fwd = time.perf_counter() - t0
    r = np.ones((cfg.height, cfg.width))
    nz = cfg.nz
    t_bwd = 0.0
    import ctypes
    lib = O._load()
    out = np.zeros((nz, cfg.height, cfg.width))
    kh = h64.shape[3]
    for z in range(nz):
        t0 = time.perf_counter()
        lib.lfmo_backward(O._dp(r), O._dp(h64), nz, cfg.nnum, kh, kh, cfg.height, cfg.width, 0, nz * cfg.nnum ** 2,
                          ctypes.c_long(z * H + r0), ctypes.c_long(z * H + r1), O._dp(out))
        t_bwd += time.perf_counter() - t0
    t0 = time.perf_counter()
    xs = x64 * 1.0001 / np.maximum(x64, 1e-6)          # full-size elementwise update cost (same shapes)
    reg = O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height, cfg.width)
    O.evaluate_iteration(xs, reg)
    O.ratio_image(y64, y64)
    t_el = time.perf_counter() - t0
    scale = H / (r1 - r0)
    # forward: one scan of every plane per call; backward: each per-plane call scans its own plane (all planes
    # together: one scan of every plane)
    per_iter = (max(t_fwd - t_scan, 0.0) + max(t_bwd - t_scan, 0.0)) * scale + 2 * t_scan + t_el
    return per_iter, dict(t_fwd=t_fwd, t_bwd=t_bwd, t_scan=t_scan, t_elementwise=t_el, rows=r1 - r0)


def oracle_flops_per_iteration(cfg):
    """Multiply-adds of the oracle's direct convolution per RL iteration (forward + backward over each plane's
    non-zero K(z) x K(z) support), 2 flops each: 4 H W sum_z K(z)^2."""
    return 4.0 * cfg.height * cfg.width * sum(plane_support(cfg, z) ** 2 for z in range(cfg.nz))


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the fp64 oracle (this tier's reference arm), each step a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import lfm_oracle as O
    cfg = CONFIGS[args.config]
    h64 = gen_psf(cfg, np.float32).astype(np.float64)
    x64 = gen_volume(cfg, 1, np.float64)
    y64 = lf_like(cfg, 7)
    O.build()
    cores = cpu_cores()
    rows = min(cfg.height, max(2, 8 * cores))   # 8 rows per core: every OpenMP thread gets work, per-call overheads
    # stay small against the extrapolated rows (4 per core measured 0.015-0.026 it/s across boxes)
    for _ in range(args.warmup):
        oracle_iteration_seconds(cfg, h64, x64, y64, rows)
    ts, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ts.append(oracle_iteration_seconds(cfg, h64, x64, y64, rows)[0])
        walls.append(time.perf_counter() - t0)
    sec = float(np.mean(ts))
    value = 1.0 / sec
    sample = (f"per step: oracle forward on {rows} of {cfg.height} output rows + backward on the same rows of all "
              f"{cfg.nz} planes + full-size update/metric, extrapolated to one iteration (the per-call PSF support "
              f"scan timed separately and counted once)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "gflops": oracle_flops_per_iteration(cfg) * value / 1e9},
            # ms_per_step is the extrapolated full iteration; the sample a step actually runs takes wall_s_per_step
            "wall_s_per_step": float(np.mean(walls)), "sample_rows": rows,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2208_11422_b200 import lfm as L

    cfg = CONFIGS[args.config]
    t_setup = time.perf_counter()
    side = torch.cuda.Stream()          # a real stream: CUDA-graph replay (LFM_PLAN_GRAPHS) cannot use the legacy one
    torch.cuda.set_stream(side)
    h = gen_psf(cfg, np.float32)
    xt = gen_volume(cfg, 1, np.float32)
    nccl_id = None
    if world > 1:
        obj = [L.lfm_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()
    plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), rank=rank, world=world,
                  nccl_id=nccl_id, flags=args.flags)
    info = plan.info()
    del h
    H, W, nz = cfg.height, cfg.width, cfg.nz
    # measurement y = Poisson(H x_true) using the product's own forward projection
    xt_d = torch.from_numpy(xt).cuda()
    yh_d = torch.zeros((H, W), device="cuda")
    plan.forward(xt_d, yh_d)
    torch.cuda.synchronize()
    y = poisson(np.maximum(yh_d.cpu().numpy().astype(np.float64), 0.0), 101).astype(np.float32)
    del xt_d
    y_d = torch.from_numpy(y).cuda()
    x_d = torch.zeros((nz, H, W), device="cuda")
    setup_s = time.perf_counter() - t_setup

    # warm-up
    plan.rl_iterate(y_d, x_d, L.make_policy(mode="fixed", n_iters=args.warmup))
    torch.cuda.synchronize()

    # timed region: exactly K iterations (no per-stage events: graph modes stay on)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    res = plan.rl_iterate(y_d, x_d, L.make_policy(mode="fixed", n_iters=args.steps, init_from_x=True))
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    # per-stage breakdown (roofline launch times, stage shares): a separate profiled run of the same K iterations
    plan.profile(True)
    plan.profile_read(reset=True)
    plan.rl_iterate(y_d, x_d, L.make_policy(mode="fixed", n_iters=args.steps, init_from_x=True))
    torch.cuda.synchronize()
    prof = plan.profile_read(reset=True)
    plan.profile(False)
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps / (ms / 1e3)

    # roofline of the dominant kernel (algorithmic bytes at the minimal alias-free transform size)
    N2 = cfg.nnum ** 2
    nu = info["fft_units"]            # units streamed by the MAC kernels (hybrid plan: frequency-path units)
    kap_min = info["lc_min_h"] * (info["lc_min_w"] // 2 + 1)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak = json.load(open(peaks_path))["hbm_gbs"]
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    stage_ms = {k: prof["ms"][k] / max(1, prof["count"][k]) for k in prof["ms"]}
    # per-kernel launch times, CUDA events on the stream (SM partition) each kernel runs on
    kern_ms = {{"mac_fwd": "fwd_mac", "mac_bwd": "bwd_mac", "tc_fwd": "dir_fwd", "tc_bwd": "dir_bwd"}[k]:
               max(1e-6, prof["kern_ms"][k] / max(1, prof["kern_count"][k])) for k in prof["kern_ms"]}
    parts = info["partition_sms"]     # [fwd, bwd] x [tensor-core SMs, MAC SMs]; 0 = whole GPU, one after the other
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    mac_sms = {"fwd_mac": parts[0][1] or nsm, "bwd_mac": parts[1][1] or nsm}
    tc_sms = {"dir_fwd": parts[0][0] or nsm, "dir_bwd": parts[1][0] or nsm}
    alg = {
        "fwd_mac": kap_min * N2 * nu * 8 + kap_min * nu * 8 + kap_min * N2 * 8,   # M + G + Y
        "bwd_mac": kap_min * N2 * nu * 8 + kap_min * N2 * 8 + kap_min * nu * 8,   # M + R + Xh
    }
    ntile = info.get("tiles", 0)
    if ntile:   # tiled frequency path: per tile group L x (L/2+1) frequencies per window, every tile
        # per pass -- M (or M^T) of the group's units + the tiles' spectra in and out, summed over groups (lfm_info)
        alg = {"fwd_mac": info["fft_bytes"], "bwd_mac": info["fft_bytes"]}
    if info["fft_units"] == 0:
        dom = max(("dir_fwd", "dir_bwd"), key=lambda k: stage_ms[k])
        roof = {"bound": "alu", "kernel": dom, "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None,
                "traffic": None}
    else:
        dom = max(("fwd_mac", "bwd_mac"), key=lambda k: kern_ms[k])
        achieved = alg[dom] / (kern_ms[dom] / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            for key, ent in tj.items():   # a capture of the same config and plan (frequency-path unit count)
                if key.split("_")[0] == cfg.name and ent.get("fft_units") == nu and ent.get("tiles", 0) == ntile:
                    traffic = ent.get(dom)
        roof = {"bound": "hbm", "kernel": (dom + " (mac_f16_kernel, tiles)") if ntile else dom,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg[dom], "avg_launch_ms": kern_ms[dom],
                "sms": mac_sms[dom],
                "partition_note": "on an SM partition (DESIGN.md §5.5) the MAC shares the GPU with the tensor-core "
                                  "kernel; its stream rate is bounded per SM, not by HBM" if parts[0][0] else None,
                "both": {k: {"avg_ms": kern_ms[k], "achieved_gbs": alg[k] / (kern_ms[k] / 1e3) / 1e9, "sms": mac_sms[k],
                             "frac": alg[k] / (kern_ms[k] / 1e3) / 1e9 / peak} for k in alg}}
    # secondary roofline: the tcgen05 direct kernel (tensor-bound), per projection stage
    roof_tc = None
    if info.get("tc_planes", 0) > 0:
        pk = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
        # the direct path runs kind::f16 MMAs (fp16 operands, fp32 accumulation) at the dense fp16 = bf16 rate
        f16_sus = pk.get("bf16_tflops_sustained", 1400.0)
        f16_burst = pk.get("bf16_tflops", 1590.0)
        peak_src_tc = ("MEASURED_PEAKS.json bf16_tflops (burst, measured near the max SM clock this step runs at; "
                       "fp16 = bf16 dense rate), / 3 for the 3-product fp16 split" if "bf16_tflops" in pk else
                       "fallback 1.59 PFLOP/s bf16 (B200_PROFILING.md), / 3")
        t = {k: kern_ms[k] for k in ("dir_fwd", "dir_bwd")}
        kk = max(t, key=lambda k: t[k])
        ex = info["tc_flops_executed"] / (t[kk] / 1e3) / 1e12
        al = info["tc_flops_algorithmic"] / (t[kk] / 1e3) / 1e12
        peak3 = f16_burst / 3.0   # an fp32-accurate contraction on fp16 tensor cores costs 3 products (3xFP16)
        tc_traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            for key, ent in json.load(open(tpath)).items():
                if (key.split("_")[0] == cfg.name and ent.get("fft_units") == info["fft_units"]
                        and ent.get("tiles", 0) == ntile):
                    tc_traffic = ent.get("tcdir_" + kk.split("_")[1])
        roof_tc = {"bound": "tensor", "kernel": "tcdir_kernel (" + kk.split("_")[1] + ")",
                   "achieved": al, "peak": peak3, "unit": "TFLOP/s", "frac": al / peak3,
                   "sms": tc_sms[kk], "frac_of_partition_peak": al / (peak3 * tc_sms[kk] / nsm),
                   "traffic": tc_traffic, "avg_launch_ms": t[kk],
                   "algorithmic_flops_per_launch": info["tc_flops_algorithmic"],
                   "achieved_is": "algorithmic fp32 flops (SURVEY 8(d): 2*H*W*K(z)^2 non-zero taps per plane) / kernel time",
                   "peak_source": peak_src_tc,
                   "frac_vs_sustained_peak": al / (f16_sus / 3.0),
                   "executed_tensor_tflops": ex, "executed_frac_of_f16_burst_peak": ex / f16_burst,
                   "executed_frac_of_f16_sustained_peak": ex / f16_sus,
                   "peak_note": "primary peak = the burst GEMM (this step runs near the max SM clock, see 'clocks'); "
                                "the sustained GEMM of MEASURED_PEAKS ran power-capped (median "
                                f"{pk.get('clocks_under_load', {}).get('sm_mhz_median', 'n/a')} MHz), its fraction "
                                "is the secondary field",
                   "executed_is": "issued tcgen05 kind::f16 flops (3 products over the union tap boxes and the tiles' "
                                  "column ranges, skipped windows excluded)",
                   "tc_planes": info["tc_planes"], "kernel_ms": t}
    # the dominant kernel carries the primary roofline: the largest SM-time (launch time x SMs of its partition) per
    # iteration -- with SM partitions the longest launch can be the one on the smaller partition
    roof_primary = roof
    if roof_tc is not None:
        sm_t_tc = sum(kern_ms[k] * tc_sms[k] for k in ("dir_fwd", "dir_bwd"))
        sm_t_mac = sum(kern_ms[k] * mac_sms[k] for k in ("fwd_mac", "bwd_mac")) if info["fft_units"] else 0.0
        if sm_t_tc > sm_t_mac:
            roof_primary = roof_tc
    share = {k: prof["ms"][k] / max(1e-9, sum(prof["ms"].values())) for k in prof["ms"]}

    # e2e: the public host-buffer call, auto-stop deconvolution of the same measurement
    y_host = torch.from_numpy(y).pin_memory()
    x_host = torch.zeros((nz, H, W), dtype=torch.float32).pin_memory()
    e2e_iters, e2e_s, auto, call_s, d2h = 0, 0.0, None, [], 0
    plan.deconvolve_host(y_host.numpy(), x_host.numpy(), L.make_policy(mode="auto", max_iters=50))   # warm-up
    plan.profile_read(reset=True)   # the library counts the device -> host bytes it moves (lfm_profile_t.d2h_bytes)
    for _ in range(max(1, args.e2e_calls)):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = plan.deconvolve_host(y_host.numpy(), x_host.numpy(), L.make_policy(mode="auto", max_iters=50))
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
        if dist:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s += float(tt.item())
        call_s.append(round(float(tt.item()), 4))
        e2e_iters += r["stop_iter"]
        auto = r
    # device -> host bytes of the timed calls as the library counted them: the 8-byte E_k read per iteration and the
    # volume copies (improving iterates once the E curve flattens, copied while the loop runs, or the final copy)
    d2h = plan.profile_read(reset=True)["d2h_bytes"]
    s = auto["series"]
    k = auto["stop_iter"]
    margin = min(abs(s[i] - s[i - 1]) / abs(s[i]) for i in range(1, k)) if k > 1 else None
    calls = max(1, args.e2e_calls)
    e2e = {"value": e2e_iters / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(H * W * 4 * calls / e2e_iters),
           "d2h_bytes_per_step": int(d2h / e2e_iters),
           "step": "one RL iteration of an auto-stop lfm_deconvolve_host call (host y in, host argmax volume out: "
                   "improving iterates after the E curve flattens (gain < 1 %) copied while the next iteration runs, "
                   "else once after the loop; plus 8 bytes of E_k per iteration; d2h counted by the library); "
                   f"{calls} timed call(s) after one warm-up call, {e2e_iters} iterations",
           "call_s": call_s}

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            h64 = gen_psf(cfg, np.float32).astype(np.float64)
            sec, det = oracle_iteration_seconds(cfg, h64, xt.astype(np.float64), y.astype(np.float64), args.cpu_rows)
            cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                   "sample": (f"oracle (fp64 direct conv, OpenMP) forward on {det['rows']} of {H} rows + backward on the "
                              f"same rows of all {nz} planes + full-size update/metric, extrapolated to one iteration "
                              f"({det['t_fwd'] + det['t_bwd'] + det['t_elementwise']:.1f} s measured; the per-call PSF "
                              f"support scan, {det['t_scan']:.2f} s, counted once per call)"),
                   "gflops": oracle_flops_per_iteration(cfg) / sec / 1e9,
                   "gflops_is": "4*H*W*sum_z K(z)^2 direct-convolution flops per iteration / oracle seconds per iteration"}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": workload_desc(cfg),
                "parallelism": f"depth/phase (z,a)-unit sharding over {world} GPU(s), NCCL allreduce sum+max per iteration"
                if world > 1 else "single GPU",
                "transform": (f"overlap-save tiles in {info['tile_groups']} group(s) (one window geometry per coarse-tap "
                              f"range; first: {info['tiles']} windows of {info['fft_h']}x{info['fft_w']} coarse pixels, "
                              f"{info['tile_T1']}x{info['tile_T2']} valid outputs each; whole-image alias-free minimum "
                              f"{info['lc_min_h']})" if info.get("tiles") else
                              f"coarse {info['fft_h']}x{info['fft_w']} (alias-free minimum {info['lc_min_h']})")
                if not info["direct"] else "direct spatial",
                "transfer_matrix_gb_per_gpu": info["transfer_bytes"] / 1e9,
                "hybrid": {"direct_planes": info["direct_planes"], "tc_planes": info["tc_planes"], "fft_units": info["fft_units"], "planes_moved_for_memory": info["planes_moved_for_memory"]},
                "l2": "inputs larger than L2: each projection streams the transfer matrices (L2 126 MB)",
                "plan_ms": info["plan_ms"], "setup_s": setup_s,
                "auto_stop": {"stop_iter": auto["stop_iter"], "best_iter": auto["best_iter"],
                              "decision_margin": margin, "series": s},
                "stage_share": share, "stage_avg_ms": stage_ms, "kernel_avg_ms": kern_ms,
                "sm_partitions": {"forward": {"tc_sms": parts[0][0], "mac_sms": parts[0][1]},
                                  "backward": {"tc_sms": parts[1][0], "mac_sms": parts[1][1]},
                                  "note": "0 = the projection's tensor-core and frequency-path halves run one after "
                                          "the other on the whole GPU"},
            },
            "roofline": roof_primary,
            "roofline_mac": roof,
            "roofline_tc": roof_tc,
            "cpu_baseline": cpu,
            "paper_context": "AutoDeconJ reports 4.4x faster deconvolution than the MATLAB GUI of Prevedel et al. 2014 "
                             "(P:17, P:33); hardware, image size and iteration count not stated -- context only",
            "e2e": e2e,
            "gpu_launches": prof["launches"],
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    plan.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_c5(args):
    """c5 (BASELINE configs[4]): time-lapse of c3-geometry frames, frame-parallel across GPUs (one process per GPU,
    each rank an independent replica of the plan holding its own slice of the frames; no per-iteration
    communication -- SURVEY §8(e) "Frame parallelism (c5). Replicas only") and frame-batched lockstep RL within a
    GPU.  A step = one lockstep iteration of every rank's batch of F frames (fixed mode); value = frame-
    iterations/s of the whole job (world x F x K / max-over-ranks device time), "scaling": "weak".  After the timed
    region every rank runs its batch to auto-stop and rank 0 gathers every frame's (stop, best) iterations."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2208_11422_b200 import lfm as L
    from lfm_inputs import gen_somata
    cfg = CONFIGS["c3"]
    F = args.frames
    # a plan built for frame batches (all planes on the frequency path, fp16-split transfer matrices)
    flags = args.flags or L.LFM_PLAN_FRAMES
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    stream = torch.cuda.current_stream()
    h = gen_psf(cfg, np.float32)
    H, W, nz = cfg.height, cfg.width, cfg.nz
    rng = np.random.default_rng(7)
    phase = rng.uniform(0, 2 * np.pi, cfg.n_objects)
    frames = [rank * F + f for f in range(F)]   # this rank's slice of the time-lapse
    ys = []
    with L.Plan(h, cfg.nnum, H, W, optics=L.make_optics(**OPTICS)) as fplan:   # single-frame plan forms the y
        for g in frames:   # soma intensities 1 + 0.5 sin(2 pi g / 64 + phi_i), noise seed 1000 + g
            xt = torch.from_numpy(gen_somata(cfg, 1, np.float32, modulation=1 + 0.5 * np.sin(2 * np.pi * g / 64 + phase))).cuda()
            yh = torch.zeros((H, W), device="cuda")
            fplan.forward(xt, yh)
            torch.cuda.synchronize()
            ys.append(poisson(np.maximum(yh.cpu().numpy().astype(np.float64), 0), 1000 + g).astype(np.float32))
            del xt
    torch.cuda.empty_cache()
    plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=flags)
    info = plan.info()
    del h
    yb = torch.from_numpy(np.stack(ys)).cuda()
    xb = torch.zeros((F, nz, H, W), device="cuda")
    plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=args.warmup))
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=args.steps, init_from_x=True))
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # per-stage breakdown: a profiled re-run of the same K iterations
    plan.profile(True)
    plan.profile_read(reset=True)
    plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=args.steps, init_from_x=True))
    prof = plan.profile_read(reset=True)
    plan.profile(False)
    groups = {"transforms_x": "r2c_x", "fwd_mac_batch": "fwd_mac", "per_frame_forward_rest": "c2r_yhat",
              "bwd_mac_batch": "bwd_mac", "per_frame_update_rest": "c2r_update"}
    stage_ms = {g: prof["ms"][k] / max(1, prof["count"][k]) for g, k in groups.items()}
    # the time-lapse result: every frame to auto-stop, (stop, best) gathered on rank 0 (volumes stay on their GPU)
    auto = plan.rl_iterate_batch(yb, xb, L.make_policy(mode="auto", max_iters=50))
    mine = [(g, auto["stop_iter"][i], auto["best_iter"][i]) for i, g in enumerate(frames)]
    allf = [None] * world
    if dist:
        dist.all_gather_object(allf, mine)
    else:
        allf = [mine]
    if rank == 0:
        per_frame = sorted(x for part in allf for x in part)
        line = {"metric": "frame-iterations/s (c5 time-lapse, frame-parallel replicas x frame-batched lockstep RL)",
                "value": world * F * args.steps / (ms / 1e3), "unit": "frame-iterations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"c5: time-lapse frames of the c3 geometry (Nnum=15, 1005x1005, 51 planes), "
                                       f"{F} frames per GPU per lockstep batch, {world * F} frames in the job",
                           "parallelism": f"frame replicas over {world} GPU(s), no per-iteration communication",
                           "frames_per_batch": F, "plan_flags": flags, "fft_units": info["fft_units"],
                           "l2": "inputs larger than L2: every batched pass streams the 58.9 GB transfer matrices",
                           "auto_stop_per_frame": [{"frame": g, "stop_iter": st, "best_iter": b} for g, st, b in per_frame],
                           "batch_stage_avg_ms": stage_ms},
                "gpu_launches": prof["launches"], "clocks": clk}
        print(json.dumps(line), flush=True)
    plan.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_c5(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
