"""Benchmark: fV-SRN network evals/s and ms/frame of 1024^2 DVR on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A step is one DVR frame of the configuration's workload (default config 2:
fV-SRN 4x32, 32^3x16 latent grid, m=14, 1024^2, stepsize 1/256 = 1 voxel of a
256^3 field, grayscale TF), cycling through the 8 fibonacci_cameras views.
Weights are random-init (ModelConfig seed 0); there is no dataset.

* value  -- evals/s with the model resident in HBM, device-timed with CUDA events
            around each frame on the launching stream (L2 flushed before every
            frame, outside the events), max over ranks.
* e2e    -- the same metric through the public API call a user makes
            (render_image -> fvsrn_render: per-frame constants host->device,
            framebuffer device->host inside the timed region).
* roofline -- tensor-core FLOPs of the unpadded MLP per eval (7,168 at 4x32)
            x evals per frame / frame time, vs MEASURED_PEAKS.json bf16 burst.
* cpu_baseline -- the reference itself (staged into oracle/_ref by oracle/stage_ref.sh;
            the numpy/numba port when absent) on the box's host cores: all cores on the
            same bounded row sample the reference arm times, plus one `taskset -c 0`
            single-core run; CPU model stated (oracle/ref_runner.py).
* --impl reference -- the reference arm: the same reference code on all host cores,
            each step that row sample of view (step mod 8), rank 0 only.

`--gpus N` without WORLD_SIZE in the environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU; it fails if fewer than N GPUs exist,
unless FVSRN_BENCH_ONE_GPU=1 puts every rank on GPU 0 to exercise the multi-rank path).
Under torchrun (N > 1) every rank renders its round-robin share of 8x8 screen tiles
straight into rank 0's frame in peer memory (CUDA IPC over NVLink; FVSRN_MULTI=gather:
NCCL gather + reassembly), and every timed frame ends with a device-side cross-rank
completion (an NCCL all-reduce on each rank's stream), so rank 0's frame time covers
every rank's tiles.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_fvsrn_b200")

METRIC = "fV-SRN network evals/sec and ms/frame at 1024² DVR (1/2/4/8 B200) vs CPU ref"

CONFIGS = {
    "cfg1": dict(model=dict(layers=4, hidden=32, grid_resolution=16, grid_channels=16, seed=0),
                 res=256, stepsize=1 / 128, kind="dvr",
                 desc="config 1: fV-SRN 4x32, 16^3x16 grid, m=14, DVR 256^2, stepsize 1/128"),
    "cfg2": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0),
                 res=1024, stepsize=1 / 256, kind="dvr",
                 desc="config 2: fV-SRN 4x32, 32^3x16 grid, m=14, DVR 1024^2, stepsize 1/256 "
                      "(1 voxel of a 256^3 field)"),
    "cfg3": dict(model=dict(layers=6, hidden=64, grid_resolution=64, grid_channels=16,
                            fourier_m=30, seed=0),
                 res=1024, stepsize=1 / 768, kind="dvr",
                 desc="config 3: fV-SRN 6x64, 64^3x16 grid, m=30, DVR 1024^2, stepsize 1/768 "
                      "(1 voxel of a 512x336x768 Jet-shaped field)"),
    "cfg4": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0),
                 res=256, kind="decode",
                 desc="config 4: batched world-space density decode of the 256^3 lattice "
                      "(config-2 weights)"),
    "cfg5": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16,
                            keyframe_times=[1, 11, 21], seed=0),
                 res=4096, stepsize=1 / 256, kind="dvr", t=6.5,
                 desc="config 5: time-varying fV-SRN (3 keyframes, R32 F16), t=6.5, DVR 4096^2, "
                      "stepsize 1/256"),
}


def mlp_flops(cfg: dict) -> int:
    """2 * sum(in_i * out_i) over the unpadded layer widths."""
    from paper_2112_01579_b200 import ModelConfig

    c = ModelConfig(**cfg)
    dims = [c.input_width] + [c.hidden] * (c.layers - 1) + [c.output_width]
    return 2 * sum(a * b for a, b in zip(dims[:-1], dims[1:]))


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period: float = 0.05):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def mufu_per_eval_of(model_cfg: dict, kernel: str) -> int:
    """MUFU (XU-pipe) instructions per evaluation in the launched kernel: one MUFU.COS per
    hidden activation except the ones evaluated on the FMA pipe (packed HFMA2 pairs in both
    kernel families, the f32 polynomial in the tcgen05 dot-product rows), plus MUFU.TANH for
    the sigmoid head and, in the
    march, MUFU.EX2 for alpha.  The NeRF base sin/cos run on
    the FMA pipe in the mma.sync kernels (FVSRN_FOURIER_POLY=1) and on MUFU.SIN/COS in the
    tcgen05 kernels (3 axes x 2)."""
    layers, hid = model_cfg["layers"], model_cfg["hidden"]
    tc = kernel.startswith(("dvr_tc", "decode_tc"))
    decode = kernel.startswith("decode")
    if not tc:
        # mma.sync kernels (fvsrn_device.cuh, FVSRN_MMA_H2): every 4th n8 column tile of a
        # snake_alt row evaluates its cosines in HFMA2 arithmetic
        return (layers - 1) * (hid - hid // 4) + (1 if decode else 2)
    # fvsrn_tc.cu, per 32-column segment of a hidden row: every 3rd packed fp16 word
    # (FVSRN_TC_H2 / FVSRN_TC_H2_64) evaluates both cosines in HFMA2 arithmetic; the
    # density head's last hidden row, when it is an f32 dot product on the FMA pipe
    # (64-wide march, 32/64-wide decode), keeps the per-element pattern (every 5th column
    # at 32-wide, every 6th column of each 32-column half at 64-wide)
    seg = max(hid // 32, 1)
    h2_words = sum(1 for g in range(16) if g % 3 == 2)
    row_h2 = hid - seg * 2 * h2_words
    row_dot = hid - ((hid + 1) // 5 if hid <= 32 else seg * (33 // 6))
    dot_last = hid >= (32 if decode else 64)
    rows = [row_h2] * (layers - 1)
    if dot_last:
        rows[-1] = row_dot
    return sum(rows) + (1 if decode else 2) + 6


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1590.0), "measured (MEASURED_PEAKS.json bf16_tflops burst)"
    return 1590.0, "fallback (B200_PROFILING.md 1.59 PFLOP/s)"


def _kernel_key(name: str) -> str:
    """'void fvsrn::dvr_tc_kernel<(int)32, (int)14, ...>(...)' / 'dvr_tc_kernel<32,14,...> (...)'
    -> 'dvr_tc_kernel<32,14,...>'"""
    n = name.replace("void ", "").replace("fvsrn::", "").replace("(int)", "").replace("(bool)", "")
    n = n.split("(")[0] if "<" not in n.split("(")[0] else n[: n.index(">") + 1]
    return n.replace(" ", "")


def ncu_traffic(config: str, kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/ncu_summary.json), used only when that capture is of the kernel this run
    launched; otherwise null."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        with open(p) as f:
            d = json.load(f)
        e = d.get(config, {})
        if e and _kernel_key(e.get("kernel", "")) == _kernel_key(kernel):
            return e.get("dram_bytes_per_launch"), e
    return None, {}


# ------------------------------------------------------------------ CPU legs (reference)
# Bounded sample of one frame per config: every k-th row of a view (rays are independent,
# so the rows cost what they cost inside the full frame); cfg 1 and the cfg 4 decode are
# timed whole.  The reference arm and the all-core cpu_baseline use the same sample.
CPU_ROW_STRIDE = {"cfg1": 1, "cfg2": 2, "cfg3": 64, "cfg5": 64}
CPU_SINGLE_STRIDE = {"cfg1": 4, "cfg2": 32, "cfg3": 256, "cfg5": 512, "cfg4": 32}


def host_cores() -> int:
    """Cores this process may run on (the affinity mask, not the machine's CPU count)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
CPU_DECODE_ARM_STRIDE = 16          # reference arm, cfg 4: x slabs [::16] per step


# (render_image threads, NUMBA_NUM_THREADS, BLAS threads) for the reference on this box's
# c cores, per config: the fastest of the candidates measured on the bench's own samples
# (tools/ref_sweep.sh, profiles/r2/ref_sweep.txt; 16 cores: cfg 2 at threads 8 x numba 2
# 11.2 M evals/s vs 8.8 (16 x 1), 6.0 (4 x 4), 1.5 (1 x 16)).  The reference's numpy glue
# holds the GIL and its naive 6x64 path calls threaded BLAS, so neither extreme wins.
REF_BEST = {"cfg1": ("c/4", 4, 4), "cfg2": ("c/2", 2, 2), "cfg3": (1, 1, "c"),
            "cfg5": ("c/2", 2, 2), "cfg4": (1, 1, "c")}


def ref_threads(cores: int, config: str = "cfg2") -> tuple[int, int, int]:
    """(render_image `threads`, NUMBA_NUM_THREADS, BLAS threads) for the reference;
    FVSRN_REF_THREADS / FVSRN_REF_NUMBA / FVSRN_REF_BLAS override."""
    def val(v):
        if isinstance(v, str):
            return max(1, cores // int(v[2:]) if "/" in v else cores)
        return v
    best = [val(v) for v in REF_BEST.get(config, ("c/2", 2, 2))]
    return (int(os.environ.get("FVSRN_REF_THREADS", best[0])),
            int(os.environ.get("FVSRN_REF_NUMBA", best[1])),
            int(os.environ.get("FVSRN_REF_BLAS", best[2])))


def _ref_env(threads_numba_blas) -> dict:
    _, numba, blas = threads_numba_blas
    return {"NUMBA_NUM_THREADS": str(numba), "OMP_NUM_THREADS": str(blas),
            "OPENBLAS_NUM_THREADS": str(blas), "MKL_NUM_THREADS": str(blas)}


def cpu_leg(config: str, cores: int, row_stride: int, step: int = 0, single: bool = False,
            timeout: float = 240.0):
    """oracle/ref_runner.py in a subprocess (its own thread settings; `taskset -c 0` for the
    single-core run); returns its JSON result or {"error": ...}."""
    import subprocess

    tnb = (1, 1, 1) if single else ref_threads(cores, config)
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", **_ref_env(tnb))
    cmd = [sys.executable, "-m", "oracle.ref_runner", "--config", config,
           "--threads", str(tnb[0]), "--step", str(step)]
    cmd += ["--full"] if row_stride == 1 else ["--row-stride", str(row_stride)]
    if single:
        cmd = ["taskset", "-c", "0"] + cmd
    try:
        r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 -- reported in the JSON line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def cpu_baseline(config: str):
    cores = host_cores()
    kind = CONFIGS[config]["kind"]
    allc = cpu_leg(config, cores, 1 if kind == "decode" else CPU_ROW_STRIDE[config],
                   timeout=420.0)
    one = cpu_leg(config, 1, CPU_SINGLE_STRIDE[config], single=True)
    if "error" in allc:
        return {"value": None, "unit": "evals/s", "cores": cores, "kind": "unavailable",
                "sample": allc["error"]}
    tnb = ref_threads(cores, config)
    out = {"value": allc["value"], "unit": "evals/s", "cores": cores, "kind": allc["kind"],
           "sample": allc["sample"] + f", render_image threads={tnb[0]}, NUMBA_NUM_THREADS="
                                      f"{tnb[1]}, BLAS threads={tnb[2]}",
           "seconds": allc["seconds"], "cpu_model": allc.get("cpu_model"),
           "single_core": ({"value": one["value"], "cores": 1, "sample": one["sample"] +
                            ", taskset -c 0, NUMBA_NUM_THREADS=1", "seconds": one["seconds"]}
                           if "error" not in one else one),
           "note": ("the reference package itself (fvsrn 0.1.0 staged into oracle/_ref), "
                    "through camera_rays + render_rays chunks exactly as render_image composes "
                    "them (render.py:314-332), ModelSource(use_fused=" +
                    ("True" if CONFIGS[config]["model"]["hidden"] <= 32 else "False") + ")")
           if allc["kind"] == "reference" else "numpy+numba port (oracle/fvsrn_oracle.py)"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on the host cores, rank 0 only."""
    if rank != 0:
        return
    cores = host_cores()
    tnb = ref_threads(cores, args.config)
    os.environ.update(_ref_env(tnb))                     # before numba / numpy's BLAS start
    from oracle.ref_runner import Runner, cpu_model

    cfg = CONFIGS[args.config]
    runner = Runner(args.config, tnb[0])
    runner.warm()
    if cfg["kind"] == "dvr":
        stride = CPU_ROW_STRIDE[args.config]
        step = lambda i: runner.render_step(i, stride)             # noqa: E731
        sample = (f"{args.config}: " + (f"whole frame of view (step mod 8)" if stride == 1 else
                  f"every {stride}th row of view (step mod 8) ({cfg['res'] // stride} rows per step)")
                  + f", render_image threads={tnb[0]}, NUMBA_NUM_THREADS={tnb[1]}, BLAS threads={tnb[2]}")
    else:
        stride = CPU_DECODE_ARM_STRIDE
        step = lambda i: runner.decode(stride)                   # noqa: E731
        sample = (f"{args.config}: decode_volume's chunked eval_density over lattice x slabs "
                  f"[::{stride}], NUMBA_NUM_THREADS={tnb[1]}")
    for i in range(args.warmup):
        runner.warm()
    tot_n = tot_t = 0.0
    for i in range(args.steps):
        n, dt = step(i)
        tot_n += n
        tot_t += dt
    value = tot_n / tot_t
    line = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 MLP, f64 ray setup/compositing (reference numpy + numba)",
            "data": "synthetic (random-init weights, ModelConfig seed 0; fibonacci_cameras(8) views)",
            "config": {"workload": cfg["desc"], "sample": sample,
                       "evals_per_step_mean": tot_n / args.steps},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores,
                             "kind": runner.kind, "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU
def relaunch(n: int):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N
    ranks on this node (rendezvous on 127.0.0.1).  Fails if fewer than N GPUs are visible,
    unless FVSRN_BENCH_ONE_GPU=1 (all ranks share GPU 0: tests the multi-rank path only)."""
    import socket

    if os.environ.get("FVSRN_BENCH_ONE_GPU") != "1":
        import torch

        have = torch.cuda.device_count()
        if have < n:
            sys.exit(f"bench.py --gpus {n}: only {have} GPU(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py")] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--csv", default=None,
                    help="append a row to this benchmark.csv (SURVEY section 5 columns) and write "
                         "manifest.json beside it")
    ap.add_argument("--check-frame", action="store_true",
                    help="N>1: compare the assembled frame with a 1-GPU render on rank 0")
    ap.add_argument("--checkpoint", default=None,
                    help="render this .fvsrn checkpoint (same shape as the config) instead of the "
                         "random-init model, e.g. tests/golden/trained_cfg2.fvsrn (trained weights: "
                         "the upload-time probe may select the exact-weight grid sampler)")
    ap.add_argument("--grid-precision", default="f16", choices=["f16", "u8"],
                    help="u8: the latent grid round-trips through a u8 .fvsrn checkpoint "
                         "(grid_quantize, grid.py:157-166) and is sampled as 8-bit codes")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus)          # does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # FVSRN_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo (exercises the multi-rank code
    # paths on a single-GPU box; the timing is then meaningless)
    one_gpu = os.environ.get("FVSRN_BENCH_ONE_GPU") == "1"
    dev = 0 if one_gpu else local
    torch.cuda.set_device(dev)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2112_01579_b200 as P
    from paper_2112_01579_b200.sharding import PeerFrameRenderer, TileShardRenderer

    cfg = CONFIGS[args.config]
    model = P.model_init(P.ModelConfig(**cfg["model"]))
    if args.checkpoint:
        model = P.checkpoint_load(args.checkpoint)
        want = P.ModelConfig(**cfg["model"])
        got = model.config
        if (got.layers, got.hidden, got.grid_resolution, got.grid_channels, got.input_width) != \
                (want.layers, want.hidden, want.grid_resolution, want.grid_channels, want.input_width):
            sys.exit(f"--checkpoint {args.checkpoint} does not have the {args.config} shape")
    if args.grid_precision == "u8":
        import tempfile

        with tempfile.TemporaryDirectory() as td:
            P.checkpoint_save(model, Path(td) / "m.fvsrn", "f16", "u8")
            model = P.checkpoint_load(Path(td) / "m.fvsrn")
    flops = mlp_flops(cfg["model"])
    t_frame = cfg.get("t")
    # temporal configs animate: every frame is at a different timestep, so every frame
    # re-blends its keyframe pair (the latent interpolation is inside the timed region)
    t_cycle = [t_frame + 0.75 * k for k in range(8)] if t_frame is not None else [None] * 8

    def t_of(i):
        return t_cycle[i % 8]
    res = cfg["res"]
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    if cfg["kind"] == "dvr":
        src = P.ModelSource(model, P.TF_PRESETS["grayscale"], t=t_frame, use_fused=True)
        cams = P.fibonacci_cameras(8, res, res)
        settings = P.RenderSettings(stepsize=cfg["stepsize"])
        peer = world > 1 and os.environ.get("FVSRN_MULTI", "peer") == "peer"
        if peer:
            # tiles stored straight into rank 0's frame over NVLink P2P by the render
            # kernel (CUDA IPC); no gather / reassembly (sharding.PeerFrameRenderer).
            # If any rank cannot map the frame, all ranks fall back to the NCCL gather.
            from paper_2112_01579_b200.sharding import PeerUnavailable
            renderer = PeerFrameRenderer(src)
            try:
                renderer._frame(res, res)
            except PeerUnavailable as e:
                if rank == 0:
                    print(f"bench: {e}; using the NCCL gather path", file=sys.stderr)
                peer = False
        if peer:

            def step(i, count_ptr=None):
                _, ptr, _ = renderer._frame(res, res, slot=i % renderer.NBUF)
                renderer.dm.render_device(src.tf, cams[i % 8], settings, t_of(i), ptr, count_ptr,
                                          stream.cuda_stream, rank=rank, world=world, compact=False)
        elif world > 1:
            renderer = TileShardRenderer(src)

            def step(i, count_ptr=None):
                renderer.dm.render_device(src.tf, cams[i % 8], settings, t_of(i),
                                          renderer._buffers(res, res)[0].data_ptr(), count_ptr,
                                          stream.cuda_stream, rank=rank, world=world, compact=True)
                local_buf, gathered, frame, _ = renderer._buffers(res, res)
                if rank == 0:
                    dist.gather(local_buf, gather_list=list(gathered.unbind(0)), dst=0)
                    from paper_2112_01579_b200.device import tiles_to_frame_device
                    tiles_to_frame_device(gathered.data_ptr(), res, res, world, frame.data_ptr(),
                                          stream.cuda_stream)
                else:
                    dist.gather(local_buf, gather_list=None, dst=0)
        else:
            frame = torch.empty((res, res, 4), dtype=torch.float32, device="cuda")

            def step(i, count_ptr=None):
                src.device_model.render_device(src.tf, cams[i % 8], settings, t_of(i),
                                               frame.data_ptr(), count_ptr, stream.cuda_stream)
    else:  # decode: lattice split in contiguous slabs across ranks
        total = res ** 3
        per = -(-total // world)
        begin, count = rank * per, max(0, min(per, total - rank * per))
        vol = torch.empty(max(count, 1), dtype=torch.float32, device="cuda")
        dm = P.device.device_model(model)

        def step(i, count_ptr=None):
            dm.decode_device(res, t_frame, begin, count, vol.data_ptr(), stream.cuda_stream)

    # ---- warm-up
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    # ---- evaluated-sample counts (same frames as the timed loop, counted once)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    evals_per_step = []
    for i in range(args.steps):
        if cfg["kind"] == "dvr":
            cnt.zero_()
            step(i, cnt.data_ptr())
            torch.cuda.synchronize()
            c = cnt.clone()
            if world > 1:
                dist.all_reduce(c)
            evals_per_step.append(int(c.item()))
        else:
            evals_per_step.append(res ** 3)
    total_evals = sum(evals_per_step)

    # ---- timed region
    from paper_2112_01579_b200 import device as DEV

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    done = torch.zeros(1, dtype=torch.int32, device="cuda")

    def complete():
        """Cross-rank frame completion inside the timed region: every rank's tiles have
        landed before this rank's end event (NCCL: an all-reduce ordered after the render
        on every rank's stream; gloo test mode: host synchronisation + barrier)."""
        if world == 1:
            return
        if dist.get_backend() == "nccl":
            dist.all_reduce(done)
        else:
            torch.cuda.synchronize()
            dist.barrier()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    DEV.kernel_timer(True)      # CUDA events around the dominant kernel, launch counts
    with ClockSampler(dev) as clocks:
        for i in range(args.steps):
            flush.zero_()                      # evict the L2 (outside the events)
            evs[i][0].record(stream)
            step(i)
            complete()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dom_ms, dom_launches, lib_launches = DEV.kernel_timer_read()
    kernel_desc = DEV.kernel_timer_info()
    DEV.kernel_timer(False)
    per_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = torch.tensor([sum(per_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot_ms, op=dist.ReduceOp.MAX)
    tot_ms = float(tot_ms.item())
    value = total_evals / (tot_ms / 1e3)
    ms_per_step = tot_ms / args.steps

    # ---- end-to-end through the public API (host buffers, copies inside the timing)
    e2e = e2e_viewer = None
    if not args.no_e2e:
        if cfg["kind"] == "dvr":
            if world == 1:
                # (1) the stock call a reference caller makes, render_image(src, cam,
                # settings): a fresh Image every frame (its array is page-locked memory
                # recycled by the library once the previous frame is dropped)
                img = None
                for i in range(2):
                    img = P.render_image(src, cams[i % 8], settings)
                with ClockSampler(dev) as e2e_clocks:
                    t0 = time.perf_counter()
                    n_e = 0
                    for i in range(args.steps):
                        src.t = t_of(i)
                        img = P.render_image(src, cams[i % 8], settings)
                        n_e += src.last_eval_count
                    dt = time.perf_counter() - t0
                del img
                # (2) an interactive viewer's loop: one caller-owned page-locked framebuffer
                fb = P.pinned_empty((res, res, 4))
                for i in range(2):
                    P.render_image(src, cams[i % 8], settings, out=fb)
                t1 = time.perf_counter()
                n_v = 0
                for i in range(args.steps):
                    src.t = t_of(i)
                    P.render_image(src, cams[i % 8], settings, out=fb)
                    n_v += src.last_eval_count
                dtv = time.perf_counter() - t1
                e2e_viewer = {"value": n_v / dtv, "unit": "evals/s", "ms_per_step": 1e3 * dtv / args.steps,
                              "api": "render_image(ModelSource, cam, settings, out=pinned_empty(...)) "
                                     "(one reused caller-owned page-locked framebuffer)"}
                h2d = 4356 + 4 * 32
                d2h = res * res * 16 + 8
            else:
                host = torch.empty((res, res, 4), dtype=torch.float32, pin_memory=True)
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                n_e = 0
                for i in range(args.steps):
                    src.t = t_of(i)
                    out = renderer.render(cams[i % 8], settings, count=True)
                    n_e += renderer.last_eval_count
                    if rank == 0:
                        host.copy_(out)
                torch.cuda.synchronize()
                dist.barrier()
                dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                dt = float(dt.item())
                h2d = 4356 + 4 * 32
                d2h = res * res * 16 if rank == 0 else 0
        else:
            # the stock call: a fresh ScalarVolume per call (page-locked, recycled by the
            # library once the previous volume is dropped; two warm-up calls populate it)
            vol = None
            for i in range(2):
                vol = P.decode_volume(model, res, t=t_frame)
            t0 = time.perf_counter()
            for i in range(args.steps):
                vol = P.decode_volume(model, res, t=t_frame)
            dt = time.perf_counter() - t0
            del vol
            n_e = args.steps * res ** 3
            h2d, d2h = 4 * 32, res ** 3 * 4
        e2e = {"value": n_e / dt, "unit": "evals/s", "h2d_bytes_per_step": h2d,
               **({"clocks": e2e_clocks.summary()} if cfg["kind"] == "dvr" and world == 1 else {}),
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * dt / args.steps,
               "api": ("render_image(ModelSource(model, tf), cam, settings) -> fvsrn_render: host "
                       "frame returned per call; the kernels store each pixel into it over PCIe "
                       "(page-locked, recycled)" if world == 1 else
                       "PeerFrameRenderer.render + rank-0 host copy (torchrun ranks)")
               if cfg["kind"] == "dvr" else "decode_volume(model, 256) -> fvsrn_decode_density "
                                            "(host volume returned per call)"}

    frame_check = None
    if args.check_frame and world > 1 and cfg["kind"] == "dvr":
        src.t = t_of(0)
        got = renderer.render(cams[0], settings)      # every rank takes part
        if rank == 0:
            want, _ = src.device_model.render(src.tf, cams[0], settings, src.t)
            frame_check = bool(np.array_equal(got.cpu().numpy(), want))

    def finish():
        if world > 1:
            dist.barrier()
            if cfg["kind"] == "dvr" and isinstance(renderer, PeerFrameRenderer):
                renderer.close()           # release rank 0's frame mapping before it is freed
                dist.barrier()
            dist.destroy_process_group()

    if rank != 0:
        finish()
        return

    peak, peak_src = measured_peaks()
    # rank 0's dominant-kernel time (the march / decode kernel alone, CUDA events on its
    # stream); its algorithmic FLOPs are rank 0's share of the evaluations
    rank0_evals = total_evals / world
    achieved = rank0_evals * flops / (dom_ms / 1e3) / 1e12
    traffic, ncu = ncu_traffic(args.config, kernel_desc)
    mufu_per_eval = mufu_per_eval_of(cfg["model"], kernel_desc)
    sm_mhz = clocks.summary().get("sm_mhz") or 1965.0
    xu_peak = 16 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_mhz * 1e6
    xu_achieved = rank0_evals * mufu_per_eval / (dom_ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f16 MMA operands / f32 accumulate, f64 ray setup",
        "data": "synthetic (random-init weights, ModelConfig seed 0; fibonacci_cameras(8) views)",
        "config": {"workload": cfg["desc"], "views": 8 if cfg["kind"] == "dvr" else None,
                   "evals_per_step_mean": total_evals / args.steps,
                   "ms_per_frame_median": statistics.median(per_ms),
                   "l2": "flushed before every frame (256 MiB memset, outside the events)",
                   "parallelism": (f"screen-tile dp{world} ("
                                   + ("peer-memory frame via CUDA IPC/NVLink"
                                      if os.environ.get("FVSRN_MULTI", "peer") == "peer"
                                      else "NCCL gather + reassembly") + ")")
                   if world > 1 else "1 GPU",
                   "tf": "grayscale", "t": t_cycle if t_frame is not None else None,
                   "grid_precision": args.grid_precision,
                   "weights": args.checkpoint or "random init (ModelConfig seed 0)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "flops_per_eval": flops, "peak_source": peak_src,
                     "kernel": kernel_desc, "kernel_ms_per_launch": dom_ms / max(1, dom_launches),
                     "kernel_share_of_step": dom_ms / tot_ms if world == 1 else None,
                     "xu_pipe": {"mufu_per_eval": mufu_per_eval, "achieved_Gops": xu_achieved / 1e9,
                                 "peak_Gops": xu_peak / 1e9, "frac": xu_achieved / xu_peak,
                                 "note": "MUFU (16/clk/SM): one cos per hidden activation not "
                                         "evaluated as a packed HFMA2 pair or f32 polynomial on "
                                         "the FMA pipe, 6 NeRF base sin/cos (tcgen05 kernels), one "
                                         "tanh (sigmoid head), one ex2 (alpha); see DESIGN.md "
                                         "sections 3-4"},
                     **({"ncu": ncu} if ncu else {})},
        "gpu_launches": lib_launches,
        "clocks": clocks.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if e2e_viewer is not None:
        line["e2e_viewer"] = e2e_viewer
    if frame_check is not None:
        line["config"]["frame_bit_identical_to_1gpu"] = frame_check
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, args.config, world, line)
    finish()


def write_csv(path: str, config: str, world: int, line: dict) -> None:
    """benchmark.csv + manifest.json, the reference's artefact convention (cli.py:64-76):
    columns config,gpus,res,spr,evals,ms_per_frame,evals_per_s,roofline_frac."""
    import platform

    cfg = CONFIGS[config]
    p = Path(path)
    p.parent.mkdir(parents=True, exist_ok=True)
    new = not p.exists()
    spr = round(1.0 / cfg["stepsize"]) if cfg["kind"] == "dvr" else ""
    with open(p, "a") as f:
        if new:
            f.write("config,gpus,res,spr,evals,ms_per_frame,evals_per_s,roofline_frac\n")
        f.write(f"{config},{world},{cfg['res']},{spr},{line['config']['evals_per_step_mean']:.0f},"
                f"{line['ms_per_step']:.4f},{line['value']:.6g},{line['roofline']['frac']:.4f}\n")
    import torch

    manifest = {"config": {k: v for k, v in cfg.items() if k != "desc"}, "workload": cfg["desc"],
                "seed": cfg["model"].get("seed", 0), "gpus": world,
                "versions": {"fvsrn_b200": __import__("paper_2112_01579_b200").__version__,
                             "torch": torch.__version__, "cuda": torch.version.cuda,
                             "python": platform.python_version(),
                             "device": torch.cuda.get_device_name(0)},
                "kernel": line["roofline"].get("kernel")}
    with open(p.parent / "manifest.json", "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
