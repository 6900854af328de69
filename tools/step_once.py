"""Run one eager key step and one tail step of a config (for ncu launch lists).

    python tools/step_once.py [--config c3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2411_01171_b200.executor import ExecConfig  # noqa: E402
from paper_2411_01171_b200.harness import Denoiser, initial_latent  # noqa: E402
from paper_2411_01171_b200.unet import UNetConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--backend", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--detail", action="store_true")
ap.add_argument("--key-only", action="store_true", help="one key step, no tail step")
ap.add_argument("--tail", action="store_true", help="--detail profiles the tail (rehash) step instead")
ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays of one key and one tail step")
a = ap.parse_args()
cfg = UNetConfig(**CONFIGS[a.config])
den = Denoiser(cfg, ExecConfig(gemm_backend=a.backend), K=2)
den.set_latent(initial_latent(cfg))
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    den.plan.run_full(st, den.emb_table[0].data_ptr())
    if not a.key_only:
        den.plan.run_tail(st)
torch.cuda.synchronize()
print("ok", len(den.plan.units), "units")
if a.detail:
    from paper_2411_01171_b200 import _native as N
    from paper_2411_01171_b200.profiling import gemm_flops
    recs = []
    orig = N.call

    def rec(name, *args):
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        orig(name, *args)
        e_.record()
        info = ""
        if name == "sf_gemm":
            g = args[0]
            info = (f"mode={g.mode} M={g.n_outer * g.n_inner} N={g.N} K={g.cin * (9 if g.mode == 1 else 3 if g.mode == 2 else 1)}"
                    f" batch={g.batch} be={N.query('sf_gemm_backend', g)}")
            recs.append((name, info, s_, e_, gemm_flops(g)))
        elif name in ("sf_group_norm_apply", "sf_layer_norm", "sf_group_norm_stats"):
            fr, ni, c = args[2:5] if name != "sf_group_norm_stats" else args[1:4]
            nbytes = fr * ni * c * 2 * (1 if name == "sf_group_norm_stats" else 2)
            info = f"frames={fr} inner={ni} C={c} bytes={nbytes}"
            recs.append((name, info, s_, e_, -nbytes))
        else:
            recs.append((name, info, s_, e_, 0.0))
    N.call = rec
    if a.tail:
        den.plan.run_tail(st)
    else:
        den.plan.run_full(st, den.emb_table[0].data_ptr())
    torch.cuda.synchronize()
    N.call = orig
    for name, info, s_, e_, fl in recs:
        ms = s_.elapsed_time(e_)
        if fl < 0:
            print(f"{ms*1e3:9.1f} us  {-fl / (ms * 1e6):7.1f} GB/s  {name} {info}")
        else:
            print(f"{ms*1e3:9.1f} us  {fl/ (ms*1e9) if fl else 0:7.1f} TF  {name} {info}")
if a.graph:
    def graph_time(fn, reps=20):
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                fn(cs.cuda_stream)
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        for _ in range(reps):
            g.replay()
        e_.record()
        torch.cuda.synchronize()
        return s_.elapsed_time(e_) / reps
    key_ms = graph_time(lambda sp: den.plan.run_full(sp, den.emb_table[0].data_ptr()))
    tail_ms = graph_time(lambda sp: den.plan.run_tail(sp))
    print(f"graph replay: key step {key_ms:.3f} ms, tail step {tail_ms:.3f} ms")
