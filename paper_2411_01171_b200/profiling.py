"""Per-launch device timing of a compiled program (CUDA events on the launch stream).

Wraps every C-ABI call of one eager (non-graph) pass with a pair of CUDA
events recorded on the stream the kernel is launched on, then aggregates by
entry point.  For ``sf_gemm`` the algorithmic FLOPs of each launch
(2*M*N*K*batch, K = taps*cin) are recorded, so the bench can report the GEMM
kernel's achieved TFLOP/s against the measured bf16 peak.
"""

from __future__ import annotations

from collections import defaultdict

import torch

from . import _native as N


def gemm_flops(args) -> float:
    taps = {N.GEMM_PLAIN: 1, N.GEMM_CONV3X3: 9, N.GEMM_TCONV3: 3}[args.mode]
    return 2.0 * args.n_outer * args.n_inner * args.N * taps * args.cin * args.batch


def gemm_bytes(args) -> float:
    """Algorithmic HBM bytes of one sf_gemm launch: activations read once (implicit-GEMM taps
    re-read from L2, not HBM), weights once (per batch when batched), output written once,
    residual read once."""
    taps = {N.GEMM_PLAIN: 1, N.GEMM_CONV3X3: 9, N.GEMM_TCONV3: 3}[args.mode]
    rows = args.n_outer * args.n_inner * args.batch
    a = rows * args.cin * 2 if args.a_bstride or args.batch == 1 else args.n_outer * args.n_inner * args.cin * 2
    b = args.N * taps * args.cin * 2 * (args.batch if args.w_bstride else 1)
    out = rows * args.N * (4 if args.out_fp32 else 2)
    res = rows * args.N * 2 if args.res.ptr else 0
    return float(a + b + out + res)


class CallProfiler:
    def __init__(self):
        self.records = []  # (name, start_event, end_event, flops, backend)
        self._orig = None

    def __enter__(self):
        self._orig = N.call

        def timed(name, *a):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            stream = torch.cuda.current_stream()
            s.record(stream)
            self._orig(name, *a)
            e.record(stream)
            flops, be, nbytes = 0.0, 0, 0.0
            if name == "sf_gemm":
                args = a[0]
                flops = gemm_flops(args)
                nbytes = gemm_bytes(args)
                be = N.query("sf_gemm_backend", args)
                name = f"sf_gemm[{'tcgen05' if be == 2 else 'mma.sync'}]"
            elif name == "sf_spatial_attention_core":
                frames, hw, c = a[4], a[5], a[6]
                flops = 4.0 * frames * hw * hw * c          # S = q k^T and P v
            elif name == "sf_temporal_attention_core":
                b, t, n_inner, c = a[4], a[5], a[6], a[7]
                flops = 4.0 * b * n_inner * t * t * c
            elif name == "sf_temporal_attention_fused":
                b, t, n_inner, c = a[4], a[5], a[6], a[7]
                # the reference op's algorithmic work: four C x C projections + two T x T products
                flops = b * n_inner * (8.0 * t * c * c + 4.0 * t * t * c)
            self.records.append((name, s, e, flops, nbytes))
        N.call = timed
        return self

    def __exit__(self, *exc):
        N.call = self._orig

    def mixed_roofline(self, peak_tflops: float, peak_gbps: float, prefix: str = "sf_gemm") -> dict:
        """Per launch the roofline time max(flops / tensor peak, bytes / HBM peak); the ratio of
        their sum to the measured sum is the family's fraction of its own (mixed) roofline."""
        torch.cuda.synchronize()
        ideal = actual = 0.0
        hbm_bound = n = 0
        for name, s, e, fl, nb in self.records:
            if not name.startswith(prefix):
                continue
            t_tc, t_hbm = fl / (peak_tflops * 1e9), nb / (peak_gbps * 1e6)   # ms
            ideal += max(t_tc, t_hbm)
            actual += s.elapsed_time(e)
            hbm_bound += t_hbm > t_tc
            n += 1
        return {"launches": n, "hbm_bound_launches": hbm_bound, "roofline_ms": round(ideal, 4),
                "measured_ms": round(actual, 4), "frac": round(ideal / actual, 4) if actual else None}

    def summary(self) -> dict:
        torch.cuda.synchronize()
        agg = defaultdict(lambda: {"calls": 0, "ms": 0.0, "flops": 0.0})
        for name, s, e, fl, _ in self.records:
            a = agg[name]
            a["calls"] += 1
            a["ms"] += s.elapsed_time(e)
            a["flops"] += fl
        total = sum(v["ms"] for v in agg.values())
        for v in agg.values():
            v["share"] = v["ms"] / total if total else 0.0
            v["tflops"] = v["flops"] / (v["ms"] * 1e9) if v["ms"] and v["flops"] else 0.0
        return {"total_ms": total, "by_call": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))}
