"""Command-line front end over the device path.

    python -m paper_2411_01171_b200 run          [--mode M] [config flags] --out DIR   -> run_report.json
    python -m paper_2411_01171_b200 compare      --modes reference,slicedloop,...  --out DIR -> compare.json
    python -m paper_2411_01171_b200 similarity   [config flags] --out DIR            -> similarity.csv + .json
    python -m paper_2411_01171_b200 search-steps --similarity FILE (--gamma G | --target-count N) --out DIR
                                                                                       -> schedule.json
    python -m paper_2411_01171_b200 export       [config flags] --out DIR            -> graph.json + weights.slfw

run / compare / similarity take ``--graph graph.json --weights weights.slfw`` (as
written by ``export`` or by the reference's Graph.save / WeightBundle.save) in
place of rebuilding the network from the config.

Exit codes: 0 success, 1 runtime error, 2 validation error (the
message names the failing field).  Every flag is validated before any device
work, and every artefact is written inside ``--out``.  ``search-steps`` runs on
the host only; the other subcommands need the CUDA library (no CPU fallback).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from .errors import SliceflowError, ValidationError
from .modes import ExecMode


class _Usage(ValidationError):
    """Flag / config validation failure (exit 2)."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):           # argparse exits 2 itself; keep one error path
        raise _Usage(message)


def _unet_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--config", help="JSON file with UNetConfig fields (and optional run fields)")
    for name, typ in (("frames", int), ("height", int), ("width", int), ("channels", int),
                      ("base-channels", int), ("norm-groups", int), ("steps", int), ("seed", int)):
        p.add_argument(f"--{name}", type=typ)
    p.add_argument("--spatial-k", type=int, help="spatial slices per group (frames per slice = T / k)")
    p.add_argument("--temporal-k", type=int, help="temporal slices (pixel bands) per group")
    p.add_argument("--temporal-kh", type=int, help="temporal tiles along H (temporal_k = kh * kw)")
    p.add_argument("--temporal-kw", type=int, help="temporal tiles along W")
    p.add_argument("--dtype", default="bfloat16", choices=["bfloat16"],
                   help="device storage type (the device path computes bf16 x bf16 -> fp32)")
    p.add_argument("--out", required=True, help="output directory")


def _model_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--graph", help="saved graph JSON (Graph.save) to run instead of the built network")
    p.add_argument("--weights", help="SLFW weight bundle (WeightBundle.save) for --graph")


def _model_files(args):
    """(graph, weights) loaded from --graph / --weights, or (None, None)."""
    if (args.graph is None) != (args.weights is None):
        raise _Usage("--graph and --weights are given together")
    if args.graph is None:
        return None, None
    from .graph import Graph
    from .weights import WeightBundle
    try:
        graph = Graph.load(args.graph)
    except (OSError, ValueError, KeyError, TypeError) as e:
        raise _Usage(f"graph: {e}") from None
    try:
        weights = WeightBundle.load(args.weights)
    except (OSError, ValueError, KeyError) as e:
        raise _Usage(f"weights: {e}") from None
    return graph, weights


def _positive(args, name):
    v = getattr(args, name.replace("-", "_"), None)
    if v is not None and v < 1:
        raise _Usage(f"{name} must be >= 1")
    return v


def _unet_cfg(args):
    from .unet import UNetConfig
    fields = {}
    if args.config:
        try:
            with open(args.config) as f:
                doc = json.load(f)
        except (OSError, json.JSONDecodeError) as e:
            raise _Usage(f"config: {e}") from None
        known = {f.name for f in UNetConfig.__dataclass_fields__.values()}
        for k, v in doc.get("unet", doc).items():
            if k not in known:
                raise _Usage(f"config: unknown field {k!r}")
            fields[k] = tuple(v) if isinstance(v, list) else v
    for name in ("frames", "height", "width", "channels", "base_channels", "norm_groups", "steps", "seed"):
        v = getattr(args, name)
        if v is not None:
            if v < (0 if name == "seed" else 1):
                raise _Usage(f"{name.replace('_', '-')} must be >= {0 if name == 'seed' else 1}")
            fields[name] = v
    try:
        return UNetConfig(**fields)
    except (TypeError, ValueError) as e:
        raise _Usage(f"config: {e}") from None


def _exec_cfg(args):
    from .executor import ExecConfig
    sk = _positive(args, "spatial-k")
    tk = _positive(args, "temporal-k")
    kh, kw = _positive(args, "temporal-kh"), _positive(args, "temporal-kw")
    if kh or kw:
        tk = (kh or 1) * (kw or 1)
    return ExecConfig(spatial_k=sk, temporal_k=tk)


def _mode(text: str) -> ExecMode:
    try:
        return ExecMode(text)
    except ValueError:
        raise _Usage(f"mode must be one of {[m.value for m in ExecMode]}, got {text!r}") from None


def _gamma(v):
    if v is not None and not 0.0 < v <= 1.0:
        raise _Usage("gamma must be in (0,1]")
    return v


def _outdir(path: str) -> str:
    os.makedirs(path, exist_ok=True)
    return path


def _write_json(path: str, doc) -> None:
    with open(path, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
        f.write("\n")


# ---------------------------------------------------------------- subcommands
def cmd_run(args) -> int:
    from .harness import DenoiseRunConfig, run_denoise
    mode = _mode(args.mode)
    ucfg, ex = _unet_cfg(args), _exec_cfg(args)
    gamma = _gamma(args.gamma)
    keys = None
    if args.key_steps:
        try:
            keys = sorted({int(v) for v in args.key_steps.split(",")})
        except ValueError:
            raise _Usage("key-steps must be a comma-separated list of step indices") from None
    if mode is ExecMode.NAIVE_CLIP and args.naive_chunk is None:
        raise _Usage("naive-chunk is required for --mode naiveclip")
    if args.target_count is not None and args.target_count < 1:
        raise _Usage("target-count must be >= 1")
    out = _outdir(args.out)
    sched = None
    if keys is not None:
        from .rehash import StepSchedule
        sched = StepSchedule(keys, ucfg.steps)
    graph, weights = _model_files(args)
    y, rep = run_denoise(DenoiseRunConfig(unet=ucfg, mode=mode, schedule=sched, gamma=gamma,
                                          target_keys=args.target_count, exec_cfg=ex,
                                          naive_chunk=args.naive_chunk, graph=graph, weights=weights))
    rep.save(os.path.join(out, "run_report.json"))
    if args.save_output:
        np.save(os.path.join(out, "output.npy"), y.data)
    print(json.dumps({"mode": rep.mode, "output_checksum": rep.output_checksum, "wall_ms": rep.wall_ms}))
    return 0


def cmd_compare(args) -> int:
    from .harness import DenoiseRunConfig, run_denoise
    modes = [_mode(m.strip()) for m in args.modes.split(",") if m.strip()]
    if not modes:
        raise _Usage("modes must list at least one mode")
    if ExecMode.NAIVE_CLIP in modes and args.naive_chunk is None:
        raise _Usage("naive-chunk is required when comparing naiveclip")
    ucfg, ex = _unet_cfg(args), _exec_cfg(args)
    graph, weights = _model_files(args)
    out = _outdir(args.out)
    rows, base = [], None
    for m in modes:
        y, rep = run_denoise(DenoiseRunConfig(unet=ucfg, mode=m, exec_cfg=ex, naive_chunk=args.naive_chunk,
                                              graph=graph, weights=weights))
        if base is None:
            base = y.data
        err = float(np.abs(y.data - base).max() / max(float(np.abs(base).max()), 1e-30))
        abs_err = float(np.abs(y.data - base).max())
        rows.append({"mode": m.value, "peak_bytes": rep.peak_bytes, "static_model_bytes": rep.static_model_bytes,
                     "ledger_peak_bytes": rep.ledger_peak_bytes, "wall_ms": rep.wall_ms, "max_rel_error": err,
                     "max_abs_error": abs_err, "diverged": abs_err > 1e-3,
                     "output_checksum": rep.output_checksum})
    _write_json(os.path.join(out, "compare.json"), {"baseline": modes[0].value, "rows": rows})
    print(json.dumps(rows))
    return 0


def cmd_similarity(args) -> int:
    from .harness import Denoiser, initial_latent
    from .unet import PROBE_LABEL
    if args.probe_label not in (None, PROBE_LABEL):
        raise _Usage(f"probe-label: the device path caches {PROBE_LABEL!r} (the rehash probe)")
    ucfg, ex = _unet_cfg(args), _exec_cfg(args)
    graph, weights = _model_files(args)
    if graph is not None:
        from .harness import DenoiseRunConfig, _model_inputs
        graph, weights = _model_inputs(DenoiseRunConfig(unet=ucfg, graph=graph, weights=weights))
    out = _outdir(args.out)
    den = Denoiser(ucfg, ex, graph=graph, weights=weights)
    _, S = den.calibrate(initial_latent(ucfg))
    with open(os.path.join(out, "similarity.csv"), "w") as f:
        f.write(S.export_csv())
    K = S.K
    adj = [float(S.values[i, i + 1]) for i in range(K - 1)]
    _write_json(os.path.join(out, "similarity.json"),
                {"probe_label": PROBE_LABEL, "K": K, "mean_adjacent": float(np.mean(adj)) if adj else 1.0,
                 "min_adjacent": float(np.min(adj)) if adj else 1.0, "mean": float(S.values.mean())})
    return 0


def cmd_search_steps(args) -> int:
    from .rehash import SimilarityMap, gamma_for_target, key_step_search
    gamma = _gamma(args.gamma)
    if (gamma is None) == (args.target_count is None):
        raise _Usage("give exactly one of --gamma / --target-count")
    try:
        with open(args.similarity) as f:
            S = SimilarityMap.parse_csv(f.read())
    except (OSError, ValueError, IndexError) as e:
        raise _Usage(f"similarity: {e}") from None
    if S.values.shape != (S.K, S.K):
        raise _Usage("similarity: not a square K x K map")
    if gamma is None:
        gamma = gamma_for_target(S, args.target_count)
    sched = key_step_search(S, gamma, S.K)
    out = _outdir(args.out)
    doc = sched.to_json_dict()
    doc["margin"] = sched.margin if sched.margin is None or np.isfinite(sched.margin) else None
    _write_json(os.path.join(out, "schedule.json"), doc)
    print(json.dumps(doc))
    return 0


def cmd_export(args) -> int:
    """Write the config's network as graph.json + weights.slfw (host only, no device work)."""
    from .unet import build_toy_unet
    ucfg = _unet_cfg(args)
    graph, weights = build_toy_unet(ucfg)
    out = _outdir(args.out)
    graph.save(os.path.join(out, "graph.json"))
    weights.save(os.path.join(out, "weights.slfw"))
    print(json.dumps({"nodes": len(graph.nodes), "weight_entries": len(weights.entries),
                      "params": int(weights.param_count())}))
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="python -m paper_2411_01171_b200", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    r = sub.add_parser("run", help="one denoising run -> run_report.json")
    _unet_flags(r)
    _model_flags(r)
    r.add_argument("--mode", default=ExecMode.SLICED_LOOP.value)
    r.add_argument("--gamma", type=float)
    r.add_argument("--target-count", type=int)
    r.add_argument("--key-steps", help="comma-separated key steps (explicit schedule)")
    r.add_argument("--naive-chunk", type=int)
    r.add_argument("--save-output", action="store_true", help="also write output.npy")
    r.set_defaults(fn=cmd_run)
    c = sub.add_parser("compare", help="run several modes, diff their outputs -> compare.json")
    _unet_flags(c)
    _model_flags(c)
    c.add_argument("--modes", default="reference,slicedloop,pipelined")
    c.add_argument("--naive-chunk", type=int)
    c.set_defaults(fn=cmd_compare)
    s = sub.add_parser("similarity", help="calibration run -> similarity.csv + similarity.json")
    _unet_flags(s)
    _model_flags(s)
    s.add_argument("--probe-label")
    s.set_defaults(fn=cmd_similarity)
    k = sub.add_parser("search-steps", help="Algorithm A1 on a similarity CSV -> schedule.json")
    k.add_argument("--similarity", required=True)
    k.add_argument("--gamma", type=float)
    k.add_argument("--target-count", type=int)
    k.add_argument("--out", required=True)
    k.set_defaults(fn=cmd_search_steps)
    e = sub.add_parser("export", help="write the config's network -> graph.json + weights.slfw")
    _unet_flags(e)
    e.set_defaults(fn=cmd_export)
    return p


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        return args.fn(args)
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except SliceflowError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
