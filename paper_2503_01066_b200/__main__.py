"""`python -m paper_2503_01066_b200 <profile|run|compare|plotdata> ...` -- the
reference driver's command line (tools/colosim.cpp:264-355: same subcommands,
options, outputs and exit codes 0 / 2 validation / 3 invariant breach) over
the GPU engine."""
from __future__ import annotations

import argparse
import os
import sys

EXIT_VALIDATION, EXIT_BREACH = 2, 3


def _profile(a) -> int:
    """tools/colosim.cpp:75-93."""
    from . import colosim as cs
    from .experiment import KvFile, _gpu_from_kv, _model_from_kv, _resolve, _out_file

    mk = KvFile.parse_file(_resolve(a.model))
    m = _model_from_kv(mk)
    mk.reject_unknown()
    gk = KvFile.parse_file(_resolve(a.gpu))
    g = _gpu_from_kv(gk)
    gk.reject_unknown()
    ctx = cs.Context(0)
    os.makedirs(a.out, exist_ok=True)
    steps = cs.GridSteps(a.cached_step, a.incoming_step, a.batch_step)
    bounds = cs.GridBounds(a.max_cached, a.max_incoming, a.max_batch)
    for mode in (cs.TrainingMode.CPT, cs.TrainingMode.CPA):
        tag = "cpt" if mode == cs.TrainingMode.CPT else "cpa"
        ms = cs.MapSet.build(ctx, m, g, steps, bounds, mode, assumed_output_tokens=a.output_tokens)
        cs.save_mapset(ms, _out_file(a.out, f"offload_{tag}.map", a.force), _out_file(a.out, f"hedge_{tag}.map", a.force))
        off, hed = ms.cells()
        print(f"wrote offload_{tag}.map ({len(off)} cells) and hedge_{tag}.map ({len(hed)} cells)")
    return 0


def _run(a) -> int:
    from . import colosim as cs
    from . import experiment as ex

    r = ex.cmd_run(cs.Context(0), a.config, a.out, a.trace or "", a.offload_map or "", a.hedge_map or "",
                   a.seed if a.seed is not None else -1, a.mode or "", a.emit_events, a.force)
    line = f"{r['mode_tag']}: {r['generated_tokens']} tokens served, {r['trained_tokens']} trained"
    if r["training_throughput"] is not None:
        line += ", %.1f tok/s training" % r["training_throughput"]
    if r["tpt_mean"] is not None:
        line += ", mean TPT %.4f s" % r["tpt_mean"]
    if r["oom_flag"]:
        line += ", training OOM"
    print(line)
    return 0


def _compare(a) -> int:
    from . import colosim as cs
    from . import experiment as ex

    ex.cmd_compare(cs.Context(0), a.config, a.out, a.force)
    print(f"comparison datasets written to {a.out}")
    return 0


def _plotdata(a) -> int:
    from . import experiment as ex

    ex.cmd_plotdata(a.report, a.out, a.force)
    print(f"plot data written to {a.out}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="colosim-b200",
                                 description="colosim on B200: co-located LLM serving and continual training")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("profile", help="build offloading and hedging maps from profiles")
    p.add_argument("--model", required=True)
    p.add_argument("--gpu", required=True)
    p.add_argument("--cached-step", type=int, default=500)
    p.add_argument("--incoming-step", type=int, default=500)
    p.add_argument("--batch-step", type=int, default=5)
    p.add_argument("--max-cached", type=int, default=8000)
    p.add_argument("--max-incoming", type=int, default=8000)
    p.add_argument("--max-batch", type=int, default=50)
    p.add_argument("--output-tokens", type=int, default=128)
    p.add_argument("--out", default="out")
    p.add_argument("--force", action="store_true")
    r = sub.add_parser("run", help="run one simulation and write its report")
    r.add_argument("--config", required=True)
    r.add_argument("--trace")
    r.add_argument("--offload-map")
    r.add_argument("--hedge-map")
    r.add_argument("--seed", type=int)
    r.add_argument("--mode")
    r.add_argument("--out", default="out")
    r.add_argument("--emit-events", action="store_true")
    r.add_argument("--force", action="store_true")
    c = sub.add_parser("compare", help="paired sweeps and figure datasets")
    c.add_argument("--config", required=True)
    c.add_argument("--out", default="out")
    c.add_argument("--force", action="store_true")
    d = sub.add_parser("plotdata", help="derive plot files from a report")
    d.add_argument("--report", required=True)
    d.add_argument("--out", default="out")
    d.add_argument("--force", action="store_true")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_VALIDATION if e.code else 0
    from ._lib import ColoBreachError

    try:
        return {"profile": _profile, "run": _run, "compare": _compare, "plotdata": _plotdata}[a.cmd](a)
    except ColoBreachError as e:
        print(f"invariant breach: {e}", file=sys.stderr)
        return EXIT_BREACH
    except Exception as e:  # the reference maps every other exception to exit code 2
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION


if __name__ == "__main__":
    sys.exit(main())
