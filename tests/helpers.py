"""Shared helpers: convert results into the golden-fixture shape."""

from paper_2110_10401_b200 import errors as E
from paper_2110_10401_b200.matrix import ModelConfig


def result_dict(res, events, with_lists=True):
    where = {id(e): i for i, e in enumerate(events)}
    out = {
        "d": res.d,
        "combined": res.combined.rows(),
        "combined_agg": res.combined.with_aggregator,
        "combined_freq": res.combined_frequency.rows(),
        "per_primitive": [[k, m.rows(), m.with_aggregator, res.per_primitive_frequency[k].rows()]
                          for k, m in res.per_primitive.items()],
        "stats": {t: [s.call_count, s.payload_bytes, s.wire_bytes] for t, s in res.stats.types.items()},
        "instances": res.stats.instances,
        "n_diagnostics": res.stats.diagnostics,
    }
    if with_lists:
        out["diagnostics"] = [[dg.reason, dg.comm, dg.ordinal, dg.detail, [where[id(e)] for e in dg.events]]
                              for dg in res.diagnostics]
        out["instance_list"] = [[i.comm, i.ordinal, i.collective.value, i.algorithm.value, i.n_ranks,
                                 i.count, i.dtype.value, i.root, list(i.per_rank_devices)]
                                for i in res.instances]
    return out


def run_case(case, analyze, **kw):
    """Analyze a golden case with ``analyze(events, d, config, **kw)``; fixture-shaped dict."""
    from paper_2110_10401_b200.events import parse_trace

    events = parse_trace(case["jsonl"])
    cfg = ModelConfig(ring_order=tuple(case["ring_order"]) if case["ring_order"] else None,
                      tree_threshold=case["tree_threshold"])
    try:
        res = analyze(events, case["d"], cfg, **kw)
    except (E.TraceError, OverflowError) as exc:
        return {"error": {"type": type(exc).__name__, "message": str(exc)}}, events
    return {"result": result_dict(res, events)}, events
