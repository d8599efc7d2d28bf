"""Generate the golden fixtures by running the REAL reference in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (pure Python ``commtrace``) lives read-only under /root/reference;
it does not exist on the GPU box, so its outputs are frozen here as small JSON
fixtures that travel with the repo.  Everything written is derived from the
reference's public functions (plus ``matrix._typed_decompositions`` to derive
the frequency matrix: freq[src][dst] += 1 per accumulated
PairTransfer).

Fixtures (all gzip'd JSON):
  traces.json.gz      named traces (JSONL text) + expected analysis results
  decomp_grid.json.gz acceptance grid N in [1,16] x S in [0,257] (test_acceptance.py:82-119)
  random_insts.json.gz 10,000 seeded instances (test_acceptance.py:130-163)
  loader.json.gz      loader error cases (events.py:352-384)
  loader_fuzz.json.gz the seeded fuzz corpus of tests/loader_fuzz.py with the reference
                      reader's events or exception per text (str and bytes input)
  siblings.json.gz    split_by_primitive / summarize on caller-ordered instance lists
                      (comm-major, shuffled, reversed), infer_device_count, merge and
                      accumulate (matrix.py:157-301)

    python tests/golden/make_golden.py [fixture ...]   (default: all)
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from commtrace import errors as E  # noqa: E402
from commtrace.decompose import decompose_instance  # noqa: E402
from commtrace.events import (  # noqa: E402
    HOST, Algorithm, CollectiveKind, CopyKind, DataType, EventKind, TraceEvent,
    gpu, parse_trace, write_trace,
)
from commtrace.grouping import CollectiveInstance  # noqa: E402
from commtrace.grouping import group_collectives  # noqa: E402
from commtrace.matrix import (  # noqa: E402
    ALL_TYPES, CommMatrix, ModelConfig, _typed_decompositions, accumulate, analyze_events,
    infer_device_count, merge, split_by_primitive, summarize,
)
from commtrace.workload import (  # noqa: E402
    TrainingConfig, generate_gnmt_trace, generate_training_trace, resnet_like_preset,
)

OUT = os.path.dirname(os.path.abspath(__file__))


def _idx(m: CommMatrix, ep) -> int:
    if ep.kind.value == "host":
        return 0
    if ep.kind.value == "gpu":
        return ep.index + 1
    return m.d + 1


def freq_matrices(events, result, config):
    """A19: frequency matrices derived from the reference's own decompositions."""
    typed, _ = _typed_decompositions(result.instances, events, config)
    d = result.d

    def blank(m):
        return [[0] * m.size for _ in range(m.size)]

    comb = blank(result.combined)
    per = {k: blank(m) for k, m in result.per_primitive.items()}
    for key, _, dec in typed:
        for t in dec.transfers:
            i, j = _idx(result.combined, t.src), _idx(result.combined, t.dst)
            comb[i][j] += 1
            pm = result.per_primitive[key]
            per[key][_idx(pm, t.src)][_idx(pm, t.dst)] += 1
    del d
    return comb, per


def run_case(name, events, d=None, config=ModelConfig()):
    jsonl = write_trace(events).decode() if events is not None else ""
    case = {"name": name, "jsonl": jsonl, "d": d,
            "ring_order": list(config.ring_order) if config.ring_order else None,
            "tree_threshold": config.tree_threshold}
    try:
        res = analyze_events(events, d=d, config=config)
    except (E.TraceError, OverflowError) as exc:
        case["error"] = {"type": type(exc).__name__, "message": str(exc)}
        return case
    fc, fp = freq_matrices(events, res, config)
    where = {id(e): i for i, e in enumerate(events)}
    case["result"] = {
        "d": res.d,
        "combined": res.combined.rows(),
        "combined_agg": res.combined.with_aggregator,
        "combined_freq": fc,
        "per_primitive": [[k, m.rows(), m.with_aggregator, fp[k]] for k, m in res.per_primitive.items()],
        "stats": {t: [s.call_count, s.payload_bytes, s.wire_bytes] for t, s in res.stats.types.items()},
        "instances": res.stats.instances,
        "n_diagnostics": res.stats.diagnostics,
        "diagnostics": [[dg.reason, dg.comm, dg.ordinal, dg.detail,
                         [where[id(e)] for e in dg.events]] for dg in res.diagnostics],
        "instance_list": [[i.comm, i.ordinal, i.collective.value, i.algorithm.value, i.n_ranks,
                           i.count, i.dtype.value, i.root, list(i.per_rank_devices)]
                          for i in res.instances],
    }
    return case


# ------------------------------------------------------------------ traces

def coll(seq, rank, n, comm="c0", c=CollectiveKind.ALLREDUCE, a=Algorithm.RING, count=256,
         dt=DataType.FLOAT32, root=None, dev=None, ts=0):
    return TraceEvent(seq=seq, ts_ns=ts, kind=EventKind.COLLECTIVE, comm=comm, n_ranks=n,
                      rank=rank, device=rank if dev is None else dev, collective=c,
                      algorithm=a, count=count, dtype=dt, root=root)


def p2p(kind, seq, rank, peer, n, count=64, dt=DataType.FLOAT32, comm="c0", dev=None, ts=0):
    return TraceEvent(seq=seq, ts_ns=ts, kind=kind, comm=comm, n_ranks=n, rank=rank,
                      device=rank if dev is None else dev, peer=peer, count=count, dtype=dt)


def copy(kind, ck, src, dst, nbytes, seq=0, rank=0, n=1, comm="c0", dev=0, ts=0):
    return TraceEvent(seq=seq, ts_ns=ts, kind=kind, comm=comm, n_ranks=n, rank=rank, device=dev,
                      copy_kind=ck, copy_src=src, copy_dst=dst, bytes=nbytes)


def random_trace(rng: random.Random, mode: str):
    """Adversarial random traces: canonical blocks, rank-major files, shuffles,
    incomplete/incompatible/duplicate-device groups, p2p mismatches, copies."""
    events = []
    n_comms = rng.randint(1, 3)
    comms = []
    for c in range(n_comms):
        n = rng.randint(1, 8)
        devmap = list(range(n)) if rng.random() < 0.7 else [rng.randrange(10) for _ in range(n)]
        if rng.random() < 0.5 and n > 1:
            devmap = rng.sample(range(12), n)
        comms.append((f"comm{c}", n, devmap))
    seqs = {}

    def nxt(comm, rank):
        s = seqs.get((comm, rank), 0)
        seqs[(comm, rank)] = s + rng.choice([1, 1, 1, 2])
        return s

    blocks = []  # list of lists (one logical item each)
    for _ in range(rng.randint(1, 25)):
        comm, n, devmap = rng.choice(comms)
        r = rng.random()
        if r < 0.55:
            c = rng.choice(list(CollectiveKind))
            a = rng.choice(list(Algorithm)) if c is CollectiveKind.ALLREDUCE else rng.choice([Algorithm.RING, Algorithm.AUTO])
            mag = rng.choice([0, 1, 3, 7, 100, 1000, 1 << 16, 1 << 20, 1 << 27])
            count = rng.randint(0, mag)
            dt = rng.choice(list(DataType))
            root = rng.randrange(n) if c in (CollectiveKind.BROADCAST, CollectiveKind.REDUCE) else None
            item = []
            for rank in range(n):
                ev_count, ev_dt = count, dt
                if rng.random() < 0.03:
                    ev_count = count + 1  # incompatible arguments
                dev = devmap[rank]
                if rng.random() < 0.02:
                    dev = devmap[0]
                item.append(coll(nxt(comm, rank), rank, n, comm, c, a, ev_count, ev_dt, root, dev,
                                 ts=rng.randint(0, 1000)))
            if rng.random() < 0.05 and n > 1:
                item.pop(rng.randrange(len(item)))  # incomplete
            blocks.append(item)
        elif r < 0.75 and n > 1:
            src, dst = rng.sample(range(n), 2)
            count = rng.randint(0, 5000)
            dt = rng.choice(list(DataType))
            item = [p2p(EventKind.SEND, nxt(comm, src), src, dst, n, count, dt, comm, devmap[src])]
            rcount, rdt = count, dt
            if rng.random() < 0.08:
                rcount = count + 3
            if rng.random() < 0.9:
                item.append(p2p(EventKind.RECV, nxt(comm, dst), dst, src, n, rcount, rdt, comm, devmap[dst]))
            if rng.random() < 0.1:
                item = item[::-1]
            blocks.append(item)
        else:
            kind = rng.choice([EventKind.MEMCPY, EventKind.UNIFIED_MEMORY, EventKind.ZERO_COPY])
            ck = rng.choice(list(CopyKind))
            rank = rng.randrange(n)
            g1 = rng.randrange(10)
            g2 = (g1 + rng.randint(1, 9)) % 10
            src = HOST if ck is CopyKind.H2D else gpu(g1)
            dst = HOST if ck is CopyKind.D2H else gpu(g2)
            blocks.append([copy(kind, ck, src, dst, rng.randint(0, 1 << rng.choice([0, 10, 20, 40])),
                                nxt(comm, rank), rank, n, comm, devmap[rank])])
    if mode == "canonical":
        for b in blocks:
            events.extend(b)
    elif mode == "rankmajor":
        # each rank's capture file concatenated (multi-file analyze, cli.py:131-135)
        flat = [e for b in blocks for e in b]
        keyed = sorted(range(len(flat)), key=lambda i: (flat[i].device, i))
        events = [flat[i] for i in keyed]
    else:
        flat = [e for b in blocks for e in b]
        rng.shuffle(flat)
        events = flat
    return events


def build_traces():
    cases = []
    c1 = TrainingConfig(n_gpus=4, tensor_sizes_bytes=tuple(4096 * (i + 1) for i in range(10)),
                        iterations_per_epoch=310, bucket_cap_bytes=1 << 15, broadcast_init=True)
    cases.append(run_case("C1", generate_training_trace(c1)))
    cases.append(run_case("gnmt_d4_s42", generate_gnmt_trace(4, 0.001, 42)))
    cases.append(run_case("gnmt_d8_s0", generate_gnmt_trace(8, 0.001, 0)))
    small_resnet = resnet_like_preset(4)
    small_resnet = TrainingConfig(**{**small_resnet.__dict__, "iterations_per_epoch": 3})
    cases.append(run_case("resnet_d4_3it", generate_training_trace(small_resnet)))
    # tree / collnet / auto with custom ring and explicit d
    ev = []
    for k, (a, cnt) in enumerate([(Algorithm.TREE, 1), (Algorithm.TREE, 7), (Algorithm.COLLNET, 5),
                                  (Algorithm.AUTO, 10), (Algorithm.AUTO, 1 << 20), (Algorithm.RING, 13)]):
        for r in range(5):
            ev.append(coll(k, r, 5, "x", a=a, count=cnt, dt=DataType.INT8, dev=4 - r))
    cases.append(run_case("algos_n5", ev))
    cases.append(run_case("algos_n5_ring", ev, config=ModelConfig(ring_order=(0, 2, 4, 1, 3))))
    cases.append(run_case("algos_n5_thresh", ev, config=ModelConfig(tree_threshold=11)))
    cases.append(run_case("algos_n5_d7", ev, d=7))
    cases.append(run_case("algos_n5_d3", ev, d=3))  # EndpointOutOfRange
    cases.append(run_case("bad_ring", ev, config=ModelConfig(ring_order=(0, 1, 2, 2, 4))))
    cases.append(run_case("empty", []))
    # fatal grouping errors
    cases.append(run_case("dup_seq", [coll(3, 0, 1), coll(3, 0, 1)]))
    cases.append(run_case("nranks", [coll(0, 0, 2), coll(0, 1, 3)]))
    cases.append(run_case("nranks_then_dup", [coll(0, 0, 2), coll(0, 0, 2), coll(0, 1, 3)]))
    # overflow
    big = (1 << 62)
    cases.append(run_case("overflow", [copy(EventKind.MEMCPY, CopyKind.H2D, HOST, gpu(0), big, seq=k)
                                       for k in range(2)]))
    cases.append(run_case("overflow_wrap", [copy(EventKind.MEMCPY, CopyKind.H2D, HOST, gpu(0), big, seq=k)
                                            for k in range(5)]))
    cases.append(run_case("no_overflow", [copy(EventKind.MEMCPY, CopyKind.H2D, HOST, gpu(0), (1 << 63) - 1)]))
    cases.append(run_case("huge_payload_nowire", [coll(0, 0, 1, count=(1 << 64) - 1, dt=DataType.FLOAT64)]))
    rng = random.Random(1234)
    for i in range(240):
        mode = ("canonical", "rankmajor", "shuffled")[i % 3]
        events = random_trace(rng, mode)
        cfg = ModelConfig()
        if rng.random() < 0.2:
            cfg = ModelConfig(tree_threshold=rng.choice([1, 100, 5000]))
        if rng.random() < 0.2:
            ns = sorted({e.n_ranks for e in events if e.kind is EventKind.COLLECTIVE})
            if ns:
                n = rng.choice(ns)
                order = list(range(n))
                rng.shuffle(order)
                cfg = ModelConfig(ring_order=tuple(order), tree_threshold=cfg.tree_threshold)
        d = None
        if rng.random() < 0.15:
            d = infer_device_count(events) + rng.choice([-1, 0, 2])
            d = max(d, 0)
        cases.append(run_case(f"rand{i}_{mode}", events, d=d, config=cfg))
    return cases


def build_grid():
    """Acceptance grid (test_acceptance.py:82-119): by_pair per (model, n, s)."""
    out = {}

    def inst(c, a, n, s, root=None):
        return CollectiveInstance("c0", 0, c, a, n, s, DataType.INT8, root, tuple(range(n)))

    for n in range(1, 17):
        for s in range(0, 258):
            models = {
                "ar_ring": inst(CollectiveKind.ALLREDUCE, Algorithm.RING, n, s),
                "ar_tree": inst(CollectiveKind.ALLREDUCE, Algorithm.TREE, n, s),
                "ar_collnet": inst(CollectiveKind.ALLREDUCE, Algorithm.COLLNET, n, s),
                "allgather": inst(CollectiveKind.ALLGATHER, Algorithm.RING, n, s),
                "reducescatter": inst(CollectiveKind.REDUCESCATTER, Algorithm.RING, n, s),
                "broadcast": inst(CollectiveKind.BROADCAST, Algorithm.RING, n, s, s % n),
                "reduce": inst(CollectiveKind.REDUCE, Algorithm.RING, n, s, s % n),
            }
            for name, i in models.items():
                dec = decompose_instance(i)
                out[f"{name}/{n}/{s}"] = [[_ep(t.src), _ep(t.dst), t.bytes] for t in dec.transfers]
    return out


def _ep(ep):
    return -1 if ep.kind.value == "net" else ep.index


def build_random_instances():
    """10,000 seeded instances (test_acceptance.py:130-163) with ring orders."""
    rng = random.Random(20240917)
    rows = []
    for _ in range(10_000):
        n = rng.randint(1, 16)
        count = rng.randint(0, 100_000)
        dtype = rng.choice(list(DataType))
        c = rng.choice(list(CollectiveKind))
        a = rng.choice([Algorithm.RING, Algorithm.TREE, Algorithm.COLLNET]) if c is CollectiveKind.ALLREDUCE else Algorithm.RING
        root = rng.randrange(n) if c in (CollectiveKind.BROADCAST, CollectiveKind.REDUCE) else None
        order = list(range(n))
        rng.shuffle(order)
        inst = CollectiveInstance("c0", 0, c, a, n, count, dtype, root, tuple(range(n)))
        dec = decompose_instance(inst, ring_order=tuple(order))
        rows.append({"n": n, "count": count, "dtype": dtype.value, "coll": c.value, "algo": a.value,
                     "root": root, "order": order,
                     "transfers": [[_ep(t.src), _ep(t.dst), t.bytes] for t in dec.transfers]})
    return rows


def build_loader_cases():
    good = write_trace([coll(0, 0, 2)]).decode()
    texts = {
        "empty": "",
        "blank_lines": "\n\n" + good + "   \n",
        "malformed": good + "{oops\n",
        "not_object": good + "[1,2]\n",
        "missing_comm": good.replace('"comm":"c0",', ""),
        "bool_count": good.replace('"count":256', '"count":true'),
        "float_count": good.replace('"count":256', '"count":256.0'),
        "unknown_kind": good.replace('"kind":"collective"', '"kind":"bogus"'),
        "rank_range": good.replace('"rank":0', '"rank":5'),
        "extra_keys": good.replace('"seq":0', '"seq":0,"zzz":{"a":[1]}'),
        "cr_split": good.rstrip("\n") + "\r" + good,
        "unicode_sep": good.rstrip("\n") + " " + "{oops",
        "bad_endpoint": write_trace([copy(EventKind.MEMCPY, CopyKind.H2D, HOST, gpu(1), 5)]).decode()
        .replace('{"kind":"host","idx":0}', '{"kind":"host","idx":3}'),
        "d2h_flip": write_trace([copy(EventKind.MEMCPY, CopyKind.H2D, HOST, gpu(1), 5)]).decode()
        .replace('"ckind":"h2d"', '"ckind":"d2h"'),
        "root_on_allreduce": good.replace('"dtype":"float32"', '"dtype":"float32","root":1'),
        "bcast_no_root": good.replace('"coll":"allreduce"', '"coll":"broadcast"'),
        "tree_on_bcast": good.replace('"coll":"allreduce","algo":"ring"', '"coll":"broadcast","algo":"tree","root":0'),
        "neg_seq": good.replace('"seq":0', '"seq":-1'),
        "big_ints": good.replace('"count":256', '"count":123456789012345678'),
    }
    out = {}
    for name, text in texts.items():
        try:
            evs = parse_trace(text)
            out[name] = {"text": text, "n_events": len(evs),
                         "roundtrip": write_trace(evs).decode()}
        except E.TraceError as exc:
            out[name] = {"text": text, "error": {"type": type(exc).__name__, "message": str(exc),
                                                  "line_no": getattr(exc, "line_no", None)}}
    return out


def dump(name, obj):
    path = os.path.join(OUT, name)
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(obj, fh, separators=(",", ":"), sort_keys=False)
    print(name, os.path.getsize(path))


def build_loader_fuzz():
    """The reference reader on every text of the fuzz corpus (tests/loader_fuzz.py)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from tests.loader_fuzz import corpus, event_row

    def ref(src):
        try:
            return {"events": [event_row(e) for e in parse_trace(src)]}
        except (E.TraceError, UnicodeDecodeError) as exc:
            return {"error": [type(exc).__name__, str(exc)]}

    out = []
    for group, text in corpus():
        r_str = ref(text)
        r_bytes = ref(text.encode("utf-8", "surrogatepass"))
        row = {"g": group, "text": text, "str": r_str}
        if r_bytes != r_str:
            row["bytes"] = r_bytes
        out.append(row)
    return out


def _inst_row(i):
    return [i.comm, i.ordinal, i.collective.value, i.algorithm.value, i.n_ranks, i.count, i.dtype.value,
            i.root, list(i.per_rank_devices)]


def _mrows(m):
    return [m.rows(), m.with_aggregator]


def _err(exc):
    return {"error": [type(exc).__name__, str(exc)]}


def build_siblings():
    """split_by_primitive / summarize (matrix.py:261-301) on instance lists in caller
    order -- comm-major as grouped, shuffled, reversed -- plus infer_device_count
    (matrix.py:250-258), merge (matrix.py:164-178) and accumulate (matrix.py:157-161)."""
    cases = build_traces()
    rng = random.Random(4321)
    out = []
    for case in cases:
        if "result" not in case:
            continue
        events = parse_trace(case["jsonl"])
        if not events:
            continue
        cfg = ModelConfig(ring_order=tuple(case["ring_order"]) if case["ring_order"] else None,
                          tree_threshold=case["tree_threshold"])
        instances, gdiags = group_collectives(events)
        shuffled = list(instances)
        rng.shuffle(shuffled)
        orders = {"grouped": instances, "shuffled": shuffled, "reversed": instances[::-1]}
        row = {"name": case["name"], "infer_d": infer_device_count(events), "orders": {}}
        for oname, lst in orders.items():
            rec = {"instances": [_inst_row(i) for i in lst]}
            for dname, d in (("auto", None), ("given", case["d"])):
                if dname == "given" and d is None:
                    continue
                try:
                    sp = split_by_primitive(lst, events, d=d, config=cfg)
                    rec["split_" + dname] = [[k, *_mrows(m)] for k, m in sp.items()]
                except (E.TraceError, OverflowError) as exc:
                    rec["split_" + dname] = _err(exc)
            try:
                sm = summarize(lst, events, config=cfg, diagnostics=gdiags)
                rec["summary"] = {"types": {t: [v.call_count, v.payload_bytes, v.wire_bytes]
                                            for t, v in sm.types.items()},
                                  "instances": sm.instances, "diagnostics": sm.diagnostics}
            except (E.TraceError, OverflowError) as exc:
                rec["summary"] = _err(exc)
            rec["summary_nodiag"] = summarize(lst, events, config=cfg).diagnostics
            row["orders"][oname] = rec
            if len(lst) < 2 and oname != "grouped":
                break
        # accumulate: every typed decomposition into one matrix (and into a too-small one)
        typed, _ = _typed_decompositions(instances, events, cfg)
        decs = [[[_ep_full(t.src), _ep_full(t.dst), t.bytes] for t in dec.transfers] for _, _, dec in typed]
        row["decs"] = decs
        for dname, d in (("infer", row["infer_d"]), ("small", max(row["infer_d"] - 1, 0))):
            m = CommMatrix(d)
            try:
                for _, _, dec in typed:
                    accumulate(m, dec)
                row["acc_" + dname] = _mrows(m)
            except (E.TraceError, OverflowError) as exc:
                row["acc_" + dname] = _err(exc)
        # merge: combined + each per-primitive matrix, in both orders, and a d mismatch
        res = analyze_events(events, d=case["d"], config=cfg)
        merges = []
        mats = [res.combined] + list(res.per_primitive.values())
        for a in mats[:3]:
            for b in mats[:3]:
                try:
                    merges.append([_mrows(a), _mrows(b), _mrows(merge(a, b))])
                except (E.TraceError, OverflowError) as exc:
                    merges.append([_mrows(a), _mrows(b), _err(exc)])
        other = CommMatrix(res.d + 1)
        try:
            merge(res.combined, other)
        except E.TraceError as exc:
            merges.append([_mrows(res.combined), [other.rows(), False], _err(exc)])
        row["merges"] = merges
        out.append(row)
    # merge overflow (matrix.py:174-175)
    a = CommMatrix(1)
    a._cells[0][1] = (1 << 62)
    b = CommMatrix(1)
    b._cells[0][1] = (1 << 62) - 1
    b.widen()
    merges = [[_mrows(a), _mrows(b), _mrows(merge(a, b))]]
    try:
        merge(a, a)
    except OverflowError as exc:
        merges.append([_mrows(a), _mrows(a), _err(exc)])
    out.append({"name": "merge_overflow", "merges": merges})
    return out


def _ep_full(ep):
    return [ep.kind.value, ep.index]


FIXTURES = {
    "traces.json.gz": build_traces,
    "decomp_grid.json.gz": build_grid,
    "random_insts.json.gz": build_random_instances,
    "loader.json.gz": build_loader_cases,
    "loader_fuzz.json.gz": build_loader_fuzz,
    "siblings.json.gz": build_siblings,
}


if __name__ == "__main__":
    for name in sys.argv[1:] or list(FIXTURES):
        dump(name, FIXTURES[name]())
    _ = ALL_TYPES
