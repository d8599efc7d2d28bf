"""Probe mismatched-pair detection at several window positions."""
import sys
sys.path.insert(0, ".")
from paper_2110_10401_b200 import EventKind, DataType, TraceEvent, HOST, gpu, CopyKind
from paper_2110_10401_b200 import matrix
from paper_2110_10401_b200.packed import pack_events


def p2p(kind, seq, rank, peer, count, dt=DataType.INT8):
    return TraceEvent(seq=seq, ts_ns=0, kind=kind, comm="c", n_ranks=4, rank=rank, device=rank, peer=peer,
                      count=count, dtype=dt)


def cp(seq):
    return TraceEvent(seq=seq, ts_ns=0, kind=EventKind.MEMCPY, comm="c", n_ranks=4, rank=0, device=0,
                      copy_kind=CopyKind.H2D, copy_src=HOST, copy_dst=gpu(0), bytes=5)


for pre in (0, 1, 5, 30, 31):
    ev = [cp(i) for i in range(pre)] + [p2p(EventKind.SEND, 100, 0, 1, 10), p2p(EventKind.RECV, 100, 1, 0, 20)]
    for f in (1, 2):
        r = matrix.analyze_packed(pack_events(ev), force_path=f)
        print("pre", pre, "force", f, "path", r.path, "sendrecv calls", r.stats.types["sendrecv"].call_count,
              "diags", r.stats.diagnostics)
