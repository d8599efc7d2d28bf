"""CPU ORACLE — test infrastructure only (tests/, smoke(), bench.py cpu_baseline / --impl reference).

Host restatement of the synthetic workloads the device generator (csrc/ct_gen.cu)
writes, built as plain event objects so the CPU oracle can analyze the same trace
without touching the GPU.  C4 follows the reference's own generator:
``generate_training_trace`` (workload.py:166-195) with ``plan_buckets``
(workload.py:69-86) and the ``resnet_like_preset`` shape (workload.py:221-235:
broadcast_init, d h2d copies of 192 KiB per iteration, 25 MiB buckets, ring), with
the ResNet-50 tensor list in place of the ResNet-18 one.
"""

from __future__ import annotations

from types import SimpleNamespace


class _E(SimpleNamespace):
    pass


def _enum(v):
    return SimpleNamespace(value=v)


def resnet50_tensor_bytes() -> list[int]:
    p = []

    def conv(cin, cout, k):
        p.append(cout * cin * k * k)

    def bn(c):
        p.extend([c, c])

    conv(3, 64, 7)
    bn(64)
    cin = 64
    for blocks, w in zip((3, 4, 6, 3), (64, 128, 256, 512)):
        for b in range(blocks):
            cout = 4 * w
            conv(cin, w, 1); bn(w)
            conv(w, w, 3); bn(w)
            conv(w, cout, 1); bn(cout)
            if b == 0:
                conv(cin, cout, 1); bn(cout)
            cin = cout
    p.extend([2048 * 1000, 1000])
    return [4 * x for x in p]


def plan_buckets(sizes, cap):
    """Reverse greedy packing (workload.py:69-86)."""
    out, cur = [], 0
    for s in reversed(list(sizes)):
        if s > cap:
            if cur:
                out.append(cur)
                cur = 0
            out.append(s)
            continue
        if cur and cur + s > cap:
            out.append(cur)
            cur = 0
        cur += s
    if cur:
        out.append(cur)
    return out


def c4_events(n_records: int, d: int = 8, lo: int = 0):
    """Events [lo, n_records) of the C4 trace (whole calls; lo a multiple of d)."""
    tensors = resnet50_tensor_bytes()
    buckets = plan_buckets(tensors, 25 << 20)
    seq = [0] * d
    out = []
    pos = [0]  # records emitted so far, materialised only from ``lo``

    class _Sink(list):
        def __len__(self):
            return pos[0]

        def append(self, ev):
            if pos[0] >= lo:
                list.append(self, ev)
            pos[0] += 1

    out = _Sink()

    def coll(kind, count, root):
        for r in range(d):
            out.append(_E(seq=seq[r], ts_ns=seq[r], kind=_enum("collective"), comm="comm0", n_ranks=d,
                          rank=r, device=r, collective=_enum(kind), algorithm=_enum("ring"),
                          root=root, peer=None, count=count, dtype=_enum("float32"),
                          copy_kind=None, copy_src=None, copy_dst=None, bytes=None))
            seq[r] += 1

    def h2d(r, nbytes):
        out.append(_E(seq=seq[r], ts_ns=seq[r], kind=_enum("memcpy"), comm="comm0", n_ranks=d, rank=r,
                      device=r, collective=None, algorithm=None, root=None, peer=None, count=None,
                      dtype=None, copy_kind=_enum("h2d"),
                      copy_src=SimpleNamespace(kind=_enum("host"), index=0),
                      copy_dst=SimpleNamespace(kind=_enum("gpu"), index=r), bytes=nbytes))
        seq[r] += 1

    for s in tensors:
        if len(out) + d > n_records:
            return list(out)
        coll("broadcast", -(-s // 4), 0)
    while True:
        if len(out) + d > n_records:
            return list(out)
        for r in range(d):
            h2d(r, 192 << 10)
        for b in buckets:
            if len(out) + d > n_records:
                return list(out)
            coll("allreduce", -(-b // 4), None)
