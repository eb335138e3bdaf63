"""Byte-ledger definition and closed forms (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

The paper approximates communication volume as "total data received per device
per iteration" and states that TawPipe "transfers a single weight shard and its
corresponding gradients per step, totaling 24H²" (§3.5).
§8(c) R14 and Appendix A turn that into integer per-device counters of LOGICAL
elements (algorithm-independent):

  all-gather of a G-striped vector  : each participant receives (G−1)s, sends (G−1)s
  reduce-scatter of a G·s vector    : each participant receives (G−1)s, sends (G−1)s
  P2P of x                          : receiver x, sender x

Counter order (shared by this module, include/tawpipe.h and DESIGN.md):
  index = ((kind·2 + cls)·2 + dir)·3 + unit
  kind ∈ {0: weight, 1: grad}, cls ∈ {0: intra-group, 1: inter-group},
  dir ∈ {0: received, 1: sent}, unit ∈ {0: decoder blocks, 1: E, 2: F}.
"""
from __future__ import annotations

N_COUNTERS = 24
KINDS = ("w", "g")
CLASSES = ("intra", "inter")
DIRS = ("recv", "sent")
UNITS = ("block", "E", "F")


def index(kind: str, cls: str, dir_: str, unit: str) -> int:
    return ((KINDS.index(kind) * 2 + CLASSES.index(cls)) * 2 + DIRS.index(dir_)) * 3 + UNITS.index(unit)


def name(i: int) -> str:
    u = i % 3
    d = (i // 3) % 2
    c = (i // 6) % 2
    k = i // 12
    return f"{KINDS[k]}_{CLASSES[c]}_{DIRS[d]}_{UNITS[u]}"


def closed_form(L: int, P: int, G: int, k: int, s: int, e: int, f: int, r: int = 1) -> list:
    """SURVEY.md Appendix A, per device (k, j) per iteration, in elements.

    L layers, P devices, G = devices per group, D = P/G groups, k = group index
    of the device, s / e / f = stripe lengths of a decoder layer / E / F,
    r = 1 when layer L−1's forward buffer is reused for its backward (R12).
    """
    D = P // G
    assert P % G == 0 and L % D == 0
    Lr = L * (D - 1) // D
    out = [0] * N_COUNTERS

    def put(kind, cls, dir_, unit, val):
        out[index(kind, cls, dir_, unit)] = int(val)

    # decoder blocks
    put("w", "intra", "recv", "block", (2 * L - r) * (G - 1) * s)
    put("w", "intra", "sent", "block", (2 * L - r) * (G - 1) * s)
    put("w", "inter", "recv", "block", (2 * Lr - r * (1 if k != D - 1 else 0)) * s)
    put("w", "inter", "sent", "block", (2 * (L // D) * (D - 1) - r * (D - 1) * (1 if k == D - 1 else 0)) * s)
    put("g", "intra", "recv", "block", L * (G - 1) * s)
    put("g", "intra", "sent", "block", L * (G - 1) * s)
    put("g", "inter", "sent", "block", Lr * s)
    put("g", "inter", "recv", "block", (L // D) * (D - 1) * s)
    # pseudo-layers E (owner group 0) and F (owner group D−1): one gather, one reduction each
    for unit, n, owner in (("E", e, 0), ("F", f, D - 1)):
        put("w", "intra", "recv", unit, (G - 1) * n)
        put("w", "intra", "sent", unit, (G - 1) * n)
        put("w", "inter", "recv", unit, n if k != owner else 0)
        put("w", "inter", "sent", unit, (D - 1) * n if k == owner else 0)
        put("g", "intra", "recv", unit, (G - 1) * n)
        put("g", "intra", "sent", unit, (G - 1) * n)
        put("g", "inter", "sent", unit, n if k != owner else 0)
        put("g", "inter", "recv", unit, (D - 1) * n if k == owner else 0)
    return out


def block_received(ledger: list) -> int:
    """Total decoder-block elements received (weights + grads, intra + inter)."""
    return sum(ledger[index(kd, c, "recv", "block")] for kd in KINDS for c in CLASSES)


def ring_ledger(L: int, P: int, d: int, s: int, e: int, f: int, r: int = 1) -> list:
    """WeiPipe-style ring schedule, written from its definition:
    whole units, unit u owned by device o(u) (layer l: l mod P; E: 0; F: P−1); a weight gather moves u
    o → o+1 → … → o−1 (each device except o receives it once, each device except o−1 forwards it once); a
    gradient reduction moves the running partial o+1 → … → o (each device except o+1 receives one partial,
    each device except o sends one).  Same step sequence as the GWPS schedule (r = 1 reuses layer L−1)."""
    out = [0] * N_COUNTERS
    if P == 1:
        return out
    units = [("block", l % P, s) for l in range(L)]
    E, F = ("E", 0, e), ("F", P - 1, f)

    def gather(u):
        cls, o, n = u
        if d != o:
            out[index("w", "inter", "recv", cls)] += n
        if (d + 1) % P != o:
            out[index("w", "inter", "sent", cls)] += n

    def reduce(u):
        cls, o, n = u
        if d != (o + 1) % P:
            out[index("g", "inter", "recv", cls)] += n
        if d != o:
            out[index("g", "inter", "sent", cls)] += n

    gather(E)
    for u in units:
        gather(u)
    gather(F)
    reduce(F)
    for l in range(L - 1, -1, -1):
        if not (r == 1 and l == L - 1):
            gather(units[l])
        reduce(units[l])
    reduce(E)
    return out


def literal_ledger(L: int, P: int, D: int, d: int, x_block: int, x_e: int, x_f: int, r: int = 1) -> list:
    """Paper-literal collective mode, by enumerating its transfers for device d.

    Ownership (oracle/routes.py): layer l is shard l mod P, held whole by owner_table[l mod P]; the
    holder / staging / exit device of a unit in group k is its rail counterpart (k, i) (R7); E lives on device 0
    (i = 0), F on device P − 1 (i = G − 1).  A gather is the owner's P2P to (k, i) of every other group, then a
    broadcast from (k, i) to its group ("broadcasts weight shard W_0 within group g_0 ... sends W_0 to
    P_{P/D}"); a reduction is a reduce to (k, i) in every group, then (k, i)'s P2P to the owner (PAPER.md:127
    "reduced to device P_{P/D−1}, and then transferred to P_{P−1}").  Every delivered copy of x is one transfer:
    the receiver counts x received, the sender x sent (so a broadcast root sends (G−1)·x, reading R23).  Same step
    sequence as the striped schedule; x_* are the whole (padded) unit lengths."""
    from .routes import owner_table, rail_counterpart
    G = P // D
    own = owner_table(P, D)
    out = [0] * N_COUNTERS

    def xfer(kind, src, dst, cls_unit, n):
        cls = "intra" if src // G == dst // G else "inter"
        if dst == d:
            out[index(kind, cls, "recv", cls_unit)] += n
        if src == d:
            out[index(kind, cls, "sent", cls_unit)] += n

    def where(u):
        cls_unit, l = u
        if cls_unit == "block":
            o = own[l % P]
            hold = [rail_counterpart(l, kk, P, D) for kk in range(D)]
            return o, hold, x_block
        if cls_unit == "E":
            return 0, [kk * G for kk in range(D)], x_e
        return P - 1, [kk * G + G - 1 for kk in range(D)], x_f

    def gather(u):
        o, hold, n = where(u)
        for h in hold:
            if h != o:
                xfer("w", o, h, u[0], n)
        for h in hold:
            for m in range((h // G) * G, (h // G) * G + G):
                if m != h:
                    xfer("w", h, m, u[0], n)

    def reduce(u):
        o, hold, n = where(u)
        for h in hold:
            for m in range((h // G) * G, (h // G) * G + G):
                if m != h:
                    xfer("g", m, h, u[0], n)
        for h in hold:
            if h != o:
                xfer("g", h, o, u[0], n)

    E, F = ("E", None), ("F", None)
    gather(E)
    for l in range(L):
        gather(("block", l))
    gather(F)
    reduce(F)
    for l in range(L - 1, -1, -1):
        if not (r == 1 and l == L - 1):
            gather(("block", l))
        reduce(("block", l))
    reduce(E)
    return out
