"""Simulated GWPS / DBS / CCO schedule over P devices (oracle, float64).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Follows SURVEY.md §8(a) rows a1-a11 in order, which restate PAPER.md:123-127
(§3.3) and PAPER.md:140-142 (§3.4) under the striped-ownership reading R6:

  * layer l belongs to group o(l) = l mod D; its padded flat vector is split into
    G stripes, stripe j on device (o(l), j).  E belongs to group 0, F to group D−1.
  * device d = (k, j) trains on micro-batches [d·m, (d+1)·m), m = N/P (R4).
  * gather(u): if o(u) ≠ k, rail P2P of stripe j from (o(u), j); then an
    intra-group all-gather of the G stripes ("intra-group
    communication … weight broadcasting"; "inter-group … P2P transfers").
  * forward over l = 0..L−1, head F (forward + backward back to back), backward
    over l = L−1..0 re-gathering every layer except L−1 (r = 1, R12), then E.
  * reduce(u): intra-group reduce-scatter in member order, then, if o(u) ≠ k,
    rail P2P of the group-partial stripe to (o(u), j); the owner adds the D group
    contributions in ascending group index (R16) and applies AdamW
    to its stripe "locally using colocated optimizer states".

A simulated device computes only with what it has gathered into its own buffer;
every byte between devices goes through ``Fabric`` which counts the byte ledger
(oracle/ledger.py).  The six validator checks of SPEC.md:440-445 are asserted
inline; ``mutate`` injects one fault at a time so that tests can show each check
catches exactly its fault.

The stagger of groups (R11) and CCO (prefetching l+1 during l) change only
*when* messages move; this sequential emulation moves them in the same order,
so results and ledger are those of the overlapped schedule.
"""
from __future__ import annotations

from collections import defaultdict, deque

import numpy as np

from . import ledger as L_
from . import layout
from .model import (ModelConfig, adamw_update, head_fwd_bwd, layer_bwd, layer_fwd, phi,
                    rope_tables)


class ValidationError(AssertionError):
    def __init__(self, check: str, detail: str):
        super().__init__(f"[{check}] {detail}")
        self.check = check


CHECKS = ("weight-presence", "gradient-exactly-once", "update-ordering",
          "activation-consume-once", "buffer-bounds", "matching")


class Fabric:
    """Point-to-point mailboxes with a per-device logical-element ledger."""

    def __init__(self, P: int):
        self.P = P
        self.box = defaultdict(deque)            # (src, dst, tag) -> payloads
        self.ledger = [[0] * L_.N_COUNTERS for _ in range(P)]
        self.log = []                            # (src, dst, tag, elements, kind, cls)

    def send(self, src, dst, tag, payload, kind, cls, unit):
        self.box[(src, dst, tag)].append(np.array(payload, copy=True))
        n = int(np.asarray(payload).size)
        self.log.append((src, dst, tag, n, kind, cls))
        self.ledger[src][L_.index(kind, cls, "sent", unit)] += n
        self.ledger[dst][L_.index(kind, cls, "recv", unit)] += n

    def recv(self, src, dst, tag):
        q = self.box.get((src, dst, tag))
        if not q:
            raise ValidationError("matching", f"device {dst} expected a message {tag} from {src}")
        return q.popleft()

    def assert_drained(self):
        left = {k: len(v) for k, v in self.box.items() if v}
        if left:
            raise ValidationError("matching", f"unreceived messages: {left}")


class Unit:
    """A DBS unit: decoder layer l, or pseudo-layer 'E' / 'F'."""

    def __init__(self, uid, n, owner_group, G, unit_class, no_decay):
        self.uid, self.n, self.owner, self.cls = uid, n, owner_group, unit_class
        self.n_pad = layout.padded(n, G)
        self.s = self.n_pad // G
        nd = np.zeros(self.n_pad, bool)
        nd[:n] = no_decay
        self.no_decay = nd


class Device:
    def __init__(self, d, G):
        self.d, self.k, self.j = d, d // G, d % G
        self.master, self.m, self.v = {}, {}, {}   # uid -> stripe arrays (float64)
        self.buffers = {}                          # uid -> (version, full padded vector)
        self.peak_buffers = 0


class GWPSSimulation:
    """P simulated devices running the striped GWPS/DBS schedule on the oracle model."""

    def __init__(self, cfg: ModelConfig, P: int, G: int, params: dict, r: int = 1,
                 mutate: str | None = None):
        if P % G:
            raise ValueError("P mod G != 0")
        self.cfg, self.P, self.G, self.D = cfg, P, G, P // G
        if cfg.n_layers % self.D:
            raise ValueError("L mod D != 0")
        self.r, self.mutate = r, mutate
        H, V, Lc = cfg.hidden, cfg.vocab, cfg.n_layers
        self.units = {}
        for l in range(Lc):
            self.units[l] = Unit(l, phi(cfg), l % self.D, G, "block", layout.no_decay_mask_layer(cfg))
        self.units["E"] = Unit("E", V * H, 0, G, "E", np.zeros(V * H, bool))
        self.units["F"] = Unit("F", H + V * H, self.D - 1, G, "F", layout.no_decay_mask_F(cfg))
        self.devices = [Device(d, G) for d in range(P)]
        full = self._unit_vectors(params)
        for dev in self.devices:
            for uid, u in self.units.items():
                if u.owner == dev.k:
                    st = full[uid][dev.j * u.s:(dev.j + 1) * u.s].astype(np.float64)
                    dev.master[uid] = st.copy()
                    dev.m[uid] = np.zeros_like(st)
                    dev.v[uid] = np.zeros_like(st)
        self.t = 0
        self.cos, self.sin = rope_tables(cfg.seq, cfg.head_dim, cfg.rope_theta)

    # -- helpers -------------------------------------------------------------
    def _unit_vectors(self, params):
        out = {}
        for uid, u in self.units.items():
            if uid == "E":
                vec = np.asarray(params["embed"], np.float64).reshape(-1)
            elif uid == "F":
                vec = layout.flatten_F(params["final_norm"], params["head"]).astype(np.float64)
            else:
                vec = layout.flatten_layer(params["layers"][uid], self.cfg).astype(np.float64)
            pad = np.zeros(u.n_pad)
            pad[:u.n] = vec
            out[uid] = pad
        return out

    def dev(self, k, j):
        return self.devices[k * self.G + j]

    def gather(self, uid, version):
        """a3: rail P2P of stripe j from the owner group (if remote), then intra-group all-gather."""
        u, G = self.units[uid], self.G
        tag = ("W", uid, version)
        # inter-group: owner (o, j) sends its stripe to (k, j) for every k != o
        for j in range(G):
            src = self.dev(u.owner, j)
            for k in range(self.D):
                if k != u.owner:
                    self.fabric.send(src.d, self.dev(k, j).d, tag, src.master[uid],
                                     "w", "inter", u.cls)
        stripes = {}
        for dev in self.devices:
            if dev.k == u.owner:
                stripes[dev.d] = dev.master[uid]
            else:
                stripes[dev.d] = self.fabric.recv(self.dev(u.owner, dev.j).d, dev.d, tag)
        # intra-group all-gather: every member sends its stripe to the G−1 others
        for dev in self.devices:
            for jj in range(G):
                if jj != dev.j:
                    self.fabric.send(dev.d, self.dev(dev.k, jj).d, tag + ("ag",), stripes[dev.d],
                                     "w", "intra", u.cls)
        for dev in self.devices:
            full = np.empty(u.n_pad)
            for jj in range(G):
                src = self.dev(dev.k, jj)
                piece = stripes[dev.d] if jj == dev.j else self.fabric.recv(src.d, dev.d, tag + ("ag",))
                full[jj * u.s:(jj + 1) * u.s] = piece
            ver = version - 1 if (self.mutate == "stale_version" and uid == 0) else version
            dev.buffers[uid] = (ver, full)
            nb = len(dev.buffers)
            if self.mutate == "extra_buffer":
                nb += 2
            dev.peak_buffers = max(dev.peak_buffers, nb)
            if nb > 2:
                raise ValidationError("buffer-bounds", f"device {dev.d} holds {nb} gathered units")

    def weights(self, dev, uid, version):
        """Check 1 (weight-presence / version) and return the gathered vector."""
        if uid not in dev.buffers:
            raise ValidationError("weight-presence", f"device {dev.d} computes unit {uid} without its weights")
        ver, full = dev.buffers[uid]
        if ver != version:
            raise ValidationError("weight-presence", f"device {dev.d} unit {uid} version {ver} != {version}")
        return full

    def release(self, uid):
        for dev in self.devices:
            dev.buffers.pop(uid, None)

    def reduce(self, uid, local_grads):
        """a8 + a9: intra-group reduce-scatter, rail P2P to the owner, ascending-k sum, AdamW."""
        u, G = self.units[uid], self.G
        tag = ("G", uid, self.t)
        for dev in self.devices:                    # reduce-scatter: send slice jj to member jj
            for jj in range(G):
                if jj != dev.j:
                    self.fabric.send(dev.d, self.dev(dev.k, jj).d, tag,
                                     local_grads[dev.d][jj * u.s:(jj + 1) * u.s], "g", "intra", u.cls)
        partial = {}
        for dev in self.devices:
            acc = np.zeros(u.s)
            for jj in range(G):                     # member order (R16)
                src = self.dev(dev.k, jj)
                piece = local_grads[dev.d][dev.j * u.s:(dev.j + 1) * u.s] if jj == dev.j \
                    else self.fabric.recv(src.d, dev.d, tag)
                acc = acc + piece
            partial[dev.d] = acc
        for dev in self.devices:                    # rail P2P of the group partial to the owner
            if dev.k != u.owner:
                if self.mutate == "drop_grad_msg" and uid == 0 and dev.k == (u.owner + 1) % self.D:
                    continue
                self.fabric.send(dev.d, self.dev(u.owner, dev.j).d, tag + ("p2p",), partial[dev.d],
                                 "g", "inter", u.cls)
        for j in range(G):
            own = self.dev(u.owner, j)
            contribs = []
            for k in range(self.D):                 # ascending group index (R16)
                if k == u.owner:
                    contribs.append(partial[own.d])
                else:
                    q = self.fabric.box.get((self.dev(k, j).d, own.d, tag + ("p2p",)))
                    if q:
                        contribs.append(self.fabric.recv(self.dev(k, j).d, own.d, tag + ("p2p",)))
            if len(contribs) != self.D:
                raise ValidationError("gradient-exactly-once",
                                      f"unit {uid} iteration {self.t}: owner {own.d} got {len(contribs)} of {self.D}")
            g = np.zeros(u.s)
            for c in contribs:
                g = g + c
            self.pending_updates.append((own, uid, g))

    def apply_updates(self):
        for own, uid, g in self.pending_updates:
            u = self.units[uid]
            if self.bwd_done[uid] != self.P:
                raise ValidationError("update-ordering", f"unit {uid} updated before all backward computes")
            nd = u.no_decay[own.j * u.s:(own.j + 1) * u.s]
            th, m, v = own.master[uid], own.m[uid], own.v[uid]
            th_d, m_d, v_d = adamw_update(th, g, m, v, self.t, self.cfg, decay=True)
            th_n, m_n, v_n = adamw_update(th, g, m, v, self.t, self.cfg, decay=False)
            own.master[uid] = np.where(nd, th_n, th_d)
            own.m[uid] = np.where(nd, m_n, m_d)
            own.v[uid] = np.where(nd, v_n, v_d)
        self.pending_updates = []

    # -- one iteration ---------------------------------------------------------
    def step(self, tokens):
        cfg, P = self.cfg, self.P
        N, B, S1 = tokens.shape
        if N % P:
            raise ValueError("N mod P != 0")
        m = N // P
        denom = float(N * B * cfg.seq)
        self.t += 1
        ver = self.t
        self.fabric = Fabric(P)
        self.pending_updates = []
        self.bwd_done = defaultdict(int)
        Lc = cfg.n_layers
        H, V = cfg.hidden, cfg.vocab
        seqs = {dev.d: [tokens[n, b] for n in range(dev.d * m, (dev.d + 1) * m) for b in range(B)]
                for dev in self.devices}
        # ---- E: gather, embed (a4) ----
        self.gather("E", ver)
        hs, cache = {}, {}
        for dev in self.devices:
            E = self.weights(dev, "E", ver)[:V * H].reshape(V, H)
            hs[dev.d] = [E[sq[:-1]] for sq in seqs[dev.d]]
        self.release("E")
        # ---- forward (a3, a5) ----
        for l in range(Lc):
            self.gather(l, ver)
            for dev in self.devices:
                W = layout.unflatten_layer(self.weights(dev, l, ver)[:self.units[l].n], cfg)
                for i, h in enumerate(hs[dev.d]):
                    hs[dev.d][i], cache[(dev.d, l, i)] = layer_fwd(h, W, cfg, self.cos, self.sin)
            if not (self.r == 1 and l == Lc - 1):
                self.release(l)
        # ---- head F: gather, forward + backward back to back (a6) ----
        self.gather("F", ver)
        loss_parts, dhs, gF = [], {}, {}
        for dev in self.devices:
            full = self.weights(dev, "F", ver)
            fn, head = layout.unflatten_F(full[:self.units["F"].n], cfg)
            g = np.zeros(self.units["F"].n_pad)
            dhs[dev.d] = []
            lp = 0.0
            for i, sq in enumerate(seqs[dev.d]):
                loss, dh, dfn, dhead = head_fwd_bwd(hs[dev.d][i], fn, head, sq[1:], denom, cfg)
                lp += loss
                dhs[dev.d].append(dh)
                g[:H] += dfn
                g[H:H + V * H] += dhead.reshape(-1)
            loss_parts.append(lp)
            gF[dev.d] = g
        self.release("F")
        self.bwd_done["F"] = P
        self.reduce("F", gF)
        # ---- backward (a7, a8) ----
        consumed = set()
        for l in range(Lc - 1, -1, -1):
            if not (self.r == 1 and l == Lc - 1):
                self.gather(l, ver)
            if self.mutate == "update_before_bwd" and l == 0:
                self.reduce(0, {dev.d: np.zeros(self.units[0].n_pad) for dev in self.devices})
                self.apply_updates()
            grads = {}
            for dev in self.devices:
                W = layout.unflatten_layer(self.weights(dev, l, ver)[:self.units[l].n], cfg)
                g = np.zeros(self.units[l].n_pad)
                for i in range(len(seqs[dev.d])):
                    key = (dev.d, l, i)
                    if key in consumed or key not in cache:
                        raise ValidationError("activation-consume-once", f"activation {key} consumed twice")
                    consumed.add(key)
                    c = cache.pop(key)
                    if self.mutate == "double_consume" and l == 0 and i == 0:
                        cache[key] = c
                    dhs[dev.d][i], gl = layer_bwd(dhs[dev.d][i], W, c, cfg, self.cos, self.sin)
                    g[:self.units[l].n] += layout.flatten_layer(gl, cfg)
                grads[dev.d] = g
                self.bwd_done[l] += 1
            self.release(l)
            self.reduce(l, grads)
        if cache:
            raise ValidationError("activation-consume-once", f"activations never consumed: {sorted(cache)[:3]}")
        # ---- E backward (a4): scatter-add, sequential ----
        gE = {}
        for dev in self.devices:
            g = np.zeros((V, H))
            for i, sq in enumerate(seqs[dev.d]):
                np.add.at(g, sq[:-1], dhs[dev.d][i])
            ge = np.zeros(self.units["E"].n_pad)
            ge[:V * H] = g.reshape(-1)
            gE[dev.d] = ge
        self.bwd_done["E"] = P
        self.reduce("E", gE)
        if self.mutate == "unmatched_send":
            self.fabric.send(0, P - 1, ("X",), np.zeros(1), "w", "inter", "block")
        # ---- a9: owner updates (after every backward of the iteration) ----
        self.apply_updates()
        self.fabric.assert_drained()
        # ---- a10: loss = Σ device partials / (N·B·S) ----
        return float(sum(loss_parts)) / denom

    # -- read back -------------------------------------------------------------
    def assemble(self) -> dict:
        """Reassemble full float64 parameters from the owners' stripes."""
        vecs = {}
        for uid, u in self.units.items():
            full = np.empty(u.n_pad)
            for j in range(self.G):
                full[j * u.s:(j + 1) * u.s] = self.dev(u.owner, j).master[uid]
            vecs[uid] = full[:u.n]
        cfg = self.cfg
        fn, head = layout.unflatten_F(vecs["F"], cfg)
        return {"embed": vecs["E"].reshape(cfg.vocab, cfg.hidden),
                "layers": [layout.unflatten_layer(vecs[l], cfg) for l in range(cfg.n_layers)],
                "final_norm": fn, "head": head}

    def stripe_lengths(self):
        return self.units[0].s, self.units["E"].s, self.units["F"].s
