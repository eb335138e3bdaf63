"""Compare the owned shards of two multi-GPU runs (tests/mp_worker.py outputs), per rank and per unit:
python tools/p2p_compare.py DIR_A DIR_B P G L H I V"""
import sys
import numpy as np

a, b = sys.argv[1], sys.argv[2]
P, G, L, H, I, V = (int(x) for x in sys.argv[3:9])
D = P // G
phi = 4 * H * H + 3 * H * I + 2 * H


def padded(n, G):
    q = G * 64
    return q * ((n + q - 1) // q)


for r in range(P):
    xa, xb = np.load(f"{a}/rank{r}.npz"), np.load(f"{b}/rank{r}.npz")
    sa, sb = xa["shard"], xb["shard"]
    k = r // G
    units = [(l, phi) for l in range(L) if l % D == k] + ([("E", V * H)] if k == 0 else []) + \
            ([("F", H + V * H)] if k == D - 1 else [])
    off = 0
    out = []
    for uid, n in units:
        s = padded(n, G) // G
        d = np.abs(sa[off:off + s] - sb[off:off + s])
        out.append(f"{uid}:{d.max():.2e}")
        off += s
    print(f"rank {r} losses {xa['losses']} vs {xb['losses']}  " + " ".join(out))
