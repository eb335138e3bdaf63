"""The paper's literal shard map and role routing (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

PAPER.md:123 §3.3: "group g_0 includes devices {P_0, …, P_{P/D−1}}, group g_1 …
Within group g_k (k ∈ [0, D−1]), device P_i (i ∈ [0, P/D−1]) holds weight shard
W_{(D·i+k) mod P}".  Master / staging roles are defined there but their selection
is not; SURVEY.md §8(c) R7 reads it as the *rail counterpart*: the holder, staging
and exit device for layer l inside group k is (k, ⌊l/D⌋ mod G) -- the member with
the same within-group index as the owner.
"""
from __future__ import annotations


def device_id(k: int, i: int, G: int) -> int:
    """Device index of member i of group k (contiguous groups; R5)."""
    return k * G + i


def shard_of_device(k: int, i: int, P: int, D: int) -> int:
    """device P_i of group g_k holds W_{(D·i+k) mod P}."""
    G = P // D
    if not (0 <= k < D and 0 <= i < G):
        raise ValueError("index out of range")
    return (D * i + k) % P


def owner_table(P: int, D: int) -> list:
    """owner_table[w] = device holding shard W_w (inverse of shard_of_device)."""
    G = P // D
    own = [None] * P
    for k in range(D):
        for i in range(G):
            w = shard_of_device(k, i, P, D)
            if own[w] is not None:
                raise AssertionError("shard map is not a bijection")
            own[w] = device_id(k, i, G)
    return own


def rail_counterpart(layer: int, k: int, P: int, D: int) -> int:
    """R7: the device of group k that holds / stages / exits layer ``layer`` (L = P layers)."""
    G = P // D
    return device_id(k, (layer // D) % G, G)


def forward_exchange(layer: int, k: int, P: int, D: int):
    """Who delivers W_layer to group k in forward, and who inside g_k receives it.

    Returns (source device, receiving device): the owner sends its shard to the
    rail counterpart of group k (R8: from the owner, not chained).  When the
    owner is in g_k, source == receiver.
    """
    own = owner_table(P, D)[layer]
    return own, rail_counterpart(layer, k, P, D)


def backward_route(layer: int, k: int, P: int, D: int):
    """Gradient of W_layer computed in group k: reduced to the exit device of g_k, then sent to the owner."""
    return rail_counterpart(layer, k, P, D), owner_table(P, D)[layer]
