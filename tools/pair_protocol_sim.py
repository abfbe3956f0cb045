"""Randomised simulation of attn_fwd_pair.cu's synchronisation protocol (deadlock check, CPU).

Models the producer (item claims, Q loads, the merged K/V schedule with its meta words, a ring of
R slots), the polling MMA issuer (two streams; S after the stream's previous PV completed, PV after
P and, for an item's first PV, after the epilogue drained O), the two softmax streams, the
epilogue (per item, stream 0 then 1; releases O, then the Q buffer after its store) and
asynchronous MMA completion. Every step runs one random actor that can make progress; a state in
which no actor can move before all work is done is a deadlock.

    python tools/pair_protocol_sim.py [--trials 2000]
"""
from __future__ import annotations

import argparse
import random


def schedule(L0, L1):
    """The producer's merged load list for one item: [(kind, streams, first, last)] in load order."""
    loads = []
    i0 = i1 = 0
    n0, n1 = len(L0), len(L1)
    INF = 1 << 30
    while i0 < n0 or i1 < n1:
        a = L0[i0] if i0 < n0 else INF
        b = L1[i1] if i1 < n1 else INF

        def soon(L, i, c):
            return any(i + d < len(L) and L[i + d] == c for d in (1, 2))

        if a == b:
            u0 = u1 = True
        elif a < b:
            u0, u1 = True, i1 < n1 and not soon(L0, i0, b)
        else:
            u1, u0 = True, i0 < n0 and not soon(L1, i1, a)
        shared = u0 and u1 and a == b
        f = {0: u0 and i0 == 0, 1: u1 and i1 == 0}
        last = {0: u0 and i0 + 1 == n0, 1: u1 and i1 + 1 == n1}
        if shared:
            loads.append(("K", {0, 1}, f, last))
            loads.append(("V", {0, 1}, f, last))
        else:
            if u0:
                loads.append(("K", {0}, f, last))
            if u1:
                loads.append(("K", {1}, f, last))
            if u0:
                loads.append(("V", {0}, f, last))
            if u1:
                loads.append(("V", {1}, f, last))
        i0 += u0
        i1 += u1
    return loads


def simulate(items, R, rng):
    # ---- producer state
    all_loads = []
    for (L0, L1) in items:
        all_loads.append(("ITEM", (len(L0), len(L1))))
        all_loads.extend(schedule(L0, L1))
    all_loads.append(("END",))
    prod_i = 0
    ring = {}                 # position -> meta
    released = set()          # positions released
    lpos = 0
    q_loaded = {0: [], 1: []}  # per stream: list of items whose Q was loaded (buffer = index % 2)
    q_free = {(s, 0): True for s in (0, 1)}
    qb_prod = {0: 0, 1: 0}
    item_idx = -1
    # ---- issuer
    pos = [0, 0]
    pend = [None, None]
    done = [False, False]
    pv_out = [None, None]     # id of the stream's latest PV (must complete before its next S)
    cons = {}
    q_ready = {}              # (s, buffer) -> loaded & not consumed (bool)
    qb_iss = [0, 0]
    # ---- async MMA completions
    inflight = []             # (kind, stream, id)
    completed = set()
    mma_id = 0
    s_ready = {0: 0, 1: 0}    # completed S count per stream
    s_issued = {0: 0, 1: 0}
    p_ready = {0: 0, 1: 0}    # P written by the engine
    pv_issued = {0: 0, 1: 0}
    o_empty = {0: 1, 1: 1}    # epilogue drains granted (first PV of an item consumes one)
    o_full = {0: [], 1: []}   # PV-last completions pending (per item of that stream)
    last_pv_pending = {0: [], 1: []}
    # engine: tiles per stream per item
    eng_items = {0: [len(a) for a, _ in items], 1: [len(b) for _, b in items]}
    eng_pos = {0: [0, 0], 1: [0, 0]}  # (item, tile)
    stats = {0: [], 1: []}
    epi_item = 0
    epi_stream = 0
    epi_stage = 0
    total_tiles = {0: sum(eng_items[0]), 1: sum(eng_items[1])}

    def producer_step():
        nonlocal prod_i, lpos, item_idx
        if prod_i >= len(all_loads):
            return False
        e = all_loads[prod_i]
        if e[0] == "ITEM":
            n0, n1 = e[1]
            # Q loads wait for the buffer (epilogue of the item two back)
            for s, n in ((0, n0), (1, n1)):
                if n and not q_free[(s, 0)]:
                    return False
            item_idx += 1
            for s, n in ((0, n0), (1, n1)):
                if n:
                    q_free[(s, 0)] = False
                    q_ready[(s, 0)] = True
            prod_i += 1
            return True
        # a K/V load or END into ring slot lpos % R: the position R back must be released
        if lpos >= R and (lpos - R) not in released:
            return False
        ring[lpos] = e
        lpos += 1
        prod_i += 1
        return True

    def release_pass(p):
        cons[p] = cons.get(p, 0) + 1
        if cons[p] == 2:
            released.add(p)

    def issuer_step(s):
        nonlocal mma_id
        if done[s]:
            return False
        if pend[s] is None:
            p = pos[s]
            if p not in ring:
                return False
            e = ring[p]
            if e[0] == "END":
                done[s] = True
                return True
            if s not in e[1]:
                release_pass(p)
                pos[s] += 1
                return True
            pend[s] = (p, e)
            pos[s] += 1
            return True
        p, e = pend[s]
        kind, _, first, last = e
        if kind == "K":
            if first[s] and not q_ready.get((s, 0), False):
                return False
            if pv_out[s] is not None and pv_out[s] not in completed:
                return False
            if first[s]:
                q_ready[(s, 0)] = False
            pv_out[s] = None
            mma_id += 1
            inflight.append(("S", s, mma_id, last[s]))
            s_issued[s] += 1
        else:
            if p_ready[s] <= pv_issued[s]:
                return False
            if first[s] and o_empty[s] == 0:
                return False
            if first[s]:
                o_empty[s] -= 1
            mma_id += 1
            inflight.append(("PV", s, mma_id, last[s]))
            pv_out[s] = mma_id
            pv_issued[s] += 1
        release_pass(p)
        pend[s] = None
        return True

    def complete_step():
        if not inflight:
            return False
        # in order per issuing thread: complete the oldest
        op = inflight.pop(0)
        completed.add(op[2])
        if op[0] == "S":
            s_ready[op[1]] += 1
            if op[3]:
                q_free[(op[1], 0)] = True
        elif op[3]:
            o_full[op[1]].append(True)
        return True

    def engine_step(s):
        it, t = eng_pos[s]
        while it < len(items) and eng_items[s][it] == 0:
            it += 1
            t = 0
        eng_pos[s] = [it, t]
        if it >= len(items):
            return False
        done_tiles = sum(eng_items[s][:it]) + t
        if s_ready[s] <= done_tiles:
            return False
        p_ready[s] += 1
        t += 1
        if t == eng_items[s][it]:
            stats[s].append(it)
            it, t = it + 1, 0
        eng_pos[s] = [it, t]
        return True

    def epilogue_step():
        nonlocal epi_item, epi_stream, epi_stage
        while epi_item < len(items):
            n = len(items[epi_item][epi_stream])
            if n:
                break
            epi_stream += 1
            if epi_stream == 2:
                epi_stream, epi_item = 0, epi_item + 1
        if epi_item >= len(items):
            return False
        s = epi_stream
        if epi_item not in stats[s] or not o_full[s]:
            return False
        o_full[s].pop(0)
        o_empty[s] += 1
        epi_stream += 1
        if epi_stream == 2:
            epi_stream, epi_item = 0, epi_item + 1
        return True

    actors = [producer_step, lambda: issuer_step(0), lambda: issuer_step(1), complete_step,
              lambda: engine_step(0), lambda: engine_step(1), epilogue_step]
    steps = 0
    while True:
        order = list(range(len(actors)))
        rng.shuffle(order)
        moved = False
        for a in order:
            if actors[a]():
                moved = True
                break
        steps += 1
        if not moved:
            finished = (done[0] and done[1] and epi_item >= len(items) and not inflight)
            return finished, steps


def random_lists(rng, kcols):
    kind = rng.choice(["band", "disjoint", "random", "empty", "same", "long"])
    def band(c, w):
        return list(range(max(0, c - w), min(kcols, c + w + 1)))
    if kind == "band":
        c = rng.randrange(kcols)
        w = rng.randrange(0, 3)
        return band(c, w), band(min(kcols - 1, c + 1), w)
    if kind == "disjoint":
        cut = rng.randrange(1, kcols)
        return sorted(rng.sample(range(cut), rng.randrange(1, cut + 1))), sorted(
            rng.sample(range(cut, kcols), rng.randrange(1, kcols - cut + 1)))
    if kind == "random":
        return (sorted(rng.sample(range(kcols), rng.randrange(0, kcols + 1))),
                sorted(rng.sample(range(kcols), rng.randrange(0, kcols + 1))))
    if kind == "empty":
        return ([], sorted(rng.sample(range(kcols), rng.randrange(1, kcols + 1)))) if rng.random() < .5 else \
            (sorted(rng.sample(range(kcols), rng.randrange(1, kcols + 1))), [])
    if kind == "same":
        L = sorted(rng.sample(range(kcols), rng.randrange(1, kcols + 1)))
        return L, list(L)
    L0 = list(range(kcols))
    return L0, sorted(rng.sample(range(kcols), rng.randrange(0, 3)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=2000)
    a = ap.parse_args()
    rng = random.Random(1)
    for trial in range(a.trials):
        kcols = rng.randrange(2, 12)
        items = [random_lists(rng, kcols) for _ in range(rng.randrange(1, 7))]
        R = rng.choice([3, 4, 8])
        ok, steps = simulate(items, R, rng)
        if not ok:
            print("DEADLOCK", trial, "R", R, items)
            return 1
    print(f"{a.trials} trials: no deadlock")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
