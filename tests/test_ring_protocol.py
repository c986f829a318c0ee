"""Protocol model of the persistent multi-GPU ring (k_ring, csrc/bfly_ring.cu), run
under random interleavings on the CPU — the 8-GPU ring cannot be run through gpurun,
so this checks the exchange itself for G up to 8:

* rank 0 deals tiles from a shared counter (one per chain step of a lane) and writes
  the schedule ahead; lane c of every later rank processes the tiles lane c of rank 0
  took, in the same order, and a tile id of -1 ends the lane's round;
* chain: rank g adds its miners to the running sums of a tile and stores them into
  rank g+1's slot ring (NB slots per lane); the last rank divides and stores the final
  tile into rank 0's final-value ring; relay: last -> 0 -> 1 -> ... -> G-2;
* a producer publishes a step `lag` steps after storing it (or at the end of the lane);
  a consumer returns a slot (credit) once its contents are read; a producer waits for
  the credit of step j - NB before storing step j; step counts persist across rounds.

Checked: no deadlock, every tile reduced exactly once from the sums of all ranks in
rank order, every rank's replicas receive every final tile exactly once, and the
schedule ring is never overwritten before it is read (kSR >= (G-1)(kNT+NB)+1 slack is
modelled by the loader lead kNT)."""

import random

import pytest

KNT = 8  # chain steps a loader may lead its storer by (tile-id ring)


class Ring:
    def __init__(self, G, L, NB, lag, T, SR, rng):
        self.G, self.L, self.NB, self.lag, self.T, self.SR, self.rng = G, L, NB, lag, T, SR, rng
        self.Z = G - 1
        # flags in the waiter's region: [rank][lane]
        z = lambda: [[0] * L for _ in range(G)]  # noqa: E731
        self.acc_ready, self.acc_free, self.fin_ready, self.fin_free = z(), z(), z(), z()
        self.acc_slot = [[[None] * NB for _ in range(L)] for _ in range(G)]
        self.fin_slot = [[[None] * NB for _ in range(L)] for _ in range(G)]
        self.sched = [[[None] * SR for _ in range(L)] for _ in range(G)]
        self.steps_c = z()  # persisted step counts (chain side, relay side)
        self.steps_r = z()

    # -- one round -----------------------------------------------------------
    def round(self):
        G, Z, L = self.G, self.Z, self.L
        self.counter = 0
        self.reduced = {}  # tile -> sums (list of ranks, in order)
        self.received = [dict() for _ in range(G)]  # rank -> tile -> count
        procs = []
        for c in range(L):
            for g in range(G):
                procs.append(self.chain(g, c))
                if g < Z:
                    procs.append(self.relay(g, c))
        live = {i: p for i, p in enumerate(procs)}
        # each generator yields a predicate it is waiting on; None = runnable
        waits = {i: None for i in live}
        while live:
            runnable = [i for i in live if waits[i] is None or waits[i]()]
            if not runnable:
                raise AssertionError("deadlock")
            i = self.rng.choice(runnable)
            try:
                waits[i] = next(live[i])
            except StopIteration:
                del live[i]
        T = self.T
        assert sorted(self.reduced) == list(range(T)), "every tile reduced exactly once"
        for t, sums in self.reduced.items():
            assert sums == list(range(G)), (t, sums)  # rank order 0..G-1
        for g in range(G):
            assert sorted(self.received[g]) == list(range(T)) and set(self.received[g].values()) == {1}, g

    def chain(self, g, c):
        """Loader + compute + storer of one lane of rank g, at slot granularity."""
        NB, lag, Z = self.NB, self.lag, self.Z
        base = self.steps_c[g][c]
        out_rank = g + 1 if g < Z else 0
        i = 0
        dealt = []  # rank 0: tiles dealt ahead of the store (the loader leads by up to KNT steps)
        next_deal = base
        while True:
            j = base + i
            # the tile of step j
            if g == 0:
                while len(dealt) < KNT and (not dealt or dealt[-1] >= 0):
                    if self.counter < self.T:
                        t = self.counter
                        self.counter += 1
                    else:
                        t = -1
                    for r in range(1, self.G):
                        w = self.sched[r][c][next_deal % self.SR]
                        # the word of step next_deal - SR must have been read by now
                        assert w is None or w[2], ("schedule overwritten before it was read", r, c, next_deal)
                        self.sched[r][c][next_deal % self.SR] = [next_deal + 1, t, False]
                    dealt.append(t)
                    next_deal += 1
                    yield None
                tile = dealt.pop(0)
            else:
                yield lambda: (self.sched[g][c][j % self.SR] or [0])[0] == j + 1
                w = self.sched[g][c][j % self.SR]
                tile = w[1]
                w[2] = True
            yield None
            # incoming sums (ranks > 0), then the slot goes back to the producer
            sums = []
            if g > 0:
                yield lambda: self.acc_ready[g][c] >= j + 1
                slot = self.acc_slot[g][c][j % NB]
                assert slot is not None and slot[0] == tile and slot[2] == j, (g, c, j, slot, tile)
                sums = list(slot[1])
                self.acc_slot[g][c][j % NB] = None
                self.acc_free[g - 1][c] = j + 1
            yield None
            if tile >= 0:
                sums = sums + [g]
            # the downstream slot must be free
            free = self.fin_free if g == Z else self.acc_free
            yield lambda: j < NB or free[g][c] >= j + 1 - NB
            ring = self.fin_slot if g == Z else self.acc_slot
            assert ring[out_rank][c][j % NB] is None, "slot overwritten before it was read"
            if g == Z:
                ring[out_rank][c][j % NB] = (tile, None, j)
                if tile >= 0:
                    assert tile not in self.reduced
                    self.reduced[tile] = sums
                    self.received[Z][tile] = self.received[Z].get(tile, 0) + 1
            else:
                ring[out_rank][c][j % NB] = (tile, sums, j)
            ready = self.fin_ready if g == Z else self.acc_ready
            if i >= lag:
                ready[out_rank][c] = max(ready[out_rank][c], j + 1 - lag)
            yield None
            if tile < 0:
                break
            i += 1
        ready = self.fin_ready if g == Z else self.acc_ready
        ready[out_rank][c] = base + i + 1
        self.steps_c[g][c] = base + i + 1

    def relay(self, g, c):
        NB, lag, Z = self.NB, self.lag, self.Z
        base = self.steps_r[g][c]
        pred = Z if g == 0 else g - 1
        succ = g + 1 if g + 1 < Z else None
        i = 0
        while True:
            j = base + i
            yield lambda: self.fin_ready[g][c] >= j + 1
            slot = self.fin_slot[g][c][j % NB]
            assert slot is not None and slot[2] == j
            tile = slot[0]
            self.fin_slot[g][c][j % NB] = None
            self.fin_free[pred][c] = j + 1
            if tile >= 0:
                self.received[g][tile] = self.received[g].get(tile, 0) + 1
            yield None
            if succ is not None:
                yield lambda: j < NB or self.fin_free[g][c] >= j + 1 - NB
                assert self.fin_slot[succ][c][j % NB] is None
                self.fin_slot[succ][c][j % NB] = (tile, None, j)
                if i >= lag:
                    self.fin_ready[succ][c] = max(self.fin_ready[succ][c], j + 1 - lag)
            yield None
            if tile < 0:
                break
            i += 1
        if succ is not None:
            self.fin_ready[succ][c] = base + i + 1
        self.steps_r[g][c] = base + i + 1


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("NB,lag", [(2, 1), (3, 1), (4, 2), (10, 1)])
def test_ring_protocol_random_interleavings(G, NB, lag):
    for seed in range(6):
        rng = random.Random(1000 * G + 10 * NB + seed)
        T = rng.choice([1, 5, 17, 40])
        L = rng.choice([1, 3, 4])
        SR = (G - 1) * (KNT + NB) + 1 + 8
        ring = Ring(G, L, NB, lag, T, SR, rng)
        for _ in range(3):  # persisted step counts carry the flags across rounds
            ring.round()
