"""Host test double of the device store's migration interface (TEST ONLY).

Moves particles with the C oracle (bit-identical to the reference mover) and
splits them into stay / prev / next exactly as partition_outgoing does
(runtime.cpp:46-62), so SlabWorld's exchange protocol can run over gloo on
CPU and be compared with the reference Simulation as a bitwise multiset.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_1904_03684_b200.errors import CflViolation
from paper_1904_03684_b200.partition import decompose, owner_of


class HostStore:
    def __init__(self, grid, species_p6, E, B, rank: int, world: int, lose_one: bool = False):
        self.grid = grid
        self.p = [[np.ascontiguousarray(a, dtype=np.float64).copy() for a in p6]
                  for p6 in species_p6]
        self.E, self.B = E, B
        self.rank, self.world = rank, world
        sub = decompose(grid, world)[rank]
        self.prev, self.next = sub.prev, sub.next
        self.out = [[None, None] for _ in self.p]
        self.cfl = None
        self.lose_one = lose_one

    def count(self, s):
        return len(self.p[s][0])

    def move_migrate(self, s, mp):
        p6 = self.p[s]
        bad = oracle.port_move_batch(p6, self.E, self.B, self.grid.as_tuple(), mp.dt, mp.qom,
                                     mp.pc_iterations)
        assert bad == -1
        dest = owner_of(p6[1], self.grid, self.world)
        ok = (dest == self.rank) | (dest == self.prev) | (dest == self.next)
        if not ok.all() and self.cfl is None:
            i = int(np.argmax(~ok))
            self.cfl = (f"particle {i} of species {s} moved from slab {self.rank} to "
                        f"non-neighbor slab {int(dest[i])} in one step")
        to_prev = (dest == self.prev) & (dest != self.rank)
        to_next = (dest == self.next) & (dest != self.rank) & ~to_prev
        stay = ~(to_prev | to_next)
        rec = np.stack(p6, axis=1)
        self.out[s] = [torch.from_numpy(rec[to_prev].copy()), torch.from_numpy(rec[to_next].copy())]
        self.p[s] = [np.ascontiguousarray(a[stay]) for a in p6]
        if self.lose_one and len(self.p[s][0]):
            self.p[s] = [a[1:].copy() for a in self.p[s]]

    def sync(self):
        if self.cfl is not None:
            raise CflViolation(self.cfl)

    def outbox(self, s, direction):
        return self.out[s][direction]

    def inbox_append(self, s, recs):
        r = recs.numpy()
        self.p[s] = [np.concatenate([a, r[:, k]]) for k, a in enumerate(self.p[s])]
