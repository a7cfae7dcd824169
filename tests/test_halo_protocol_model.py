"""Model check of the fused-halo flag protocol (halo mode 2; rtm_host.cpp
step_slabs_signal).  The distributed form of this protocol cannot run on this round's single
GPU, so its ordering rules are checked here on an abstract model, CPU only:

  * G ranks; rank r's stream executes, per step n:
        wait(flag_lo[r] >= n)   (skipped on the first step after a synchronising reset)
        wait(flag_hi[r] >= n)
        kernel(n): READS its halo planes of buffer n&1 (pushed by the neighbours' step n-1) and
                   its own interior; WRITES its interior of buffer (n+1)&1 and PUSHES its boundary
                   planes into the neighbours' halo planes of buffer (n+1)&1
        signal(n+1) into flag_hi[r-1] and flag_lo[r+1]
  * A kernel is an interval (start ... end), not an atomic event, and streams interleave
    arbitrarily (random schedules).

Checked: every halo read sees exactly the neighbour's step n-1 data (RAW), and — with pushes
allowed anywhere inside the kernel interval — no push can land in a halo plane before the
neighbour's kernel that reads it has ended (WAR); no deadlock.  A mutated protocol (one wait dropped) must be caught — so the model can fail."""
from __future__ import annotations

import random

import pytest


def simulate(G, steps, seed, drop_wait=None, fresh=True, initial_flag=0):
    """Random interleaving of the G streams; returns a list of violations.  initial_flag models
    what the flag words hold when the run starts: 0 in a fresh generation (the library compares
    against gen << 40 | n, so a previous generation's values are always smaller)."""
    rng = random.Random(seed)
    # flags[r] = [from_lo, from_hi]: steps completed by the neighbour (this generation)
    flags = [[initial_flag, initial_flag] for _ in range(G)]
    # halo[r][b][side] = step index whose data is in that halo of buffer b (-1 = initial fill)
    # the reset exchange fills the halos of both initial time levels (u^0 in buffer 0, u^{-1}
    # in buffer 1) before the first step
    halo = [[[0, 0], [-1, -1]] for _ in range(G)]
    running = [None] * G  # (step, buffer read) of the kernel in flight on rank r
    completed = [0] * G   # steps whose kernel has ended, per rank
    pc = [0] * G          # program counter: 4 ops per step (wait lo, wait hi, start, end)
    violations = []

    def op(r):
        n, k = divmod(pc[r], 4)
        lo, hi = r > 0, r < G - 1
        if k in (0, 1):  # waits
            side = k
            exists = lo if side == 0 else hi
            skip = (fresh and n == 0) or not exists or drop_wait == (r, side)
            if skip or flags[r][side] >= n:
                pc[r] += 1
                return True
            return False  # blocked
        if k == 2:  # kernel start: reads halos of buffer n&1 (both sides that exist)
            b = n & 1
            for side, exists in ((0, lo), (1, hi)):
                want = n  # u^n in the halo: pushed by the neighbour's step n-1 (or the reset, n=0)
                if exists and halo[r][b][side] != want:
                    violations.append(f"RAW rank {r} step {n} side {side}: halo holds "
                                      f"u^{halo[r][b][side]}, wants u^{want}")
            # pushes may land any time during this kernel: each neighbour must already have
            # finished its step n-1, the last reader of the halo planes this kernel overwrites
            for q in (r - 1, r + 1):
                if 0 <= q < G and completed[q] < n:
                    violations.append(f"WAR rank {r} step {n} may push while rank {q} has only "
                                      f"completed {completed[q]} steps")
            running[r] = (n, b)
            pc[r] += 1
            return True
        # k == 3: kernel end: pushes u^{n+1} into the neighbours' halos of buffer (n+1)&1, then
        # the signal kernel (stream-ordered after the stencil) releases steps done = n+1
        b2 = (n + 1) & 1
        for d, side_at_nb in ((-1, 1), (1, 0)):
            q = r + d
            if 0 <= q < G:
                if running[q] is not None and running[q][1] == b2:
                    violations.append(f"WAR rank {r} step {n} pushes into rank {q} buffer {b2} "
                                      f"while its step {running[q][0]} reads it")
                if halo[q][b2][side_at_nb] != n - 1 and not (n == 0 and halo[q][b2][side_at_nb] == -1):
                    violations.append(f"WAR rank {r} step {n}: rank {q}'s halo of buffer {b2} "
                                      f"held u^{halo[q][b2][side_at_nb]} (not yet consumed?)")
                halo[q][b2][side_at_nb] = n + 1
        running[r] = None
        completed[r] += 1
        if r > 0:
            flags[r - 1][1] = n + 1
        if r < G - 1:
            flags[r + 1][0] = n + 1
        pc[r] += 1
        return True

    total = 4 * steps
    while any(p < total for p in pc):
        ready = [r for r in range(G) if pc[r] < total]
        rng.shuffle(ready)
        progressed = False
        for r in ready:
            if op(r):
                progressed = True
                break
        if not progressed:
            violations.append("deadlock")
            break
    return violations


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_protocol_is_race_free_and_live(G):
    for seed in range(300):
        v = simulate(G, steps=7, seed=seed)
        assert not v, (seed, v[:3])


def test_model_catches_a_dropped_wait():
    """Drop rank 1's wait on its lo neighbour: some schedule must expose a RAW or WAR hazard."""
    found = any(simulate(3, steps=6, seed=s, drop_wait=(1, 0)) for s in range(300))
    assert found


def test_model_catches_stale_flags_without_a_generation_tag():
    """Flag words left high by a previous run (a protocol without the generation tag, or without
    the synchronising reset) let every wait pass at once: some schedule must expose a hazard,
    while the same schedules are clean in a fresh generation."""
    stale = [simulate(3, steps=6, seed=s, fresh=False, initial_flag=99) for s in range(300)]
    assert any(stale)
    assert not any(simulate(3, steps=6, seed=s, fresh=False) for s in range(300))
