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


# ----------------------------------------------------------------------------------------
# Halo mode 3: copy-engine pull ordered by flags (rtm_host.cpp step_slabs_pull).  Per rank r
# and step n, with b = n&1, b2 = (n+1)&1:
#   main stream: boundary kernel (after its own pulls of step n-1, stream order): reads its
#                  halos of b (must hold u^n), writes its boundary planes of b2 (u^{n+1})
#                  anywhere inside the kernel interval
#                signal B := n+1 into both neighbours ("boundary ready")
#                interior kernel (own planes only: no cross-rank hazard, not modelled)
#                wait for its own comm stream's pulls of step n (event)
#   comm stream: after the boundary kernel (local event): wait B_lo >= n+1, copy the lo
#                neighbour's boundary of b2 into its own lo halo of b2 (an interval); the same
#                for hi
# There is no "step complete" flag: the WAR hazard (my step-n boundary overwrites the u^{n-1}
# planes my neighbour pulled at its step n-2) is ordered transitively — my boundary n follows
# my pulls of n-1, which wait for the neighbour's boundary n-1, which follows the neighbour's
# pulls of n-2.  The model checks exactly that (with_f=True adds the redundant F wait back).
# The rank's reset pull of u^0 (peer contexts: barrier, then copies) precedes its first step
# and may overlap the neighbours' first steps.  Checked: halo reads see u^n (RAW), copies read
# the neighbour's u^{n+1} and never overlap a write of it (RAW / WAR), no deadlock.

def simulate_pull(G, steps, seed, drop=None, fresh=True, initial_flag=0, with_f=False):
    rng = random.Random(seed)
    F = [[initial_flag, initial_flag] for _ in range(G)]  # F[r][side]: neighbour's steps done
    B = [[initial_flag, initial_flag] for _ in range(G)]  # B[r][side]: neighbour's boundary ready
    halo = [[[0, 0], [-1, -1]] for _ in range(G)]  # u^k held by r's halo of buffer b, side
    bnd = [[0, -1] for _ in range(G)]              # u^k held by r's own boundary planes of b
    writing = [None] * G                            # buffer r's boundary kernel is writing
    reading = [dict() for _ in range(G)]            # copies in flight reading r's boundary: id -> b
    violations = []
    lo_ex = [r > 0 for r in range(G)]
    hi_ex = [r < G - 1 for r in range(G)]
    # programs: lists of ops; each op is a function returning True (done) or False (blocked)
    main_pc, comm_pc = [0] * G, [0] * G
    bnd_done = [-1] * G    # last step whose boundary kernel ended (event for the comm stream)
    comm_done = [-2] * G   # last step whose pulls ended (-1: the reset pull)

    def main_ops(r, n):
        b, b2 = n & 1, (n + 1) & 1
        ops = []

        def war(side):
            def f():
                exists = lo_ex[r] if side == 0 else hi_ex[r]
                if not with_f or not exists or (fresh and n == 0):
                    return True
                return F[r][side] >= n - 1
            return f
        ops += [war(0), war(1)]

        def start_bnd():
            # stream order: own pulls of step n-1 (or the reset pull) done
            if comm_done[r] < n - 1 and drop != (r, "join"):
                return False
            for side, ex in ((0, lo_ex[r]), (1, hi_ex[r])):
                if ex and halo[r][b][side] != n:
                    violations.append(f"RAW rank {r} step {n} side {side}: halo holds u^{halo[r][b][side]}")
            for q in (r - 1, r + 1):
                if 0 <= q < G and b2 in reading[r].values():
                    violations.append(f"WAR rank {r} step {n}: rank {q} still copies its boundary of buffer {b2}")
            writing[r] = b2
            return True

        def end_bnd():
            for cid, bb in reading[r].items():
                if bb == b2:
                    violations.append(f"WAR rank {r} step {n}: a copy of buffer {b2} overlapped the write")
            bnd[r][b2] = n + 1
            writing[r] = None
            bnd_done[r] = n
            if r > 0:
                B[r - 1][1] = n + 1
            if r < G - 1:
                B[r + 1][0] = n + 1
            return True

        def join_and_signal():
            if comm_done[r] < n:
                return False
            if r > 0:
                F[r - 1][1] = n + 1
            if r < G - 1:
                F[r + 1][0] = n + 1
            return True
        return ops + [start_bnd, end_bnd, join_and_signal]

    def comm_ops(r, n):
        b2 = (n + 1) & 1
        ops = [lambda: bnd_done[r] >= n]
        for side, d in ((0, -1), (1, 1)):
            if not (lo_ex[r] if side == 0 else hi_ex[r]):
                continue
            q = r + d
            cid = (r, n, side)

            def wait_b(side=side):
                return drop == (r, "raw", side) or B[r][side] >= n + 1

            def copy_start(q=q, cid=cid):
                if writing[q] == b2 or bnd[q][b2] != n + 1:
                    violations.append(f"RAW rank {r} step {n}: pull from rank {q} buffer {b2} "
                                      f"holding u^{bnd[q][b2]} (writing={writing[q]})")
                reading[q][cid] = b2
                return True

            def copy_end(q=q, cid=cid, side=side):
                if bnd[q][b2] != n + 1:
                    violations.append(f"WAR rank {r} step {n}: rank {q} overwrote buffer {b2} during the pull")
                del reading[q][cid]
                halo[r][b2][side] = n + 1
                return True
            ops += [wait_b, copy_start, copy_end]

        def done():
            comm_done[r] = n
            return True
        return ops + [done]

    def reset_pull(r):
        ops = []
        for side, d in ((0, -1), (1, 1)):
            if not (lo_ex[r] if side == 0 else hi_ex[r]):
                continue
            q = r + d
            cid = (r, -1, side)

            def cs(q=q, cid=cid):
                reading[q][cid] = 0
                return True

            def ce(q=q, cid=cid):
                if bnd[q][0] != 0:
                    violations.append(f"WAR rank {q} overwrote buffer 0 during rank {r}'s reset pull")
                del reading[q][cid]
                return True
            ops += [cs, ce]

        def done():
            comm_done[r] = -1
            return True
        return ops + [done]

    mains = [[op for n in range(steps) for op in main_ops(r, n)] for r in range(G)]
    comms = [reset_pull(r) + [op for n in range(steps) for op in comm_ops(r, n)] for r in range(G)]
    while True:
        cand = [("m", r) for r in range(G) if main_pc[r] < len(mains[r])] + \
               [("c", r) for r in range(G) if comm_pc[r] < len(comms[r])]
        if not cand:
            break
        rng.shuffle(cand)
        progressed = False
        for kind, r in cand:
            prog, pc = (mains, main_pc) if kind == "m" else (comms, comm_pc)
            if prog[r][pc[r]]():
                pc[r] += 1
                progressed = True
                break
        if not progressed:
            violations.append("deadlock")
            break
    return violations


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_pull_protocol_is_race_free_and_live(G):
    for seed in range(300):
        v = simulate_pull(G, steps=7, seed=seed)
        assert not v, (seed, v[:3])


def test_pull_protocol_with_the_redundant_step_flag_is_also_clean():
    for seed in range(200):
        assert not simulate_pull(3, steps=7, seed=seed, with_f=True)


@pytest.mark.parametrize("drop", [(1, "raw", 0), (1, "raw", 1), (0, "raw", 1), (1, "join")])
def test_pull_model_catches_a_dropped_wait(drop):
    """Drop a 'boundary ready' wait, or the boundary kernel's stream order after its own pulls
    (the link the WAR argument rests on): some schedule must expose a hazard."""
    assert any(simulate_pull(3, steps=6, seed=s, drop=drop) for s in range(400))


def test_pull_model_catches_stale_flags():
    assert any(simulate_pull(3, steps=6, seed=s, initial_flag=99) for s in range(300))
    assert not any(simulate_pull(3, steps=6, seed=s) for s in range(300))
