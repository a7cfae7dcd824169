"""Host logic of bench.py's tuner refinement (no GPU): finalists are the fastest distinct
(tile, z-chunk) pairs of the selection phase, re-timed in interleaved rounds, and the lowest
MEAN wins — not the lowest single window (power-cap drift)."""
from __future__ import annotations

import importlib.util
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


class FakeLib:
    """Stands in for the binding: rtm_autotune returns scripted per-entry times."""

    def __init__(self, per_tile_rounds):
        self.per_tile_rounds = per_tile_rounds  # tile -> list of times, one per round
        self.calls, self.tile, self.zchunk = [], None, None

    def rtm_autotune(self, h, nI, tiles, zchunks):
        self.calls.append((nI, list(tiles), list(zchunks)))
        seen = {}
        out = []
        for t in tiles:
            r = seen.get(t, 0)
            seen[t] = r + 1
            out.append(self.per_tile_rounds[t][r])
        return {}, np.array(out)

    def rtm_set_tile(self, h, t):
        self.tile = t

    def rtm_set_zchunk(self, h, z):
        self.zchunk = z

    def rtm_tile_name(self, t):
        return f"t{t}"


def test_refine_picks_lowest_mean_not_lowest_window():
    b = _bench()
    # selection: tile 48 looked fastest once; 35 is faster on average when interleaved
    cands = [10, 35, 48, 49, 35]
    zcs = [0, 0, 0, 0, 0]
    times = np.array([40.0, 33.0, 32.6, 33.5, 33.1])
    fake = FakeLib({35: [99.0, 99.0, 99.0], 48: [98.0, 101.0, 101.0], 49: [102.0, 102.0, 102.0]})
    r = b.refine_selection(fake, None, 12, cands, zcs, times, top=3)
    nI, t2, z2 = fake.calls[0]
    assert nI == 37                                   # >= 100 ms windows: ceil(100 / (32.6 / 12))
    assert t2 == [48, 35, 49] * 3 and z2 == [0] * 9      # distinct finalists, interleaved rounds
    assert r["selected"] == "t35" and fake.tile == 35 and fake.zchunk == 0
    assert r["mean_ms_per_step"]["t48/z0"] > r["mean_ms_per_step"]["t35/z0"]


def test_refine_distinguishes_zchunks_and_skips_nan():
    b = _bench()
    cands = [35, 35, 48, 49]
    zcs = [0, 64, 0, 0]
    times = np.array([10.0, 11.0, np.nan, 12.0])
    fake = FakeLib({35: [5.0, 9.0, 5.0, 9.0, 5.0, 9.0], 49: [1.0, 1.0, 1.0]})
    r = b.refine_selection(fake, None, 4, cands, zcs, times, top=2)
    nI, t2, z2 = fake.calls[0]
    assert nI == 40 and r["nI"] == 40                 # ceil(100 ms / 2.5 ms)
    assert t2 == [35, 35] * 3 and z2 == [0, 64] * 3       # NaN (failed) candidate never a finalist
    assert fake.tile == 35 and fake.zchunk == 0 and r["zchunk"] == 0


def test_refine_window_at_least_three_selection_windows():
    b = _bench()
    fake = FakeLib({1: [1.0] * 3, 2: [2.0] * 3})
    b.refine_selection(fake, None, 50, [1, 2], None, np.array([500.0, 600.0]), top=2)
    assert fake.calls[0][0] == 150                    # 3 nI when nI steps already exceed 100 ms


def test_refine_single_finalist_makes_no_call():
    b = _bench()
    fake = FakeLib({})
    r = b.refine_selection(fake, None, 4, [7], None, np.array([1.0]), top=4)
    assert fake.calls == [] and r["selected"] == "t7"
