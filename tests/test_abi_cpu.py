"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/rtm.h
declares, its host-only helpers are right, and it fails loudly without a GPU."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

import rtm_inputs as ri

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def P():
    from conftest import build_library
    build_library()
    import paper_1310_8232_b200 as P
    return P


def declared_functions():
    text = (ROOT / "include" / "rtm.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rtm_[a-z_]+)\s*\(", text)))


def test_header_declares_north_star_calls():
    names = declared_functions()
    for n in ("rtm_create", "rtm_set_velocity", "rtm_inject_source", "rtm_step", "rtm_read_field"):
        assert n in names


def test_library_exports_every_declared_symbol(P):
    import ctypes
    lib = ctypes.CDLL(str(ROOT / "paper_1310_8232_b200" / "librtm_b200.so"))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding wraps each one under the same name
    assert not [n for n in declared_functions() if not hasattr(P, n)]


def test_no_cpu_fallback_without_gpu(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.RtmError) as e:
        P.rtm_create(64, 64, 64, 10.0, 1e-3, ri.COEFFS_F32)
    assert "no CUDA device" in str(e.value)


def test_argument_validation_before_device(P):
    for args in [(0, 4, 4, 10.0, 1e-3), (4, 4, 4, -1.0, 1e-3), (4, 4, 4, 10.0, float("nan"))]:
        with pytest.raises(P.RtmError) as e:
            P.rtm_create(*args, ri.COEFFS_F32)
        assert e.value.code == P.RTM_EINVAL
    bad = ri.COEFFS_F32.copy()
    bad[1] = -bad[1]  # not a negative-definite second difference
    with pytest.raises(P.RtmError):
        P.rtm_create(8, 8, 8, 10.0, 1e-3, bad)


def test_nu_crit_closed_form(P):
    # 3D leapfrog bound 2/sqrt(3 S(pi)), S(pi) = 512/75 -> 5/sqrt(128)
    assert P.rtm_nu_crit(ri.COEFFS_F32) == pytest.approx(5 / np.sqrt(128), rel=1e-7)
    # second-order coefficients (-2, 1, 0...): S_max = 4 -> nu_crit = 1/sqrt(3)
    c2 = np.array([-2, 1, 0, 0, 0, 0], np.float32)
    assert P.rtm_nu_crit(c2) == pytest.approx(1 / np.sqrt(3), rel=1e-9)


@pytest.mark.parametrize("nz,world", [(1024, 8), (512, 2), (101, 3), (20, 2), (7, 1)])
def test_slab_range_partitions_exactly(P, nz, world):
    spans = [P.rtm_slab_range(nz, world, r) for r in range(world)]
    assert spans[0][0] == 0
    for (a, n), (b, _) in zip(spans, spans[1:]):
        assert a + n == b
    assert spans[-1][0] + spans[-1][1] == nz
    assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_slab_range_rejects_thin_slabs(P):
    with pytest.raises(P.RtmError):
        P.rtm_slab_range(19, 2, 0)
    with pytest.raises(P.RtmError):
        P.rtm_slab_range(64, 2, 2)


def test_halo_plan_layout(P):
    nx, ny, nzl = 8, 6, 12
    plane = nx * ny
    offs, cnt = P.rtm_halo_plan(nx, ny, nzl, 1, 3)
    assert cnt == 5 * plane
    assert offs == [5 * plane, 0, nzl * plane, (nzl + 5) * plane]
    offs0, _ = P.rtm_halo_plan(nx, ny, nzl, 0, 3)
    assert offs0[:2] == [-1, -1] and offs0[2] >= 0
    offs2, _ = P.rtm_halo_plan(nx, ny, nzl, 2, 3)
    assert offs2[2:] == [-1, -1] and offs2[0] >= 0


def test_tile_table(P):
    n = P.rtm_num_tiles()
    assert n >= 2 and P.rtm_tile_name(0) == "naive"
    assert all(P.rtm_tile_name(i).startswith(("tma", "stream", "tb2", "resident", "ms", "s2r")) for i in range(1, n))
    assert P.rtm_tile_name(n) is None and P.rtm_tile_name(-5) is None


def test_sass_has_tma_and_no_legacy_tensor_ops():
    """The tiled kernels use TMA (UTMALDG) and mbarrier sync; the path is not a GEMM, so no
    HMMA/UTC*MMA (BASELINE.json north_star: no tensor cores)."""
    import shutil
    import subprocess
    so = ROOT / "paper_1310_8232_b200" / "librtm_b200.so"
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in sass or "SM100" in sass.upper()
    assert "UTMALDG" in sass
    assert "SYNCS" in sass  # mbarrier operations
    assert "HMMA" not in sass
    # Blackwell-specific instructions the design relies on: packed FP32x2
    # arithmetic of the point update, TMA tensor stores of the two-step publication, and the
    # programmatic-dependent-launch wait / trigger of k_stream (griddepcontrol)
    for m in ("FFMA2", "FADD2", "UTMASTG", "ACQBULK", "PREEXIT"):
        assert m in sass, m


def test_select_mwmb_is_eq2_minmax(P):
    """MWMB (Eq. (2)): per candidate the worst time over processes, then
    the candidate with the smallest worst case.  Differs from min-of-min (MMMB, Eq. (1))."""
    t = np.array([[1.0, 2.0, 3.0],     # rank 0
                  [9.0, 2.5, 2.9]])    # rank 1: candidate 0 is fast on rank 0 only
    assert P.rtm_select_mwmb(t) == 1            # max = (9, 2.5, 3.0) -> candidate 1
    assert int(np.argmin(t.min(axis=0))) == 0    # MMMB would pick candidate 0
    rng = np.random.default_rng(0)
    for _ in range(50):
        m = rng.uniform(1, 10, (rng.integers(1, 9), rng.integers(1, 20)))
        assert P.rtm_select_mwmb(m) == int(np.argmin(m.max(axis=0)))
    m = np.array([[np.nan, 5.0, 4.0], [1.0, 4.0, 6.0]])
    assert P.rtm_select_mwmb(m) == 1  # a candidate that failed anywhere is never chosen
    assert P.rtm_select_mwmb(np.array([[2.0, 2.0]])) == 0  # ties -> lowest index


def test_async_calls_validate_before_device(P):
    """The asynchronous calls read/write caller memory after returning, so the binding refuses
    arrays it would have to convert (a temporary copy would die first); NULL contexts are
    rejected by the library itself (no device needed)."""
    with pytest.raises(ValueError):
        P.rtm_read_field_async(None, np.empty(8, np.float64))
    with pytest.raises(ValueError):
        P.rtm_set_velocity_async(None, np.ones((2, 4), np.float32)[:, ::2])
    for fn, args in ((P.rtm_sync, ()), (P.rtm_step_async, (1,)),
                     (P.rtm_read_field_async, (np.empty(4, np.float32),)),
                     (P.rtm_set_velocity_async, (np.ones(4, np.float32),))):
        with pytest.raises(P.RtmError) as e:
            fn(None, *args)
        assert e.value.code == P.RTM_EINVAL


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the oracle arm) prints one JSON line with the driver's keys;
    config 1 keeps it to a second of CPU."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]


def test_blocksize_lattice_paper_worked_example(P):
    """for 200x200x800 and P = 5, b_i = b_j = <1, 51, 101, 151, 200> and
    b_k = <1, 201, 401, 601, 800>, nC = 125; P = 10 / 20 give nC = 1000 / 8000."""
    assert P.rtm_blocksize_lattice(200, 5) == [1, 51, 101, 151, 200]
    assert P.rtm_blocksize_lattice(800, 5) == [1, 201, 401, 601, 800]
    for parts, nc in ((5, 125), (10, 1000), (20, 8000)):
        dims = [P.rtm_blocksize_lattice(s, parts) for s in (200, 200, 800)]
        assert all(len(b) == parts for b in dims)
        assert len(dims[0]) * len(dims[1]) * len(dims[2]) == nc
        for s, b in zip((200, 200, 800), dims):
            assert b[0] == 1 and b[-1] == s and b == sorted(set(b)) and all(1 <= x <= s for x in b)
    assert P.rtm_blocksize_lattice(3, 10) == [1, 2, 3]  # duplicates of a small S collapse
    for bad in ((0, 5), (10, 1)):
        with pytest.raises(P.RtmError):
            P.rtm_blocksize_lattice(*bad)


def test_peer_and_ipc_calls_validate_before_device(P):
    """The NCCL-free slab bootstrap (peer contexts): NULL contexts and impossible slab requests
    are rejected by the host code itself; without a GPU no peer context is created."""
    with pytest.raises(P.RtmError) as e:
        P.rtm_ipc_export(None)
    assert e.value.code == P.RTM_EINVAL
    with pytest.raises(P.RtmError) as e:
        P.rtm_ipc_import(None, None, None)
    assert e.value.code == P.RTM_EINVAL
    with pytest.raises(ValueError):
        P.rtm_ipc_import(None, b"short", None)
    with pytest.raises(P.RtmError) as e:
        P.rtm_set_host_barrier(None, lambda: None)
    assert e.value.code == P.RTM_EINVAL
    with pytest.raises(P.RtmError) as e:
        P.rtm_get_dims(None)
    assert e.value.code == P.RTM_EINVAL
    assert P.rtm_last_enqueue_ms(None) == -1.0
    for rank, world, nz in [(2, 2, 64), (0, 4, 30), (-1, 2, 64)]:  # rank out of range, thin slabs
        with pytest.raises(P.RtmError) as e:
            P.rtm_create_peer(16, 16, nz, 10.0, 1e-3, ri.COEFFS_F32, rank, world, 0)
        assert e.value.code == P.RTM_EINVAL
    assert P.RTM_IPC_RECORD_BYTES == 512


def _build_c_example(tmp_path):
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        pytest.skip("no C compiler")
    lib_dir = ROOT / "paper_1310_8232_b200"
    exe = tmp_path / "rtm_c1"
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "rtm_c1.c"), "-L", str(lib_dir), "-lrtm_b200",
                    f"-Wl,-rpath,{lib_dir}", "-lm", "-o", str(exe)], check=True)
    return exe


def test_c_example_builds_against_the_header_and_library(P, tmp_path):
    """examples/rtm_c1.c uses the C ABI from plain C (no Python): it compiles with -Wall -Werror
    against include/rtm.h, links librtm_b200.so, and without a GPU fails loudly (no fallback)."""
    import subprocess
    import torch
    exe = _build_c_example(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present (tests/test_gpu_round2.py runs it)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 1 and "no CUDA device" in r.stderr


def test_bench_slab_parity_sums_detect_changes():
    """bench.py's N > 1 self-check (`slab_parity`) compares two 64-bit sums of the fp32 bit
    patterns per slab: one flipped bit, a sign change of a zero, or two swapped planes must all
    change them; a bitwise-equal copy must not."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    g = torch.Generator().manual_seed(5)
    t = torch.randn((7, 5, 12), generator=g, dtype=torch.float32)
    t[3, 2, 4] = 0.0
    ref = bench.field_sums(t, planes_per_chunk=2)
    assert bench.field_sums(t.clone(), planes_per_chunk=3) == ref  # chunking does not matter
    a = t.clone()
    a.view(torch.int32)[1, 1, 1] ^= 1  # one ulp
    assert bench.field_sums(a) != ref
    b = t.clone()
    b[3, 2, 4] = -0.0  # equal as floats, different bits
    assert bench.field_sums(b) != ref
    c = t.clone()
    c[[2, 5]] = t[[5, 2]]  # two planes swapped: same plain sum, different weighted sum
    s1, s2 = bench.field_sums(c)
    assert s1 == ref[0] and s2 != ref[1]
