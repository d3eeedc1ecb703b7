"""Host-side checks (CPU, no GPU needed): the C-ABI library loads and exports
every symbol include/pf_gpu.h declares; validate() mirrors the reference's
rules; new_environment (the library's host C++) equals the oracle; the device
entry points fail loudly without a GPU."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

from tests.helpers import hashes_of, to_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pf_gpu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1412_4933_b200 import _lib

    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), n
    assert set(names) == set(_lib.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_library_is_sm100a():
    from paper_1412_4933_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    import ctypes as C

    from paper_1412_4933_b200 import _lib

    assert _lib.AGENT_DTYPE.itemsize == 40 and _lib.REPORT_DTYPE.itemsize == 16
    assert C.sizeof(_lib.PfConfig) == 4 * 4 + 8 + 8 * 8 + 5 * 4 + 4


def test_ctypes_layouts_match_the_header(tmp_path):
    """Every struct the Python binding mirrors has the C header's size and
    field offsets (compiled here with gcc against include/pf_gpu.h)."""
    import ctypes as C

    from paper_1412_4933_b200 import _lib

    structs = {"pf_config": _lib.PfConfig, "pf_halo_rows": _lib.PfHalo, "pf_peer_desc": _lib.PfPeerDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pf_gpu.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-std=c11", "-I", inc, "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} sizeof"]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname} {fname}"]) == getattr(py, fname).offset, (cname, fname)


@pytest.mark.parametrize("kw,msg", [
    (dict(width=100), "multiple of 16"),
    (dict(height=8), "multiple of 16"),
    (dict(rho=0.0), "rho"),
    (dict(rho=1.5), "rho"),
    (dict(tau0=0.0), "tau0"),
    (dict(q=-1.0), "q must"),
    (dict(d0=1.0), "d0"),
    (dict(alpha=-1.0), "alpha"),
    (dict(beta=-0.1), "beta"),
    (dict(sel_sigma=-0.1), "sel_sigma"),
    (dict(width=16, height=16, agents_per_side=200), "capacity"),
    (dict(steps=-1), "steps"),
    (dict(repeats=0), "repeats"),
])
def test_validate_rejects_like_reference(kw, msg):
    import paper_1412_4933_b200 as p

    with pytest.raises(p.ConfigError, match=msg):
        p.validate(p.ScenarioConfig(**kw))


def test_band_height():
    import paper_1412_4933_b200 as p

    assert p.band_height(1280, 480) == 3
    assert p.band_height(6720, 480) == 14
    assert p.band_height(0, 480) == 0
    assert p.band_height(25_000_000, 16384) == 1526


@pytest.mark.parametrize("kw", [
    dict(width=480, height=480, agents_per_side=1024, model="aco"),
    dict(width=480, height=480, agents_per_side=51200, model="lem"),
    dict(width=96, height=96, agents_per_side=900, model="lem", seed=11),
    dict(width=16, height=16, agents_per_side=128, model="aco"),
    dict(width=32, height=32, agents_per_side=0, model="aco"),
])
def test_new_environment_matches_oracle(kw):
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState, Scenario

    o = OracleState(Scenario(**kw))
    s = p.new_environment(to_config(kw), kw.get("seed", 42))
    assert hashes_of(s) == o.hashes()
    assert (s.agents == o.agents).all()
    # The second call is served from the library's placement cache.
    s2 = p.new_environment(to_config(kw), kw.get("seed", 42))
    assert hashes_of(s2) == o.hashes()
    assert (s2.agents == o.agents).all()


def test_placement_cache_keys_and_speed():
    """Placements are cached per (W, H, n, seed): a different seed or density
    is placed afresh (and still equals the oracle), and a repeated large
    placement (1.3M agents per side) comes back well under the cold time."""
    import time

    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState, Scenario

    kw = dict(width=96, height=96, agents_per_side=900, model="lem")
    for seed, n in ((5, 900), (6, 900), (5, 700)):
        k = dict(kw, seed=seed, agents_per_side=n)
        s = p.new_environment(to_config(k), seed)
        assert hashes_of(s) == OracleState(Scenario(**k)).hashes()
    big = p.ScenarioConfig(width=4096, height=1024, agents_per_side=1_300_000, model=p.Model.Lem)
    t0 = time.perf_counter()
    a = p.new_environment(big, 99)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    b = p.new_environment(big, 99)
    warm = time.perf_counter() - t0
    assert (a.index == b.index).all() and (a.agents == b.agents).all()
    assert warm < cold


def test_device_calls_fail_loudly_without_gpu():
    import torch

    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = p.ScenarioConfig(width=32, height=32, agents_per_side=16, model=p.Model.Lem)
    s = p.new_environment(cfg, 1)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 1))
    with pytest.raises(_lib.DeviceError):
        eng.step(s)
    with pytest.raises(_lib.DeviceError):
        p.Ensemble(cfg, replicas=2)


def test_placement_cache_concurrent_requests():
    """Several threads asking for the same (and different) placements at once
    get identical, correct results (one computation per key, shared)."""
    import threading

    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState, Scenario

    kw = dict(width=96, height=96, agents_per_side=1200, model="aco")
    out = {}

    def work(i):
        seed = 30 + (i % 3)
        out[i] = (seed, p.new_environment(to_config(dict(kw, seed=seed)), seed))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(9)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for seed in (30, 31, 32):
        want = OracleState(Scenario(**dict(kw, seed=seed))).hashes()
        for i, (sd, st) in out.items():
            if sd == seed:
                assert hashes_of(st) == want
