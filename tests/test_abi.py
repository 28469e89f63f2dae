"""CPU-side checks of the boundary: libsim.so builds, loads and exports every entry point
include/sim.h declares; the ctypes structs match the C layout; host-only validation works
without a GPU; without a GPU the library refuses to run (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sim.h")

sim = pytest.importorskip("paper_2302_09334_b200.sim")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^SIM_API\s+[\w\s\*]+?\b(sim_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = sim.lib()
    decl = declared_functions()
    assert len(decl) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only", L._name]).decode()
    exported = set(re.findall(r" T (sim_\w+)", out))
    for f in decl:
        assert f in exported, f
        assert hasattr(L, f)
    assert set(decl) == set(sim.EXPORTED)


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include "sim.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(sim_config), sizeof(sim_state),'
                    ' sizeof(sim_step_record), sizeof(sim_totals), sizeof(sim_state_sizes_t),'
                    ' sizeof(sim_step_timing), offsetof(sim_config, cuda_stream)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", f"-I{os.path.join(ROOT, 'include')}", str(prog), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(sim.SimConfig), ctypes.sizeof(sim.SimState), sim.RECORD_DTYPE.itemsize,
            ctypes.sizeof(sim.SimTotals), ctypes.sizeof(sim.SimStateSizes), ctypes.sizeof(sim.SimStepTiming),
            sim.SimConfig.cuda_stream.offset]
    assert got == want
    assert sim.lib().sim_kernels_per_step() == sim.NUM_KERNELS


def test_host_validation_and_sizes():
    for wc in (workloads.tiny(), workloads.paper_scale(), workloads.regrowth_micro(8192, 16384),
               workloads.large_world(), workloads.ensemble()):
        sim.validate(wc)
    sz = sim.state_sizes(workloads.paper_scale())
    assert sz["params"] == 16933 and sz["inputs"] == 98 and sz["cells"] == 80000
    assert sz["device_bytes"] > 8192 * 16933 * 4
    for kw, field in [(dict(rows=1), "rows"), (dict(cols=42), "cols"), (dict(hidden=12), "hidden"),
                      (dict(obs_radius=4), "obs_radius"), (dict(n_initial=33), "n_initial"),
                      (dict(regrow_r2=9), "regrow_r2"), (dict(f_value=(0, 2.0, 0, 0)), "f_value"),
                      (dict(f_class_min_k=(0, 3, 1, 5)), "f_class_min_k"), (dict(n_actions=4), "n_actions")]:
        with pytest.raises(sim.SimError) as ei:
            sim.validate(workloads.tiny().replace(**kw))
        assert ei.value.status == sim.SIM_E_INVALID and field in str(ei.value)
    # device index arithmetic is 32-bit: the bit-plane words of all worlds must stay < 2^31
    big = workloads.regrowth_micro(8192, 16384)
    sim.validate(big.replace(seeds=tuple(range(127))))
    with pytest.raises(sim.SimError) as ei:
        sim.validate(big.replace(seeds=tuple(range(512))))
    assert ei.value.status == sim.SIM_E_INVALID and "n_worlds" in str(ei.value)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(sim.SimError) as ei:
        sim.World(workloads.tiny())
    assert ei.value.status == sim.SIM_E_CUDA


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2302_09334_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                for needle in ("import oracle", "from oracle", "liboracle", "orc_"):
                    assert needle not in src, f"{f} references the oracle ({needle})"


def test_network1_validation_and_sizes():
    """Network 1 (the paper's CNN-LSTM): 2445 parameters per slot, the
    architecture fixes the window (r = 7) and the LSTM (4), banded mode is refused."""
    wc = workloads.paper_world_cnn()
    sim.validate(wc)
    sz = sim.state_sizes(wc)
    assert sz["params"] == 2445 and sz["hidden"] == 4
    for kw, field in [(dict(obs_radius=3), "obs_radius"), (dict(hidden=8), "hidden"), (dict(network=2), "network")]:
        with pytest.raises(sim.SimError) as ei:
            sim.validate(wc.replace(**kw))
        assert ei.value.status == sim.SIM_E_INVALID and field in str(ei.value)
    with pytest.raises(sim.SimError) as ei:
        sim.validate(wc, bands=dict(n_bands=2))
    assert ei.value.status == sim.SIM_E_INVALID and "n_bands" in str(ei.value)
