"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol that
include/dr.h declares, its default parameters are the paper's values, its struct layout matches
the binding, host-side validation errors, and the oracle/product separation."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT
from workload import presets


@pytest.fixture(scope="module")
def lib():
    from paper_1906_11633_b200 import dr
    return dr.load()


def _declared_symbols():
    """Every function declared in include/*.h (dr.h and dr_vision.h)."""
    import glob
    src = ""
    for h in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))):
        with open(h) as f:
            src += f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dr_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = _declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"libdr.so does not export {s}"


def test_sass_is_sm100a():
    from paper_1906_11633_b200 import build
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_params_are_the_paper_values(lib):
    from paper_1906_11633_b200 import dr
    p = dr.dr_params_default()
    assert p.abi_version == dr.ABI_VERSION
    assert p.struct_size == C.sizeof(dr.DrParams)        # layout of binding == layout of dr.h
    assert p.layer_mask == dr.ALL
    P = presets.PAPER
    for name, _ in dr.DrParams._fields_:
        if name in P and name not in ("phys", "delta_cal_neg", "delta_cal_pos", "layer_mask"):
            assert getattr(p, name) == pytest.approx(P[name], rel=1e-15), name
    for j in range(20):
        assert p.delta_cal_neg[j] == pytest.approx(P["delta_cal_neg"][j])
        assert p.delta_cal_pos[j] == pytest.approx(P["delta_cal_pos"][j])
    for i, (k, a, b, base) in enumerate(P["phys"]):
        assert (p.phys[i].kind, p.phys[i].a, p.phys[i].b) == (k, pytest.approx(a), pytest.approx(b))
        assert p.phys[i].base == pytest.approx(base)
    assert (p.n_act, p.n_tips, p.n_substeps) == (20, 5, 10)


def test_state_struct_is_168_words():
    from paper_1906_11633_b200 import dr
    assert C.sizeof(dr.DrEnvState) == 168 * 4


@pytest.mark.parametrize("field,value,needle", [
    ("act_sigma_uadd", -0.1, "act_sigma_uadd"),
    ("delay_prob", 1.5, "delay_prob"),
    ("force_decay_per_step", 0.0, "force_decay_per_step"),
    ("force_p_lo", 0.5, "force_p_lo"),       # lo > hi
    ("occl_dist", -1.0, "occl_dist"),
    ("dt_base", 0.0, "dt_base"),
    ("dropout_hold_steps", 16, "dropout_hold_steps"),
    ("n_phys", 0, "n_phys"),
    ("abi_version", 99, "abi_version"),
    ("struct_size", 8, "struct_size"),
    ("layer_mask", 0x400, "layer_mask"),
    ("backlash_eps", 1e-3, "backlash_eps"),   # the kernels' gate identity needs eps < 2^-24
])
def test_validation_errors_name_the_field(lib, field, value, needle):
    from paper_1906_11633_b200 import dr
    p = dr.params_from_preset(presets.preset())
    setattr(p, field, value)
    rc = lib.dr_init(C.byref(p), 16, 1)
    assert rc == -1, (rc, dr.dr_last_error())
    assert needle in dr.dr_last_error()


def test_validation_calibrated_delta_and_mass(lib):
    from paper_1906_11633_b200 import dr
    p = dr.params_from_preset(presets.preset())
    p.delta_cal_neg[3] = -0.5
    assert lib.dr_init(C.byref(p), 16, 1) == -1 and "delta_cal_neg[3]" in dr.dr_last_error()
    p = dr.params_from_preset(presets.preset())
    p.phys[0].base = 0.0
    assert lib.dr_init(C.byref(p), 16, 1) == -1 and "mass" in dr.dr_last_error()
    p = dr.params_from_preset(presets.preset())
    assert lib.dr_init(C.byref(p), 0, 1) == -1 and "n_env" in dr.dr_last_error()
    p = dr.params_from_preset(presets.preset(), env_offset=10, n_env_global=12)
    assert lib.dr_init(C.byref(p), 4, 1) == -1 and "env_offset" in dr.dr_last_error()
    p = dr.params_from_preset(presets.preset())
    p.n_act = 16
    assert lib.dr_init(C.byref(p), 4, 1) == -6


def test_calls_before_init(lib):
    assert lib.dr_step(None, None, None, None, None, None) == -2
    assert lib.dr_reset(None) == -2
    assert lib.dr_finalize() == -2
    assert lib.dr_step_index() == 0
    assert lib.dr_phys_params() is None


def test_workspace_bytes(lib):
    from paper_1906_11633_b200 import dr
    p = dr.params_from_preset(presets.preset())
    small = dr.dr_workspace_bytes(p, 4)
    big = dr.dr_workspace_bytes(p, 1 << 20)
    assert 0 < small < big
    # SoA record + state planes + phys rows dominate: (89 + 60) words + 256 phys per env
    assert big >= (1 << 20) * 4 * (89 + 60 + 256)
    assert dr.dr_workspace_bytes(p, 0) == 0


def _code_refs(path):
    """#include targets and imported modules of a source file."""
    src = open(path).read()
    inc = re.findall(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', src, flags=re.M)
    imp = re.findall(r'^\s*(?:from|import)\s+([\w.]+)', src, flags=re.M)
    return inc, imp


def test_oracle_and_product_share_no_code():
    """The oracle (oracle/) and the CUDA path (include/, paper_1906_11633_b200/) must not include,
    import or link each other (they share only the workload input generators)."""
    for d in ("include", "paper_1906_11633_b200"):
        for dp, _, fs in os.walk(os.path.join(ROOT, d)):
            for f in fs:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                    inc, imp = _code_refs(os.path.join(dp, f))
                    assert not any("oracle" in x for x in inc + imp), (f, inc, imp)
    for dp, _, fs in os.walk(os.path.join(ROOT, "oracle")):
        for f in fs:
            if f.endswith((".py", ".c", ".h")):
                inc, imp = _code_refs(os.path.join(dp, f))
                assert all(x in ("oracle.h", "stdint.h", "math.h", "stdlib.h", "string.h") for x in inc), (f, inc)
                assert not any(x.startswith(("paper_1906_11633_b200", "workload")) for x in imp), (f, imp)
