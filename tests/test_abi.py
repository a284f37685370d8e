"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/*.h declares, and the headers compile as C and C++."""
import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "tqp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tqp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2209_04579_b200 import tqp
    lib = tqp.lib
    syms = declared_symbols()
    assert len(syms) >= 70
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.tqp_abi_version() == 1


def test_nm_exports_match_header():
    lib = ROOT / "paper_2209_04579_b200" / "libtqp_b200.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.split()[-1].startswith("tqp_")}
    assert set(declared_symbols()) <= exported


@pytest.mark.parametrize("compiler,std", [("gcc", "-std=c99"), ("g++", "-std=c++17")])
def test_headers_compile(tmp_path, compiler, std):
    src = tmp_path / ("t.c" if compiler == "gcc" else "t.cpp")
    src.write_text('#include "tqp_b200.h"\n#include "tqp_gen.h"\nint main(void){return tqp_gen_dummy();}\n'
                   .replace("tqp_gen_dummy()", "(int)tqp_lineitem_rows(0.001) == 6000 ? 0 : 1"))
    exe = tmp_path / "t"
    subprocess.run([compiler, std, "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def test_status_struct_layout():
    import ctypes
    from paper_2209_04579_b200 import tqp
    assert ctypes.sizeof(tqp.Status) == 4 + 4 + 8 + 1024  # int, pad, int64, msg


def test_plan_builder_without_gpu():
    """Plans are host objects: building one from a committed lowered plan
    needs no device."""
    from paper_2209_04579_b200 import tqp
    p = tqp.Plan.from_file(ROOT / "paper_2209_04579_b200" / "plans" / "q6.opplan.json")
    assert p.h


def test_nvrtc_bound_from_build_toolkit():
    """The specialised kernels compile with the toolkit the library was built
    with even when torch (bundling an older libnvrtc.so.12) is imported
    first: kernel speed must not depend on import order."""
    import subprocess
    import sys
    code = ("import torch, sys; sys.path.insert(0, %r); "
            "from paper_2209_04579_b200 import tqp; print(tqp.nvrtc_version())" % str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    nvcc = subprocess.run(["/usr/local/cuda/bin/nvcc", "--version"], capture_output=True, text=True).stdout
    rel = nvcc.split("release ")[1].split(",")[0]
    major, minor = (int(x) for x in rel.split("."))
    assert int(out.stdout.strip()) == major * 1000 + minor * 10


def test_plan_builder_rejects_bad_arguments():
    """The plan builder validates what crosses the C ABI (no step yet, bad
    constant dtype, null constant data) instead of dereferencing it."""
    import ctypes as C
    from paper_2209_04579_b200 import tqp
    st = tqp.Status()
    h = tqp.lib.tqp_plan_create(4, C.byref(st))
    assert h
    slots = (C.c_int * 1)(0)
    assert tqp.lib.tqp_plan_set_step_outputs(h, slots, 1, C.byref(st)) != 0
    assert b"before tqp_plan_begin_step" in st.msg
    assert tqp.lib.tqp_plan_begin_step(h, b"s#0", b"scan", C.byref(st)) == 0
    d = tqp.InstrDesc()
    d.op = b"const"
    d.num_inputs = 0
    d.output = 0
    d.const_dtype = 9
    d.const_rows = d.const_cols = 1
    assert tqp.lib.tqp_plan_add_instr(h, C.byref(d), C.byref(st)) != 0
    assert b"bad constant dtype" in st.msg
    d.const_dtype = tqp.I64
    d.const_data = None
    assert tqp.lib.tqp_plan_add_instr(h, C.byref(d), C.byref(st)) != 0
    assert b"null constant data" in st.msg
    tqp.lib.tqp_plan_free(h)
