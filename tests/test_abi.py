"""The C-ABI library loads and exports every symbol include/mpsf.h declares; struct
layouts and constants agree between the header, ctypes, numpy and constants.py.
No compute calls (no GPU needed)."""

import ctypes as C
import os
import re

from paper_2605_26461_b200 import _lib
from paper_2605_26461_b200 import constants as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = open(os.path.join(ROOT, "include", "mpsf.h")).read()


def declared_functions():
    return set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(mpsf_\w+)\(", HEADER, re.M))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)
    for n in names:
        assert hasattr(lib, n), n


def test_version_and_strerror_without_gpu():
    lib = _lib.load()
    assert lib.mpsf_version() == 1
    for code in range(0, -11, -1):
        assert lib.mpsf_strerror(code)


def test_struct_layouts_match_numpy_and_header():
    assert _lib.sizes_match_numpy()
    assert C.sizeof(_lib.Params) == 32 and C.sizeof(_lib.Summary) == 40


def header_define(name):
    m = re.search(rf"#define {name} \(?(-?0?x?[0-9a-fA-F]+)u?\)?", HEADER)
    return int(m.group(1), 0)


def test_constants_agree_with_header():
    assert header_define("MPSF_PF_ISOLATION") == K.PF_ISOLATION
    assert header_define("MPSF_WF_GR_DEAD") == K.WF_GR_DEAD
    from paper_2605_26461_b200 import errors as E
    for name, val in (("MPSF_E_NO_CHANNEL", E.E_NO_CHANNEL), ("MPSF_E_WORLD", E.E_WORLD),
                      ("MPSF_E_OVERFLOW", E.E_OVERFLOW), ("MPSF_E_TOO_LARGE", E.E_TOO_LARGE)):
        assert header_define(name) == val


def test_library_is_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        return
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout


def test_plain_c_consumer_links_and_runs(tmp_path):
    """The boundary is a C ABI: a C program compiled against include/mpsf.h links libmpsf.so
    and calls the host-only entry points (version, strerror, trace rendering)."""
    import subprocess
    lib = _lib.LIB_PATH
    exe = str(tmp_path / "abi_smoke")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_smoke.c"),
                    lib, "-Wl,-rpath," + os.path.dirname(lib), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stderr)
    lines = out.stdout.splitlines()
    assert lines[0] == "t=42 who=c1.sm kind=fault_raised scenario=mmu.oob.sm va=4096 access=write engine=sm"
    assert "t=42 who=uvm kind=isolate_begin mechanism=M1 scenario=mmu.oob.sm pid=c1 latency_us=131" in lines
    assert "t=42 who=uvm kind=parse_fatal scenario=parse.channel_state" in lines
