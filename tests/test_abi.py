"""The C ABI library loads and exports exactly what include/*.h declares
(no compute calls: runs on CPU-only hosts)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2311_15393_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kronprec_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    names = declared()
    assert names, "no declarations parsed"
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == names


def test_symbols_are_extern_c():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for n in declared():
        assert n in exported, n


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu\\n", sizeof(kp_format), sizeof(kp_solver_options),
         sizeof(kp_history), sizeof(kp_param_choice));
  printf("%zu %zu %zu\\n", offsetof(kp_solver_options, x_true),
         offsetof(kp_history, abort_reason), offsetof(kp_param_choice, grid_index));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([cc, str(src), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [C.sizeof(_lib.kp_format), C.sizeof(_lib.kp_solver_options),
                     C.sizeof(_lib.kp_history), C.sizeof(_lib.kp_param_choice)]
    assert offs == [_lib.kp_solver_options.x_true.offset, _lib.kp_history.abort_reason.offset,
                    _lib.kp_param_choice.grid_index.offset]


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    """Without a device every entry point reports KP_ERR_CUDA — there is no
    CPU fallback behind the ABI."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    st = _lib.lib().kp_init(0)
    assert st == _lib.KP_ERR_CUDA
    assert "CPU fallback" in _lib.lib().kp_last_error().decode() or st != 0
