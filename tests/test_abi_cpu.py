"""Host-side checks that need no GPU: the C-ABI library loads, exports every symbol that
include/im.h declares, and rejects bad call order / arguments before touching the device."""
import os
import re
import subprocess

import pytest

import paper_2105_04023_b200 as im

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "im.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(im_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("im_load_csr", "im_build_sketches", "im_estimate", "im_select_seeds"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", im.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (im_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(declared_symbols()) == set(im.SIGNATURES), "binding and header disagree"


def test_library_loads_and_binds():
    L = im.lib()
    for name in declared_symbols():
        assert hasattr(L, name)
    assert im.im_version() == 103


def test_call_order_errors_without_gpu():
    im.im_free()
    with pytest.raises(im.IMError) as e:
        im.im_build_sketches(64, 1)
    assert e.value.code == im.IM_ESTATE
    with pytest.raises(im.IMError) as e:
        im.im_estimate(4)
    assert e.value.code == im.IM_ESTATE
    with pytest.raises(im.IMError) as e:
        im.im_select_seeds(1, 0.05)
    assert e.value.code == im.IM_ESTATE


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2105_04023_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in txt and "liboracle" not in txt and "from oracle" not in txt, f
    out = subprocess.run(["ldd", im.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out


def test_binding_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of im_stats / im_step have the C sizes and field offsets (gcc on include/im.h)."""
    import ctypes

    fields = {"im_stats": im.im_stats, "im_step": im.im_step}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "im.h"', "int main(void) {"]
    for cname, cls in fields.items():
        src.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            src.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, f, v = line.split()
        cls = fields[cname]
        want = ctypes.sizeof(cls) if f == "size" else getattr(cls, f).offset
        assert int(v) == want, (cname, f, v, want)


def test_c_program_consumes_the_header(tmp_path):
    """A plain C program compiled against include/im.h and linked to libim_b200.so: the
    declarations, error codes and call-order checks work from C without Python or a GPU."""
    src = r'''
#include <stdio.h>
#include <string.h>
#include "im.h"
int main(void) {
    im_stats st;
    int32_t seeds[1]; double scores[1];
    if (im_version() != 103) return 1;
    im_free();
    if (im_build_sketches(64, 1) != IM_ESTATE) return 2;
    if (strlen(im_last_error()) == 0) return 3;
    if (im_select_seeds(1, 0.05, seeds, scores) != IM_ESTATE) return 4;
    if (im_get_stats(NULL) != IM_EINVAL) return 5;
    if (im_get_stats(&st) != IM_OK || st.n != 0 || st.J != 0) return 6;
    if (im_set_policy(-1.0, 0.0, 0.0) != IM_EINVAL) return 7;
    if (im_get_step_log(NULL, -1) != IM_EINVAL) return 8;
    printf("ok %s\n", im_last_error());
    return 0;
}
'''
    c = tmp_path / "consumer.c"
    c.write_text(src)
    exe = tmp_path / "consumer"
    libdir = os.path.dirname(im.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe),
                    f"-L{libdir}", "-l:libim_b200.so", f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.startswith("ok"), (r.returncode, r.stdout, r.stderr)
