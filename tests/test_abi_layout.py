"""The ctypes mirrors in paper_1809_05018_b200/_native.py match the structs
include/dpmrf_cuda.h declares: same field names, order, offsets and sizes
(gcc compiles a probe of the header; no GPU, no library load)."""
import ctypes as ct
import os
import shutil
import subprocess

import pytest

from paper_1809_05018_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MIRRORS = {
    "dpmrf_optimizer_config": N.CConfig,
    "dpmrf_run_options": N.CRunOptions,
    "dpmrf_run_stats": N.CRunStats,
    "dpmrf_phantom_spec": N.CPhantomSpec,
    "dpmrf_group_info": N.CGroupInfo,
}


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    d = tmp_path_factory.mktemp("abi")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dpmrf_cuda.h"',
             "int main(void) {"]
    for name, cls in MIRRORS.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name} {f} %zu %zu\\n", offsetof({name}, {f}), '
                         f'sizeof((({name}*)0)->{f}));')
    lines += ["  return 0;", "}"]
    src = d / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    exe = d / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    layout = {}
    for line in out.splitlines():
        parts = line.split()
        if parts[1] == "size":
            layout[(parts[0], None)] = int(parts[2])
        else:
            layout[(parts[0], parts[1])] = (int(parts[2]), int(parts[3]))
    return layout


@pytest.mark.parametrize("name", sorted(MIRRORS))
def test_struct_mirror_matches_header(c_layout, name):
    cls = MIRRORS[name]
    assert ct.sizeof(cls) == c_layout[(name, None)], name
    for f, ctype in cls._fields_:
        off, size = c_layout[(name, f)]
        assert getattr(cls, f).offset == off, (name, f)
        assert ct.sizeof(ctype) == size, (name, f)


def test_run_stats_fields_cover_header():
    """Every member the header declares has a mirror field (a member added
    to the header and not to _native.py would shift nothing but would be
    invisible to Python; this keeps the two lists in step)."""
    import re
    hdr = open(os.path.join(ROOT, "include", "dpmrf_cuda.h")).read()
    body = re.search(r"typedef struct dpmrf_run_stats \{(.*?)\} dpmrf_run_stats;", hdr, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b(\w+)\s*;", body)
    assert names == [f for f, _ in N.CRunStats._fields_]
