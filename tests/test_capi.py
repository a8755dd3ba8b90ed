"""The C-ABI library loads (no GPU needed), exports every symbol include/sdgr.h
declares, and the ctypes mirrors agree with the C struct layouts."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "sdgr.h"


def declared_functions():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|uint64_t|const char\*)\s+(sdgr_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_21633_b200 import _lib
    from paper_2506_21633_b200.csrc.build import build

    if not _lib.LIB_PATH.exists():
        build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n


def test_bindings_cover_header():
    from paper_2506_21633_b200 import _lib
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_functions())


def test_host_only_calls(lib):
    from paper_2506_21633_b200 import _lib
    assert lib.sdgr_version() == _lib.ABI_VERSION == 2
    assert lib.sdgr_status_string(1).decode() == "invalid parameter"
    assert lib.sdgr_workspace_bytes(1_000_000, 2_000_000) > 20 * 2**20
    assert isinstance(lib.sdgr_launch_count(), int)


def test_invalid_arguments_rejected_without_device(lib):
    from paper_2506_21633_b200 import _lib
    v = _lib.View()
    v.n_u = v.n_v = v.n_az = v.n_rg = 0        # invalid plane size
    sd, pd = _lib.SceneDesc(), _lib.ProjectionDesc()
    assert lib.sdgr_project(C.byref(sd), C.byref(v), C.byref(pd), None) == _lib.ERR_INVALID
    v.n_u = v.n_v = v.n_az = v.n_rg = 16
    v.cutoff = float("nan")
    assert lib.sdgr_project(C.byref(sd), C.byref(v), C.byref(pd), None) == _lib.ERR_INVALID


def test_struct_layouts_match_c(tmp_path):
    """Compile a tiny C program against sdgr.h and compare sizeof/offsetof."""
    from paper_2506_21633_b200 import _lib
    structs = {"sdgr_view": _lib.View, "sdgr_scene": _lib.SceneDesc, "sdgr_plane": _lib.Plane,
               "sdgr_projection": _lib.ProjectionDesc, "sdgr_tiles": _lib.TilesDesc,
               "sdgr_grads": _lib.GradsDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sdgr.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append('printf("sdgr_pair_rec %zu\\n", sizeof(sdgr_pair_rec));')
    lines.append("return 0;}")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", str(HEADER.parent), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(out[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(out[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"
    assert int(out["sdgr_pair_rec"]) == _lib.PAIR_REC_BYTES


def test_batch_entry_points_validate_without_device(lib):
    from paper_2506_21633_b200 import _lib
    mb = lib.sdgr_max_batch()
    assert mb == _lib.MAX_BATCH == 24
    # workspace sizing: 0 outside 1..max_batch, growing with the batch
    assert lib.sdgr_batch_workspace_bytes(1_000_000, 1_500_000, 0) == 0
    assert lib.sdgr_batch_workspace_bytes(1_000_000, 1_500_000, mb + 1) == 0
    w1 = lib.sdgr_batch_workspace_bytes(1_000_000, 1_500_000, 1)
    assert w1 == lib.sdgr_workspace_bytes(1_000_000, 1_500_000)
    assert lib.sdgr_batch_workspace_bytes(1_000_000, 1_500_000, mb) > 8 * w1
    sd = _lib.SceneDesc()
    views = (_lib.View * (mb + 1))()
    projs = (_lib.ProjectionDesc * (mb + 1))()
    tiles = (_lib.TilesDesc * (mb + 1))()
    ptrs = (C.c_void_p * (mb + 1))()
    for k in (0, mb + 1):   # batch size out of range
        assert lib.sdgr_project_batch(C.byref(sd), k, views, projs, None) == _lib.ERR_INVALID
        assert lib.sdgr_depth_order_batch(k, projs, ptrs, None, 0, None) == _lib.ERR_INVALID
        assert lib.sdgr_bin_batch(k, projs, views, 0, ptrs, ptrs, tiles, None, 0, None) == _lib.ERR_INVALID
        assert lib.sdgr_grad_geometry_batch(C.byref(sd), k, views, projs, tiles, ptrs, ptrs,
                                            C.byref(_lib.GradsDesc()), 1, None) == _lib.ERR_INVALID
    # NULL orders / unset views inside a valid batch size
    assert lib.sdgr_depth_order_batch(2, projs, None, None, 0, None) == _lib.ERR_INVALID
    assert lib.sdgr_bin_batch(2, projs, views, 0, None, ptrs, tiles, None, 0, None) == _lib.ERR_INVALID
    assert lib.sdgr_project_batch(C.byref(sd), 2, views, projs, None) == _lib.ERR_INVALID


def test_eval_entry_points_validate_without_device(lib):
    from paper_2506_21633_b200 import _lib
    lo = (C.c_double * 3)(0.0, 0.0, 0.0)
    dims = (C.c_int32 * 3)(4, 4, 4)
    bad_dims = (C.c_int32 * 3)(4096, 4096, 4096)   # > 2^24 cells
    assert lib.sdgr_grid_workspace_bytes(1000, 64) > 0
    one = C.c_void_p(1)
    assert lib.sdgr_nn_sqdist(one, 10, one, 10, lo, 0.0, dims, one, one, 1 << 30, None) == _lib.ERR_INVALID
    assert lib.sdgr_nn_sqdist(one, 10, one, 10, lo, 1.0, bad_dims, one, one, 1 << 30, None) == _lib.ERR_INVALID
    assert lib.sdgr_nn_sqdist(one, 10, one, 10, lo, 1.0, dims, one, one, 16, None) == _lib.ERR_CAPACITY
    # DBSCAN needs cells at least eps wide and min_pts >= 1
    assert lib.sdgr_dbscan(one, 10, lo, 0.5, dims, 1.0, 3, one, one, 1 << 30, None) == _lib.ERR_INVALID
    assert lib.sdgr_dbscan(one, 10, lo, 1.0, dims, 1.0, 0, one, one, 1 << 30, None) == _lib.ERR_INVALID
