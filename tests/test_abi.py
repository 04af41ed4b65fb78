"""The C-ABI library: loads without a GPU, exports every symbol include/hm.h declares, and
reports errors through status codes (GPU part marked)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hm.h")).read()
    return sorted(set(re.findall(r"\b(hm_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_all_symbols():
    from paper_1806_11558_b200 import hm
    L = hm.lib()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), f"libhm.so does not export {n}"


def test_mesh_struct_matches_header():
    # the ctypes hm_mesh of the binding has the header's fields, in order, with its C layout
    from paper_1806_11558_b200 import hm
    src = open(os.path.join(ROOT, "include", "hm.h")).read()
    body = re.search(r"typedef struct \{([^}]*)\} hm_mesh;", src).group(1)
    fields = re.findall(r"\b(\w+)\s*;", body)
    assert fields == [f[0] for f in hm._Mesh._fields_]
    assert fields[-1] == "panel_vertices"
    assert ctypes.sizeof(hm._Mesh) == 40 and hm._Mesh.panel_vertices.offset == 36   # x86-64 C layout


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_1806_11558_b200", "libhm.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_quadrature_table_without_gpu():
    from paper_1806_11558_b200 import hm
    x, w = hm.hm_quadrature_table(6)
    assert abs(w.sum() - 1.0) < 1e-15 and (np.diff(x) > 0).all()
    with pytest.raises(hm.HMError):
        hm.hm_quadrature_table(0)


def test_no_oracle_in_product_path():
    pkg = os.path.join(ROOT, "paper_1806_11558_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle's", "").lower() or f == "gen_gauss.py", f


@pytest.mark.gpu
def test_error_codes_and_state_machine():
    import torch
    from inputs.meshes import icosphere
    from paper_1806_11558_b200 import HMatrix, HMError
    H = HMatrix(device=0)
    x = torch.zeros(10, dtype=torch.float64, device="cuda")
    with pytest.raises(HMError) as e:
        H.setup(1e-6)
    assert e.value.status == 2                                 # HM_ERR_STATE
    V, T = icosphere(2)
    with pytest.raises(HMError) as e:
        H.build_tree(V, T, leaf_size=0)
    assert e.value.status == 1
    with pytest.raises(HMError):
        H.build_tree(V, T, eta=-1.0)
    bad = T.copy(); bad[0, 0] = 10 ** 6
    with pytest.raises(HMError) as e:
        H.build_tree(V, bad)
    assert e.value.status == 1 and "out of range" in str(e.value)
    deg = T.copy(); deg[0, 1] = deg[0, 0]
    with pytest.raises(HMError):
        H.build_tree(V, deg)
    H.build_tree(V, T)
    with pytest.raises(HMError) as e:
        H.matvec(torch.zeros(320, dtype=torch.float64, device="cuda"))
    assert e.value.status == 2
    with pytest.raises(HMError):
        H.setup(-1e-6)                                         # eps_aca = 0 is the fixed-rank mode
    with pytest.raises(HMError):
        H.setup(float("nan"))
    with pytest.raises(HMError):
        H.set_option("nope", 1)
    with pytest.raises(HMError):
        H.set_option("k_max", 0)
    # peer-memory collectives: single-rank contexts cannot export, solve_comm 1 needs an import
    from paper_1806_11558_b200 import hm
    with pytest.raises(HMError) as e:
        hm.hm_p2p_export(H.ctx, 320)
    assert e.value.status == 2
    with pytest.raises(HMError) as e:
        H.set_option("solve_comm", 1)
    assert e.value.status == 2
    assert H.get_option("solve_comm") == 0
    H.setup(1e-6)
    st = H.stats()
    assert st["N"] == 320 and st["adm_leaves"] == 0 and st["dense_leaves"] == 256
    with pytest.raises(HMError):
        H.solve(torch.ones(320, dtype=torch.float64, device="cuda"), tol=0.0)
    # quadrilateral meshes: panel_vertices 4 accepted, others rejected
    from inputs.meshes import cube
    Vq, Qq = cube(2)
    H3 = HMatrix(device=0)
    H3.build_tree(Vq, Qq)
    assert H3.stats()["N"] == 96
    with pytest.raises(HMError):
        H3.build_tree(Vq, np.ascontiguousarray(np.concatenate([Qq, Qq[:, :1]], axis=1)))   # 5 vertices
    # device-resident mesh input gives the same tree
    H2 = HMatrix(device=0)
    H2.build_tree(torch.from_numpy(V).cuda(), torch.from_numpy(T).cuda())
    assert np.array_equal(H2.perm(), H.perm())
