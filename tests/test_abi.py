"""C-ABI library: loads without a GPU and exports every symbol the header declares."""
import ctypes
import os
import re

import pytest

from paper_2506_01120_b200 import liecl, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "liecl_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(liecl_b200_\w+)\s*\(", text)))


def test_header_matches_binding_list():
    assert header_functions() == sorted(native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = native.load()
    missing = [s for s in header_functions() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.liecl_b200_abi_version() == 1


def test_library_is_sm100a():
    # the fatbin must carry sm_100a SASS (cuobjdump is in the image)
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kernels_use_fp64_tensor_pipe():
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # mma.sync f64 -> DMMA.8x8x4 (no tcgen05 kind::f64 exists)


def test_library_is_self_contained():
    """Every kernel is this repository's: no CUB / cuBLAS / cuSOLVER kernels in
    the fatbin and no CUDA math library among the dynamic dependencies (the
    runtime is linked statically, NCCL is resolved with dlopen)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump") or not shutil.which("readelf"):
        pytest.skip("cuobjdump / readelf missing")
    names = subprocess.run(["cuobjdump", "--dump-elf-symbols", native.LIB_PATH], capture_output=True, text=True).stdout
    for lib in ("cub", "cublas", "cusolver", "thrust"):
        assert f"N{len(lib)}{lib}" not in names and f"{lib}::" not in names, lib
    needed = subprocess.run(["readelf", "-d", native.LIB_PATH], capture_output=True, text=True).stdout
    for lib in ("cublas", "cusolver", "cusparse", "nccl", "cudart"):
        assert f"lib{lib}" not in needed, lib


def test_method_strings_roundtrip():
    for m in liecl.Method:
        assert liecl.method_from_string(liecl.to_string(m)) == m
    with pytest.raises(liecl.InvalidInputError):
        liecl.method_from_string("gram")


def test_validation_errors_before_device():
    with pytest.raises(liecl.InvalidInputError):
        liecl.run_closure([], liecl.Method.orthonorm_dimonly)
    import numpy as np
    a = liecl.DenseOperator(np.eye(2))
    b = liecl.DenseOperator(np.eye(4))
    with pytest.raises(liecl.InvalidInputError):
        liecl.run_closure([a, b], liecl.Method.orthonorm_dimonly)
    with pytest.raises(liecl.InvalidInputError):  # close_standard vectorizes dense operators only
        liecl.close_standard([liecl.PauliSum.single(liecl.PauliString(1, 0, 1), 1.0)])


def test_pair_index_roundtrip():
    # cursor order (R:src/closure.cpp:412-417): g = l(l-1)/2 + m; mirror of common.cuh
    def pair_from_index(g):
        import math
        l = int((1 + math.sqrt(1 + 8 * g)) / 2)
        while l * (l - 1) // 2 > g:
            l -= 1
        while (l + 1) * l // 2 <= g:
            l += 1
        return l, g - l * (l - 1) // 2
    g = 0
    for l in range(1, 300):
        for m in range(l):
            assert pair_from_index(g) == (l, m)
            g += 1
    assert pair_from_index(8382464) == (4094, 4093)


def test_shard_range_partitions_every_operator():
    # liecl_b200_shard_range makes no CUDA call; the host mirror must agree
    from paper_2506_01120_b200.distributed import shard_bounds
    for d in (1, 2, 3, 16, 256):
        for P in range(1, 9):
            if P > d * d:
                continue
            got = [liecl.shard_range(d, P, r) for r in range(P)]
            assert got == [shard_bounds(d, P, r) for r in range(P)]
            assert got[0][0] == 0 and got[-1][1] == d * d
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
    with pytest.raises(liecl.InvalidInputError):
        liecl.shard_range(2, 5, 0)


def test_no_device_fails_loudly_without_deadlock():
    # no GPU here: the product path must raise (never fall back to the CPU)
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import numpy as np
    with pytest.raises((native.NativeUnavailable, liecl.Error)):
        liecl.run_closure([liecl.DenseOperator(np.eye(2))], liecl.Method.standard_rank)


def test_header_is_plain_c_and_links():
    # the C-ABI is C: a C11 translation unit includes the header and links the library
    import shutil
    import subprocess
    import tempfile
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("gcc missing")
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "c_abi_demo")
        r = subprocess.run([gcc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                            os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", os.path.dirname(native.LIB_PATH),
                            "-lliecl_b200", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
