"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/simplexmg_b200.h declares (no compute calls on the CPU box)."""

import ctypes
import subprocess

from paper_2402_12947_b200 import _lib, build_lib


def test_library_builds_and_loads():
    path = build_lib.build()
    lib = ctypes.CDLL(path)
    assert lib is not None


def test_every_header_symbol_is_exported_and_bound():
    declared = set(_lib.header_symbols())
    assert declared, "no declarations parsed from the header"
    assert declared == set(_lib.PROTOTYPES), declared ^ set(_lib.PROTOTYPES)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_error_string():
    lib = _lib.load()
    assert lib.smg_abi_version() == 1
    assert isinstance(lib.smg_last_error(), bytes)


def test_sass_is_sm100a_and_parity_kernels_have_no_fma():
    """SpMV/residual/restriction/prolong kernels must not contract to DFMA
    (bitwise parity with scipy's separately rounded multiply-add)."""
    out = subprocess.run(["cuobjdump", "-sass", build_lib.LIB], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    funcs = {}
    current = None
    for line in out.splitlines():
        if "Function : " in line:
            current = line.split("Function : ")[1].strip()
            funcs[current] = []
        elif current:
            funcs[current].append(line)
    # Epi 0 = spmv, 1 = residual, 5 = add-to (prolong): pure multiply/add
    for epi in ("0", "1", "5"):
        names = [f for f in funcs if f.startswith(f"_ZN3smg15csr_tile_kernelILNS_3EpiE{epi}E")]
        assert names, f"csr_tile_kernel<{epi}> missing"
        sell = [f for f in funcs if f.startswith(f"_ZN3smg11sell_kernelILNS_3EpiE{epi}E")]
        assert sell, f"sell_kernel<{epi}> missing"
        stage = [f for f in funcs if f.startswith(f"_ZN3smg16csr_stage_kernelILNS_3EpiE{epi}E")]
        assert stage, f"csr_stage_kernel<{epi}> missing"
        for name in names + sell + stage:  # every layout, with and without the L2 prefetch
            body = "\n".join(funcs[name])
            assert "DFMA" not in body, f"{name} contains DFMA"
            assert "DMUL" in body and "DADD" in body


def test_sass_shows_bulk_copies_and_l2_prefetch():
    """Evidence of the Blackwell data-movement paths: 1D TMA bulk copies into
    shared memory with mbarrier completion (patch factors) and bulk L2
    prefetches (SpMV tiles)."""
    out = subprocess.run(["cuobjdump", "-sass", build_lib.LIB], capture_output=True, text=True,
                         check=True).stdout
    assert "UBLKCP" in out          # cp.async.bulk.shared::cluster.global
    assert "UBLKPF" in out          # cp.async.bulk.prefetch.L2
    assert "SYNCS.PHASECHK" in out  # mbarrier try_wait
