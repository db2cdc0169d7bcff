"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/menndl_sm100.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

from paper_1909_12291_b200 import build, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "menndl_sm100.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(ce_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_abi():
    names = declared()
    for must in ("ce_net_create", "ce_train", "ce_predict", "ce_latency", "ce_conv_fwd", "ce_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(native.EXPORTED_SYMBOLS) <= set(declared())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tensor_core_kernels_present():
    sass = subprocess.run(["cuobjdump", "-sass", build.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass             # tcgen05.ld
    assert "LDGSTS" in sass           # cp.async gathers
    assert "UTCHMMA.2CTA" in sass     # tcgen05.mma.cta_group::2 (CTA-pair conv forward)
    assert "UTMALDG.4D.IM2COL.2CTA" in sass  # pair im2col TMA completing on the leader's barrier


def test_error_path_without_gpu():
    lib = native.load()
    assert lib.ce_version() == 1
    # a bad descriptor fails with CE_EINVAL and a message, before touching the device
    status = lib.ce_net_create(None, 0, 0, None)
    assert status == 1
    assert b"descriptor" in lib.ce_last_error()
