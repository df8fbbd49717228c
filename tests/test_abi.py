"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads,
exports every symbol include/mel.h declares, and the product package has no
route to the oracle (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mel.h")
PKG = os.path.join(ROOT, "paper_2309_16743_b200")


@pytest.fixture(scope="module")
def lib():
    from paper_2309_16743_b200 import build, mel
    build.build()
    return mel.load_library()


def declared_functions(header=HEADER):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:int|void|uint32_t|uint64_t|const char\*)\s+\**(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


INGEST_HEADER = os.path.join(ROOT, "include", "mel_ingest.h")


def _exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(PKG, so)], capture_output=True, text=True).stdout
    return set(l.split()[-1] for l in out.splitlines() if " T " in l)


def test_ingest_header_exported_by_both_libraries(lib):
    """include/mel_ingest.h: the server side lives in libmel.so, the clients load
    libmel_ingest.so, which must not depend on CUDA (clients run on host cores)."""
    from paper_2309_16743_b200 import mel
    names = declared_functions(INGEST_HEADER)
    assert sorted(mel.INGEST_EXPORTS) == names
    for so in ("libmel.so", "libmel_ingest.so"):
        missing = [n for n in names if n not in _exported(so)]
        assert not missing, (so, missing)
    deps = subprocess.run(["ldd", os.path.join(PKG, "libmel_ingest.so")], capture_output=True, text=True).stdout
    assert "cuda" not in deps and "nccl" not in deps
    mel.load_ingest_library()


def test_header_declares_the_paper_calls():
    names = declared_functions()
    for n in ("reservoir_put", "reservoir_close", "reservoir_sample_batch", "surrogate_step", "surrogate_eval"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(PKG, "libmel.so")], capture_output=True,
                         text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    from paper_2309_16743_b200 import mel
    assert sorted(mel.EXPORTS) == declared_functions()


def test_config_default_without_gpu(lib):
    from paper_2309_16743_b200 import mel
    c = mel._Config()
    assert lib.mel_config_default(ctypes.byref(c), 1000000, 1024) == 0
    assert c.abi_version == 2 and c.capacity == 6000 and c.threshold == 1000 and c.policy == 0
    assert list(c.hidden) == [256, 256] and c.lr0 == 1e-3 and c.lr_min == 2.5e-4
    assert c.temp_lo == 100.0 and c.temp_hi == 500.0 and c.lr_halving_samples == 10000


def test_sass_is_sm100a_tensor_core_code(lib):
    sass = subprocess.run(["cuobjdump", "-sass", os.path.join(PKG, "libmel.so")], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", os.path.join(PKG, "libmel.so")], capture_output=True,
                                       text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, flags=re.M), f
                assert not re.search(r"""["']oracle[/"']""", txt), f     # no path / module strings


def test_create_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2309_16743_b200 import mel
    with pytest.raises(mel.MelError):
        mel.Context(mel.Config(n_field=100, hidden=(32,), capacity=200, threshold=33, batch=8))


def test_dataset_header_exported(lib):
    """include/mel_dataset.h (offline baseline data path) is exported by libmel.so."""
    from paper_2309_16743_b200 import mel
    names = declared_functions(os.path.join(ROOT, "include", "mel_dataset.h"))
    assert sorted(mel.DATASET_EXPORTS) == names
    missing = [n for n in names if n not in _exported("libmel.so")]
    assert not missing, missing


def test_heat_header_exported(lib):
    """include/mel_heat.h (on-device heat-equation client) is exported by libmel.so."""
    from paper_2309_16743_b200 import mel
    names = declared_functions(os.path.join(ROOT, "include", "mel_heat.h"))
    assert sorted(mel.HEAT_EXPORTS) == names
    missing = [n for n in names if n not in _exported("libmel.so")]
    assert not missing, missing
