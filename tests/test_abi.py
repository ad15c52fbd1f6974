"""CPU: the C-ABI library loads and exports every symbol include/mihg.h declares; host-side
logic (partition validation, BMIH io, gen_uniform) matches the reference's contracts."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "mihg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mihg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1307_2982_b200 import _lib

    L = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/mihg.h but not exported"
    bound = {s[0] for s in _lib.SYMBOLS}
    assert set(declared) == bound, "python binding and header disagree"
    assert _lib.lib().mihg_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_1307_2982_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_gen_uniform_matches_reference_pins(golden):
    import paper_1307_2982_b200 as mg

    d = golden("gen_uniform_pins")
    for key, want in d.items():
        _, n, bits, seed = key.split("_")
        got = mg.gen_uniform(int(n), int(bits), int(seed)).raw_words()
        assert np.array_equal(got, want), key


def test_gen_uniform_config1_digest(golden):
    import hashlib

    import paper_1307_2982_b200 as mg

    d = golden("config1")
    got = mg.gen_uniform(int(d["n"]), 64, int(d["db_seed"])).raw_words()
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(d["codes_sha256"])


def test_partition_contract():
    import paper_1307_2982_b200 as mg

    p = mg.consecutive_partition(100, 8)
    assert [p.length(j) for j in range(8)] == [13] * 4 + [12] * 4  # codes.hpp:198-211
    p = mg.consecutive_partition(128, 6)
    assert [p.length(j) for j in range(6)] == [22, 22, 21, 21, 21, 21]
    with pytest.raises(ValueError):
        mg.consecutive_partition(4, 0)
    with pytest.raises(ValueError):
        mg.consecutive_partition(4, 5)
    mg.Partition(4, [[3, 0], [1, 2]])  # order within a substring is free
    with pytest.raises(ValueError):
        mg.Partition(4, [[0, 1], [1, 2]])  # assigned twice
    with pytest.raises(ValueError):
        mg.Partition(4, [[0, 1, 2], [3]])  # sizes differ by 2
    with pytest.raises(ValueError):
        mg.Partition(4, [[0, 1], [2, 9]])  # out of range


def test_extract_substring_pins():
    import paper_1307_2982_b200 as mg

    # codes_test.cpp:105-133
    p = mg.consecutive_partition(8, 2)
    c = mg.BinaryCode(np.array([0b11110000], np.uint64), 8)
    assert mg.extract_substring(c, p, 0) == 0 and mg.extract_substring(c, p, 1) == 15
    p = mg.Partition(4, [[3, 0], [1, 2]])
    assert mg.extract_substring(mg.BinaryCode(np.array([0b1000], np.uint64), 4), p, 0) == 0b01
    p = mg.consecutive_partition(70, 7)
    c = mg.BinaryCode(np.array([0b1011 << 60, 0b110101], np.uint64), 70)
    assert mg.extract_substring(c, p, 6) == (0b110101 << 4) | 0b1011


def test_codes_roundtrip_and_format_errors(tmp_path):
    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(37, 70, 5)
    path = str(tmp_path / "c.bmih")
    mg.write_codes(db, path)
    assert mg.read_codes(path) == db
    raw = open(path, "rb").read()
    open(path, "wb").write(b"XMIH" + raw[4:])
    with pytest.raises(mg.FormatError):
        mg.read_codes(path)
    open(path, "wb").write(raw[:-3])
    with pytest.raises(mg.FormatError):
        mg.read_codes(path)
    bad = bytearray(raw)
    bad[20 + 15] = 0xFF  # padding bits of record 0 (70-bit codes: word 1 bits 6..63)
    open(path, "wb").write(bytes(bad))
    with pytest.raises(mg.FormatError) as e:
        mg.read_codes(path)
    assert e.value.offset == 28


def test_reference_bmih_files_are_read(tmp_path):
    """Codes written by the reference's write_codes (io.hpp:151-157) read back identically."""
    import oracle
    import paper_1307_2982_b200 as mg

    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    R = oracle.ref()
    codes = R.gen_uniform(50, 130, 3)
    path = str(tmp_path / "ref.bmih")
    rc = R.lib.ref_write_codes(codes.ctypes.data_as(oracle._u64p), 50, 130, path.encode())
    assert rc == 0
    assert np.array_equal(mg.read_codes(path).raw_words(), codes)


def test_build_validation_before_gpu():
    import paper_1307_2982_b200 as mg

    db = mg.gen_uniform(10, 64, 1)
    with pytest.raises(ValueError):
        mg.MihIndex.build(db, mg.consecutive_partition(32, 2))  # width mismatch
    with pytest.raises(ValueError):
        mg.MihIndex.build(db, mg.consecutive_partition(64, 1))  # 64-bit substring


def test_cpp_facade_compiles_against_reference_types():
    """include/mihg/mih_gpu.hpp accepts mih::CodeDatabase / Partition / BinaryCode / SearchTrace
    (compile check; the GPU run is tests/test_gpu_dropin.py)."""
    import subprocess

    if not os.path.isdir("/root/reference/proj/include/mih"):
        pytest.skip("reference headers not present (GPU box)")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "_build", "facade_with_reference"))
