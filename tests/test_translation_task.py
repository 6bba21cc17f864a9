"""The file-based `translation` task (reference tasks.cpp:7-33, Dictionary /
corpus loading data.cpp:13-120, 225-271) against the reference's own
TranslationTask on the same text files: dictionary sizes and every
eos-terminated id sequence identical, with built and with loaded
dictionaries, min_count, unknown words and empty lines; error classes as the
reference's. CPU only. The reference side runs in a child process that loads
nothing but the oracle library (its iostream-based readers must not share a
process with numpy's runtime libraries)."""
import os
import subprocess
import sys

import pytest

import paper_1904_01038_b200 as sqf
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes as C, sys, json
L = C.CDLL(sys.argv[1])
f = L.sqfref_task_dump
f.restype = C.c_int
f.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), C.c_int, C.c_void_p, C.c_int64]
kv = json.loads(sys.argv[2])
keys = (C.c_char_p * len(kv))(*[k.encode() for k in kv])
vals = (C.c_char_p * len(kv))(*[str(v).encode() for v in kv.values()])
buf = C.create_string_buffer(1 << 22)
rc = f(b"transformer_base_defaults", keys, vals, len(kv), buf, 1 << 22)
if rc:
    L.sqfref_last_error.restype = C.c_char_p
    print("ERR", rc, L.sqfref_last_error().decode())
else:
    sys.stdout.write(buf.value.decode())
'''


def ref_task(kv):
    import json
    out = subprocess.run([sys.executable, "-c", CHILD, ref.LIB, json.dumps(kv)], capture_output=True, text=True,
                         timeout=120).stdout
    lines = out.splitlines()
    if lines[0].startswith("ERR"):
        return lines[0]
    sv, tv, n = map(int, lines[0].split())
    pairs = []
    for ln in lines[1:1 + n]:
        a, b = ln.split("|")
        pairs.append(([int(x) for x in a.split()], [int(x) for x in b.split()]))
    return sv, tv, pairs


def write(tmp, name, lines):
    p = tmp / name
    p.write_text("\n".join(lines) + "\n")
    return str(p)


SRC = ["das haus ist klein", "das haus ist sehr klein", "", "ein neues haus", "haus haus das  ist"]
TGT = ["the house is small", "the house is very small", "nothing here", "a new house", "house house the is"]


@pytest.mark.parametrize("min_count", [1, 2])
def test_built_dictionaries_and_pairs_match_reference(tmp_path, min_count):
    if not ref.available():
        pytest.skip("oracle not built")
    kv = {"task": "translation", "train_src": write(tmp_path, "t.src", SRC), "train_tgt": write(tmp_path, "t.tgt", TGT),
          "min_count": min_count}
    sv, tv, pairs = sqf.load_task("transformer_base_defaults", kv)
    assert (sv, tv, pairs) == ref_task(kv)
    assert all(s[-1] == 2 and t[-1] == 2 for s, t in pairs)  # eos-terminated
    if min_count == 2:
        assert 3 in pairs[3][0]  # "ein", "neues" are <unk>


def test_loaded_dictionaries_match_reference(tmp_path):
    if not ref.available():
        pytest.skip("oracle not built")
    d_src = write(tmp_path, "dict.src", ["haus 9", "das 3", "klein 2", "ist 1"])
    d_tgt = write(tmp_path, "dict.tgt", ["house 9", "the 3", "small 2"])
    kv = {"task": "translation", "train_src": write(tmp_path, "t.src", SRC), "train_tgt": write(tmp_path, "t.tgt", TGT),
          "dict_src": d_src, "dict_tgt": d_tgt}
    got = sqf.load_task("transformer_base_defaults", kv)
    assert got == ref_task(kv)
    assert got[0] == 8 and got[1] == 7


def test_errors_match_reference_classes(tmp_path):
    # Registry::make_task wraps constructor failures as RegistryError("task 'x': ...")
    # (registry.cpp:112-161); the inner message carries the reference's error
    a = write(tmp_path, "a.txt", SRC)
    with pytest.raises(Exception, match="RegistryError.*given together"):  # train_src without train_tgt
        sqf.load_task("transformer_base_defaults", {"task": "translation", "train_src": a})
    with pytest.raises(Exception, match="RegistryError.*line count mismatch"):
        sqf.load_task("transformer_base_defaults", {"task": "translation", "train_src": a,
                                                    "train_tgt": write(tmp_path, "b.txt", TGT[:3])})
    with pytest.raises(Exception, match="RegistryError.*cannot"):  # missing file
        sqf.load_task("transformer_base_defaults", {"task": "translation", "train_src": a,
                                                    "train_tgt": str(tmp_path / "nope")})
    dup = write(tmp_path, "dup.dict", ["x 1", "x 2"])
    with pytest.raises(Exception, match="RegistryError.*duplicate symbol"):
        sqf.load_task("transformer_base_defaults", {"task": "translation", "train_src": a,
                                                    "train_tgt": write(tmp_path, "c.txt", TGT), "dict_src": dup})
