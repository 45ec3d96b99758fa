"""QNTC container and the weight hand-off: the native
packer (lvsg_pack_param_store_qntc), the Python mirror (qntc.pack_tensors /
unpack_tensors) and the reference's own pack_tensors / unpack_tensors
(io.cpp:100-171, built into oracle/_ref) agree byte for byte and reject
malformed containers with the same messages. CPU only; the device load is
in test_gpu_kernels.py::test_load_weights_qntc."""
import hashlib
import struct

import numpy as np
import pytest

import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import qntc
from paper_2411_16680_b200.capi import IoError
from paper_2411_16680_b200.config import SchemaError

# sha256 of the reference's pack_tensors over init_param_store(cfg, 3) with
# qntc.param_names as entry names (oracle/_ref, generated in this container).
GOLDEN_SHA = {
    "nano": "f77f78f81858cb9b373064ad178578a98e51619769d689426df768705615fc43",
    "full_scale": "8c4279e6b1196bd8f1aa4544249e28be7529f25b5d8445517eeb968f1303ac76",
}
CONFIGS = {"nano": q.nano_config(), "full_scale": q.full_scale_config()}


def test_param_names_follow_build_params():
    names = qntc.param_names(q.full_scale_config())
    assert len(names) == 312 and len(set(names)) == 312
    # SURVEY.md App. A landmarks
    assert names[0] == "init_feature" and names[1] == "encoder.stem_w"
    assert [names[i] for i in (11, 20, 29, 38)] == [f"encoder.levels.{k}.ray_proj" for k in range(4)]
    assert names[39:44] == ["heads.w_sigma", "heads.w_depth", "heads.w_appear", "blend_w",
                            "blend_gain"]
    assert names[44] == "steps.0.cnn.stem_w" and names[250] == "steps.4.collapse.0.w1"
    assert names[-1] == "steps.5.fusions.1.mlps.0.b2"
    assert len(qntc.param_names(q.nano_config())) == 119


@pytest.mark.parametrize("name", list(CONFIGS))
def test_native_pack_matches_golden_and_python(name):
    cfg = CONFIGS[name]
    b = qntc.pack_param_store(cfg, 3)
    assert hashlib.sha256(b).hexdigest() == GOLDEN_SHA[name]
    store = q.init_param_store(cfg, 3)
    assert qntc.pack_tensors(list(zip(qntc.param_names(cfg), store))) == b
    back = qntc.unpack_tensors(b)
    assert [e.name for e in back] == qntc.param_names(cfg)
    for e, t in zip(back, store):
        assert e.array.dtype == np.float32 and np.array_equal(e.array, t)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_reference_pack_matches(reference, name):
    cfg = CONFIGS[name]
    assert reference.pack_param_store(cfg, 3, qntc.param_names(cfg)) == qntc.pack_param_store(cfg, 3)


def _mixed():
    rng = np.random.default_rng(0)
    return qntc.pack_tensors([("a", rng.standard_normal((2, 3)).astype(np.float32)),
                              ("depth_logits", rng.standard_normal((2, 1, 4))),
                              ("", np.zeros((0,), np.float32)),
                              ("scalar", np.float32(1.5).reshape(())),
                              ("near_far", np.array([0.5, 100.0]))])


def test_roundtrip_mixed_dtypes(reference):
    b = _mixed()
    assert qntc.pack_tensors([(e.name, e.array) for e in qntc.unpack_tensors(b)]) == b
    assert reference.qntc_roundtrip(b) == b
    e = qntc.unpack_tensors(b)
    assert e[1].array.dtype == np.float64 and e[1].array.shape == (2, 1, 4)
    assert qntc.find_tensor(e, "near_far").as_f64().tolist() == [0.5, 100.0]
    with pytest.raises(SchemaError, match='holds f64, expected f32'):
        qntc.find_tensor(e, "near_far").as_f32()
    with pytest.raises(SchemaError, match='missing entry "nope"'):
        qntc.find_tensor(e, "nope")


def _corrupt_cases():
    good = _mixed()
    first = 12 + 4 + 1  # header, name length, name "a"
    return {
        "magic": b"QNTX" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "empty": b"",
        "short_magic": b"QN",
        "no_count": good[:8],
        "count": good[:8] + struct.pack("<I", (1 << 20) + 1) + good[12:],
        "name_len": good[:12] + struct.pack("<I", (1 << 16) + 1) + good[16:],
        "dtype": good[:first] + b"\x02" + good[first + 1:],
        "rank": good[:first + 1] + struct.pack("<I", 17) + good[first + 5:],
        "extent": good[:first + 5] + struct.pack("<Q", (1 << 32) + 1) + good[first + 13:],
        "payload": good[:first + 5 + 16 + 8],
        "trailing": good + b"\0\0\0",
        "truncated_name": good[:14],
    }


@pytest.mark.parametrize("case", list(_corrupt_cases()))
def test_corrupt_container_messages_match_reference(reference, case):
    data = _corrupt_cases()[case]
    with pytest.raises(IoError) as mine:
        qntc.unpack_tensors(data)
    with pytest.raises(IoError) as ref:
        reference.qntc_roundtrip(data)
    assert str(mine.value) == str(ref.value)
    assert str(mine.value).startswith("tensor container: ")
