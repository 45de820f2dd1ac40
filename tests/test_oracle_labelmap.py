"""validate_label_map (label_map.cpp:38-78): the oracle's restatement against
the reference library on valid, gapped and split maps (same num_regions, same
error message), and the RLM1 format errors of read_rlm that precede
validation (graph_test.cpp:139-157)."""
import numpy as np
import pytest

from labelmap_cases import cases
from paper_1809_05018_b200 import engine as E


@pytest.mark.parametrize("name,w,h,region", cases(), ids=[c[0] for c in cases()])
def test_validate_vs_reference(orc, ref, name, w, h, region):
    assert orc.validate_label_map(w, h, region) == ref.validate_label_map(w, h, region)


def test_known_answers(orc):  # graph_test.cpp:160-190
    assert orc.validate_label_map(2, 2, [0, 0, 1, 1]) == 2
    assert orc.validate_label_map(2, 1, [0, 2]) == "label map: region id 1 unused"
    assert "not 4-connected" in orc.validate_label_map(3, 1, [0, 1, 0])
    assert "not 4-connected" in orc.validate_label_map(2, 2, [0, 1, 1, 0])
    assert orc.validate_label_map(0, 3, []) == "label map: empty"


def test_rlm_format_errors(tmp_path):
    path = str(tmp_path / "m.rlm")
    for blob in (b"RLMX\x01\x00\x00\x00\x01\x00\x00\x00\x00\x00\x00\x00",  # magic
                 b"RLM1\x02\x00\x00\x00\x02\x00\x00\x00",                  # truncated ids
                 b"RLM1\x02\x00\x00",                                      # truncated header
                 b"RLM1\x00\x00\x00\x00\x02\x00\x00\x00"):                 # zero dimension
        with open(path, "wb") as f:
            f.write(blob)
        with pytest.raises(E.InputError):
            E.read_rlm(path)
    with pytest.raises(E.InputError):
        E.read_rlm(str(tmp_path / "missing.rlm"))
    with pytest.raises(E.InputError):
        E.write_rlm(E.LabelMap(2, 2, np.zeros(3, np.uint32)), path)
    with pytest.raises(E.InputError):  # size check before any device work
        E.validate_label_map(E.LabelMap(2, 2, np.zeros(3, np.uint32)))


def test_rlm_bytes(tmp_path):
    """write_rlm's layout (label_map.cpp:135-145): magic, u32le w, h, ids."""
    path = str(tmp_path / "m.rlm")
    reg = np.arange(6, dtype=np.uint32)
    E.write_rlm(E.LabelMap(3, 2, reg), path)
    data = open(path, "rb").read()
    assert data[:4] == b"RLM1" and len(data) == 12 + 24
    assert np.array_equal(np.frombuffer(data, "<u4", 2, 4), [3, 2])
    assert np.array_equal(np.frombuffer(data, "<u4", 6, 12), reg)
