"""Host logic: SPEC's text formats BADMODEL v1, HASHSIFT v1 and DESC v1
— round trips, the frame conversion (box centre in the 32x32 patch <-> offset from (16, 16),
side s <-> radius r, R1), the LSB-first byte order of descriptor dumps (R16), and rejection of
malformed files."""
import numpy as np
import pytest

from paper_2108_08380_b200 import model_files as mf


def test_bad_model_round_trip_and_frame(tmp_path):
    rng = np.random.default_rng(1)
    pairs = rng.integers(-16, 16, size=(64, 4)).astype(np.int8)
    radii = rng.integers(0, 8, size=64).astype(np.uint8)
    thr = rng.uniform(-20, 20, size=64).astype(np.float32)
    p = tmp_path / "m.txt"
    mf.write_bad_model(p, pairs, radii, thr)
    lines = p.read_text().splitlines()
    assert lines[:2] == ["BADMODEL v1", "K 64"]
    x1, y1, x2, y2, s = (int(v) for v in lines[2].split()[:5])
    assert (x1, y1, x2, y2) == tuple(int(v) + 16 for v in pairs[0]) and s == 2 * radii[0] + 1
    p2, r2, t2 = mf.read_bad_model(p)
    assert (p2 == pairs).all() and (r2 == radii).all() and (t2 == thr).all()


def test_bad_model_hand_written(tmp_path):
    p = tmp_path / "m.txt"
    p.write_text("BADMODEL v1\nK 2\n16 16 0 31 3 -2.5\n31 0 5 7 15 10\n")
    pairs, radii, thr = mf.read_bad_model(p)
    assert pairs.tolist() == [[0, 0, -16, 15], [15, -16, -11, -9]]
    assert radii.tolist() == [1, 7] and thr.tolist() == [-2.5, 10.0]


@pytest.mark.parametrize("body", ["BADMODEL v2\nK 1\n1 1 1 1 3 0\n", "BADMODEL v1\nK 2\n1 1 1 1 3 0\n",
                                  "BADMODEL v1\nK 1\n1 1 1 1 4 0\n", "BADMODEL v1\nK 1\n1 1 32 1 3 0\n",
                                  "BADMODEL v1\nK 1\n1 1 1 1 17 0\n"])
def test_bad_model_rejects(tmp_path, body):
    p = tmp_path / "m.txt"
    p.write_text(body)
    with pytest.raises(ValueError):
        mf.read_bad_model(p)


def test_hashsift_model_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    B = rng.normal(0, 0.1, size=(32, 129)).astype(np.float32)
    p = tmp_path / "h.txt"
    mf.write_hashsift_model(p, B, rootsift=True)
    assert p.read_text().splitlines()[1] == "K 32 rootsift 1"
    B2, root = mf.read_hashsift_model(p)
    assert root and (B2 == B).all()  # 9 significant digits round-trip float32 exactly
    p.write_text("HASHSIFT v1\nK 1 rootsift 0\n" + " ".join(["0.5"] * 128) + "\n")
    with pytest.raises(ValueError):
        mf.read_hashsift_model(p)


def test_descriptor_dump_round_trip_and_bit_order(tmp_path):
    words = np.zeros((2, 8), dtype=np.uint32)  # K = 256
    words[0, 0] = 0x1                         # bit 0 -> LSB of byte 0
    words[1, 7] = 0x80000000                  # bit 255 -> MSB of byte 31
    p = tmp_path / "d.txt"
    mf.write_descriptors(p, words, 256)
    lines = p.read_text().splitlines()
    assert lines[0] == "DESC v1 bits=256 count=2"
    assert lines[1] == "01" + "00" * 31 and lines[2] == "00" * 31 + "80"
    w2, K = mf.read_descriptors(p)
    assert K == 256 and (w2 == words).all()


@pytest.mark.gpu
def test_models_from_files_match_array_models(tmp_path):
    """BadModel.from_file / HashSiftModel.from_file give the same descriptors as the models
    built from the arrays the files were written from."""
    import torch

    import paper_2108_08380_b200 as bd
    import synth
    pairs, radii, thr = synth.bad_tests(21, 256)
    B = synth.hashsift_matrix(22, 256)
    mf.write_bad_model(tmp_path / "b.txt", pairs, radii, thr)
    mf.write_hashsift_model(tmp_path / "h.txt", B)
    P = torch.from_numpy(synth.patches(23, np.arange(300))).cuda()
    a = bd.bad_compute_patches(bd.BadModel(pairs, radii, thr), P)
    b = bd.bad_compute_patches(bd.BadModel.from_file(tmp_path / "b.txt"), P)
    c = bd.hashsift_compute_patches(bd.HashSiftModel(B), P)
    d = bd.hashsift_compute_patches(bd.HashSiftModel.from_file(tmp_path / "h.txt"), P)
    torch.cuda.synchronize()
    assert (a.cpu() == b.cpu()).all() and (c.cpu() == d.cpu()).all()
