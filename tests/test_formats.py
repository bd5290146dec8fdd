"""File formats around the path: byte-identical PFM / TSPF with the
reference's writers, PNG previews, round trips.  CPU only."""
import numpy as np

from conftest import load_golden


def test_pfm_bytes_and_round_trip(tmp_path):
    from paper_2406_01579_b200.imgio import read_pfm, write_pfm
    G = load_golden("formats.npz")
    for key, arr in (("pfm1", G["a1"]), ("pfm3", G["a3"])):
        p = tmp_path / key
        write_pfm(p, arr)
        assert p.read_bytes() == G[key].tobytes()
        assert np.array_equal(read_pfm(p), arr.astype(np.float32).astype(np.float64))


def test_tspf_checkpoint_bytes_and_round_trip(tmp_path):
    from paper_2406_01579_b200.field import FieldState
    from paper_2406_01579_b200.imgio import load_checkpoint, save_checkpoint
    G = load_golden("formats.npz")
    st = FieldState.from_numpy(G["sdf"], G["deform"], float(G["limit"]), float(G["s"]), device="cpu")
    p = tmp_path / "f.tspf"
    save_checkpoint(st, p)
    assert p.read_bytes() == G["tspf"].tobytes()
    r = load_checkpoint(p, float(G["limit"]), device="cpu")
    assert np.array_equal(r.sdf.numpy(), G["sdf"]) and r.steepness == float(G["s"])


def test_png_preview_quantises_the_pfm_values(tmp_path):
    from PIL import Image
    from paper_2406_01579_b200.imgio import write_png
    a = np.linspace(-0.2, 1.2, 12).reshape(3, 4)
    write_png(tmp_path / "a.png", a)
    got = np.asarray(Image.open(tmp_path / "a.png"))
    assert np.array_equal(got, (np.clip(a.astype(np.float32), 0, 1) * 255).round().astype(np.uint8))
