"""Graph / training-set file formats: the library's
parsers restate edge_list.cpp:14-62 and training_set.cpp:51-83; the
reference's own unit tests (test_edge_list.cpp, test_training_set.cpp) are
replayed here, and a file round trip is built into a device graph and
compared with the reference's load_edge_list_file + build_undirected_csr."""
import numpy as np
import pytest


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_edge_list_plain_pairs(pg, tmp_path):  # test_edge_list.cpp:9-16
    el = pg.load_edge_list_file(write(tmp_path, "a.txt", "0 1\n1 2\n"))
    assert el.pairs.tolist() == [[0, 1], [1, 2]] and el.self_loops_dropped == 0


def test_edge_list_comments_and_self_loops(pg, tmp_path):  # :18-24
    el = pg.load_edge_list_file(write(tmp_path, "a.txt", "# c\n3 3\n0 3\n"))
    assert el.pairs.tolist() == [[0, 3]] and el.self_loops_dropped == 1


def test_edge_list_reports_line(pg, tmp_path):  # :26-36
    with pytest.raises(pg.ParseError):
        pg.load_edge_list_file(write(tmp_path, "a.txt", "0 x\n"))
    with pytest.raises(pg.ParseError) as e:
        pg.load_edge_list_file(write(tmp_path, "b.txt", "0 1\n0 x\n"))
    assert e.value.line_number == 2


@pytest.mark.parametrize("text", ["-1 2\n", "7\n", "1 2 3\n", "+1 2\n", "4294967296 1\n", "1 2x\n"])
def test_edge_list_rejects(pg, tmp_path, text):  # :38-45
    with pytest.raises(pg.ParseError):
        pg.load_edge_list_file(write(tmp_path, "a.txt", text))


def test_edge_list_whitespace(pg, tmp_path):  # :47-52
    el = pg.load_edge_list_file(write(tmp_path, "a.txt", "\n  0 1  \n\t\n2\t4\r\n"))
    assert el.pairs.tolist() == [[0, 1], [2, 4]]


def test_edge_list_missing_file(pg, tmp_path):
    with pytest.raises(pg.IoError):
        pg.load_edge_list_file(tmp_path / "nope.txt")


def test_edge_list_round_trip(pg, tmp_path, orc):
    pairs, _ = orc.gen_rmat(300, 2000, 0.45, 0.22, 0.22, 0.11, 5)
    p = tmp_path / "g.txt"
    pg.write_edge_list(p, pairs)
    el = pg.load_edge_list_file(p)
    keep = pairs[:, 0] != pairs[:, 1]
    assert np.array_equal(el.pairs, pairs[keep]) and el.self_loops_dropped == int((~keep).sum())


def test_training_set_file(pg, tmp_path):  # test_training_set.cpp:64-76
    vt = pg.sample_training_set(50, 0.2, 9)
    p = tmp_path / "vt.txt"
    pg.write_training_set(p, vt)
    assert np.array_equal(pg.load_training_set_file(p, 50), vt)
    with pytest.raises(pg.ConfigError):
        pg.load_training_set_file(write(tmp_path, "b.txt", "1\n99\n"), 10)
    # comments, blanks, duplicates, stoll prefix parse
    got = pg.load_training_set_file(write(tmp_path, "c.txt", "# x\n 5\n\n3\n5\n7abc\n"), 10)
    assert got.tolist() == [3, 5, 7]
    with pytest.raises(pg.ParseError):
        pg.load_training_set_file(write(tmp_path, "d.txt", "x\n"), 10)
    with pytest.raises(pg.ConfigError, match="empty"):
        pg.load_training_set_file(write(tmp_path, "e.txt", "# only\n"), 10)
    with pytest.raises(pg.ConfigError):
        pg.load_training_set_file(write(tmp_path, "f.txt", "-2\n"), 10)


def test_file_formats_match_reference(pg, tmp_path, orc, ref):
    """The same files through the reference's loaders."""
    pairs, _ = orc.gen_rmat(500, 3000, 0.45, 0.22, 0.22, 0.11, 8)
    p = tmp_path / "g.txt"
    pg.write_edge_list(p, pairs)
    want = ref.load_graph_file(str(p), symnorm=True)
    el = pg.load_edge_list_file(p)
    got = orc.build_graph(el.pairs, n_hint=None, symnorm=True)
    assert got.n == want.n
    assert np.array_equal(got.offsets, want.offsets) and np.array_equal(got.neighbors, want.neighbors)
    assert np.array_equal(got.weights.view(np.uint64), want.weights.view(np.uint64))


@pytest.mark.gpu
def test_graph_load_file_on_device(pg, tmp_path, orc, cuda):
    pairs, _ = orc.gen_rmat(2000, 20000, 0.45, 0.22, 0.22, 0.11, 8)
    p = tmp_path / "g.txt"
    pg.write_edge_list(p, pairs)
    g = pg.load_graph_file(p, weights="symnorm")
    offs, nb, w = g.export()
    want = orc.build_graph(pg.load_edge_list_file(p).pairs, n_hint=None, symnorm=True)
    assert g.n == want.n and np.array_equal(offs, want.offsets) and np.array_equal(nb, want.neighbors)
    assert np.array_equal(w.view(np.uint64), want.weights.view(np.uint64))
