"""Host logic of the stacked q / k / v path (no GPU): the flat-buffer order
keeps a block's wq, wk, wv back to back (stage partitions list their names
sorted), and the adjacency / column-block checks that route the fused
GEMMs accept exactly the layouts the fused path produces."""
import torch

from paper_2312_04916_b200.training import _adjacent, _column_blocks, _flat_order, _row_ld


def test_flat_order_groups_qkv():
    names = ["exit_l1.out", "layer1.attn_norm", "layer1.mlp_norm", "layer1.w1", "layer1.w2",
             "layer1.wk", "layer1.wo", "layer1.wq", "layer1.wv", "layer2.wq", "head.wq"]
    out = _flat_order(names)
    assert sorted(out) == sorted(names)
    i = out.index("layer1.wq")
    assert out[i:i + 3] == ["layer1.wq", "layer1.wk", "layer1.wv"]
    # incomplete trios keep their place
    assert out.index("layer2.wq") < out.index("head.wq")
    assert _flat_order(["a", "b"]) == ["a", "b"]


def test_adjacent_and_column_blocks():
    flat = torch.zeros(3 * 64 * 32)
    ws = [flat[i * 2048:(i + 1) * 2048].view(64, 32) for i in range(3)]
    assert _adjacent(ws)
    assert not _adjacent([ws[0], ws[2], ws[1]])
    y = torch.zeros(10, 96)
    q, k, v = y[:, :32], y[:, 32:64], y[:, 64:]
    g = _column_blocks([q, k, v])
    assert g is not None and g.shape == (10, 96) and g.data_ptr() == y.data_ptr()
    assert _column_blocks([q, v, k]) is None
    assert _column_blocks([torch.zeros(10, 32), k, v]) is None


def test_row_ld():
    y = torch.zeros(2, 8, 96)
    assert _row_ld(y[..., 32:64]) == 96
    assert _row_ld(torch.zeros(2, 8, 32)) == 32
    assert _row_ld(y.transpose(0, 1)[..., :32]) is None
