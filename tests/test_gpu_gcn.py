"""GCN-level behaviours of the drop-in (gcn.py of the reference): the loss
at known points, zero features, zero learning rate, degenerate graphs and
input validation -- on the GPU path."""

import numpy as np
import pytest

import paper_2504_04673_b200 as P

pytestmark = pytest.mark.gpu


def test_uniform_logits_loss_is_log_k():
    k = 7
    loss, grad = P.softmax_xent(np.zeros((5, k)), np.arange(5) % k, np.ones(5, bool))
    assert abs(loss - np.log(k)) < 1e-6
    assert np.allclose(grad.sum(axis=1), 0.0, atol=1e-7)


def test_confident_correct_logit_loss_vanishes():
    logits = np.full((3, 4), -30.0)
    logits[np.arange(3), [0, 2, 3]] = 30.0
    loss, _ = P.softmax_xent(logits, np.array([0, 2, 3]), np.ones(3, bool))
    assert loss < 1e-6


def test_xent_rejects_bad_inputs():
    with pytest.raises(ValueError):
        P.softmax_xent(np.zeros((2, 3)), np.array([0, 3]), np.ones(2, bool))
    with pytest.raises(ValueError):
        P.softmax_xent(np.zeros((2, 3)), np.array([0, 1]), np.zeros(2, bool))


def test_forward_zero_features_zero_logits():
    a = P.gcn_normalize(P.csr_from_edges([(0, 1, 1.0), (1, 2, 1.0)], 3, symmetrize=True))
    ws = P.init_weights(P.TrainConfig(layers=3, hidden=4), 5, 3)
    out = P.SerialGcn(a, ws).forward(np.zeros((3, 5)))
    assert np.array_equal(out, np.zeros((3, 3)))
    with pytest.raises(RuntimeError):
        P.SerialGcn(a, ws).backward(np.zeros((3, 3)))


def test_lr_zero_keeps_weights_and_loss_flat():
    a = P.gcn_normalize(P.csr_from_edges([(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)], 4,
                                         symmetrize=True))
    x = np.random.default_rng(0).standard_normal((4, 6))
    y = np.array([0, 1, 1, 0])
    cfg = P.TrainConfig(layers=3, hidden=8, lr=0.0, epochs=4, seed=3)
    res = P.train(a, x, y, np.ones(4, bool), cfg, p=2)
    assert np.all(res.losses == res.losses[0])
    w0 = P.init_weights(cfg, 6, 2)
    for w, ref in zip(res.weights, w0):
        assert np.array_equal(w, ref.astype(np.float32).astype(np.float64))


def test_single_vertex_graph_trains():
    a = P.gcn_normalize(P.csr_from_edges([], 1))
    res = P.train(a, np.ones((1, 3)), np.array([1]), np.ones(1, bool),
                  P.TrainConfig(layers=3, hidden=2, lr=0.5, epochs=5, seed=1, f_out=2))
    assert res.losses[-1] < res.losses[0]


def test_train_input_validation():
    a = P.gcn_normalize(P.csr_from_edges([(0, 1, 1.0)], 2, symmetrize=True))
    cfg = P.TrainConfig(epochs=1)
    with pytest.raises(ValueError):
        P.train(a, np.ones((2, 3)), np.array([0, 1]), np.zeros(2, bool), cfg)
    with pytest.raises(ValueError):
        P.train(a, np.ones((3, 3)), np.array([0, 1, 0]), np.ones(3, bool), cfg)
    with pytest.raises(ValueError):
        P.train(a, np.ones((2, 3)), np.array([0, 1]), np.ones(2, bool), cfg, p=4, c=3)
