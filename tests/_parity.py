"""Shared helpers of the GPU parity tests (test infrastructure, not product).

`oracle_output_streamed` evaluates the reference's moe_forward<double>
(moe_layer.hpp:114-158) through the C oracle one expert at a time, so layers
far larger than host memory in fp64 (the C3 235B-shaped layer is 19.3 GB as
double) can be checked: each active expert's weights are downloaded once,
y_e(x_t) = expert_forward<double> (moe_layer.hpp:92-107) is computed by the
oracle for every token that selected e, and the outputs are then accumulated
per token in SET ORDER starting from zero, exactly as moe_forward does
(`out.row(i) += w[j] * expert_forward(E[set[j]], x_i)`, :148-155)."""
import numpy as np

import oracle


def to_bf16_bits(x):
    xb = oracle.bf16_round(x)
    return xb, (xb.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def oracle_output_streamed(get_expert, x, sets, set_len, weights, scalar="f64"):
    """get_expert(e) -> (wg [D,H], wu [D,H], wd [H,D]) as float64 arrays."""
    x = np.asarray(x, np.float64)
    B, D = x.shape
    stride = sets.shape[1]
    users = {}
    for t in range(B):
        for j in range(int(set_len[t])):
            users.setdefault(int(sets[t, j]), []).append((t, j))
    y = np.zeros((B, stride, D), np.float64)
    for e, tj in sorted(users.items()):
        wg, wu, wd = get_expert(e)
        toks = np.array([t for t, _ in tj], np.int64)
        n = len(toks)
        one = np.zeros((n, 1), np.int32)
        ye = oracle.moe_forward(wg[None], wu[None], wd[None], x[toks], one,
                                np.ones(n, np.int32), np.ones((n, 1)), scalar=scalar)
        for (t, j), row in zip(tj, ye):
            y[t, j] = row
    out = np.zeros((B, D), np.float64)
    for t in range(B):
        for j in range(int(set_len[t])):
            out[t] += weights[t, j] * y[t, j]
    return out
