"""Evaluation of a classifier graph (reference cli.py:241-266).

The forward pass runs on the device (an eval graph: `networks.resnet50(...,
train=False)` puts every BatchNormalization on its running statistics through
`nnl_bn_fwd_eval`); the per-row argmax and log-softmax are the reference's own
numpy expressions on the logits read back, so error counts are bit-exact on
identical logits (ties go to the first index, as `np.argmax`) and the loss
matches to float32 rounding.
"""

from __future__ import annotations

import numpy as np

from .graph import Variable


def evaluate_classifier(x_var: Variable, logits_var: Variable, xs: np.ndarray,
                        labels: np.ndarray) -> tuple[float, float]:
    """(classification error, mean cross-entropy) over a dataset, in chunks of
    the graph's batch extent; the tail chunk wraps around and only real rows
    count (deterministic, as the reference)."""
    batch = x_var.shape[0]
    n = xs.shape[0]
    wrong = 0
    loss_sum = 0.0
    for start in range(0, n, batch):
        idx = np.arange(start, start + batch) % n
        real = min(batch, n - start)
        x_var.d = xs[idx]
        logits_var.forward()
        logits = logits_var.d[:real]
        want = labels[idx][:real].astype(np.int64)
        wrong += int((np.argmax(logits, axis=1) != want).sum())
        z = logits - logits.max(axis=1, keepdims=True)
        logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
        loss_sum += float(-logp[np.arange(real), want].sum())
    return wrong / n, loss_sum / n
