"""fp64 oracle of the multi-tenant AdamW adapter update -- TEST INFRASTRUCTURE ONLY.

PAPER.md P:709: "We use the Adam optimizer [adam, adamw] for all experiments."  AdamW
(decoupled weight decay), written out per element, one hyper-parameter set per group
(task), t = the group's own step count (hparams[k]["step"] when given, else `step`: a task
that joined the joint run later has taken fewer steps):
    g = s * grad
    m_t = b1 m_{t-1} + (1 - b1) g
    v_t = b2 v_{t-1} + (1 - b2) g^2
    p_t = p_{t-1} - lr ( (m_t / (1 - b1^t)) / (sqrt(v_t / (1 - b2^t)) + eps) + wd p_{t-1} )
"""
from __future__ import annotations

import numpy as np


def adamw_step(p, g, m, v, group, hparams, step, grad_scale=1.0):
    p = np.asarray(p, np.float64).copy()
    m = np.asarray(m, np.float64).copy()
    v = np.asarray(v, np.float64).copy()
    g = np.asarray(g, np.float64) * grad_scale
    group = np.zeros(p.shape, np.int64) if group is None else np.asarray(group, np.int64)
    for k, h in enumerate(hparams):
        sel = group == k
        b1, b2 = h["beta1"], h["beta2"]
        t = h.get("step") or step
        m[sel] = b1 * m[sel] + (1 - b1) * g[sel]
        v[sel] = b2 * v[sel] + (1 - b2) * g[sel] ** 2
        mh = m[sel] / (1 - b1 ** t)
        vh = v[sel] / (1 - b2 ** t)
        p[sel] = p[sel] - h["lr"] * (mh / (np.sqrt(vh) + h["eps"]) + h["weight_decay"] * p[sel])
    return p, m, v
