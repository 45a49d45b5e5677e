"""Pipeline-parallel (PP) execution of a replica's micro-batches, 1F1B.

LobRA's configurations are <TP, PP> pairs (Table tb:parallel_config_thruputs);
with PP > 1 a replica's layers are split into `p` stages on `p` ranks and its micro-batches
-- the variable-length packed chunks `lobra_dispatch` emits -- flow through the stages in
the one-forward-one-backward order whose time App. D models with the variable-length
bubble (`lobra_replica_time`):

    stage s runs min(p - s - 1, m) warm-up forwards, then alternates one forward and one
    backward, then drains the remaining backwards; activations go to stage s + 1 and
    gradients to stage s - 1 by point-to-point send / recv on the process group.

Each stage holds a contiguous range of `DecoderLayer`s (our kernels; `select_context`
keeps one activation set per micro-batch in flight, at most p - s of them).  Backwards run
in micro-batch order, so every layer's adapter gradients accumulate in the same order as
in a single-process run (bitwise equal, tests/test_gpu_pipeline.py).  The process group
may be NCCL (device tensors) or gloo (host staging: tests with several processes on one
GPU).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def schedule_1f1b(num_stages: int, stage: int, num_micro: int):
    """The ops of one stage in 1F1B order: [("F", k) | ("B", k)]."""
    warm = min(num_stages - stage - 1, num_micro)
    ops = [("F", k) for k in range(warm)]
    f, b = warm, 0
    while f < num_micro:
        ops.append(("F", f))
        f += 1
        ops.append(("B", b))
        b += 1
    while b < num_micro:
        ops.append(("B", b))
        b += 1
    return ops


def simulate_1f1b(num_stages: int, t_fwd, t_bwd):
    """Makespan of the 1F1B schedule with per-micro-batch stage times t_fwd[k], t_bwd[k]
    (every stage alike, transfers free): each op starts when its stage is free and its
    input exists (F_k on stage s after F_k on s - 1; B_k on s after B_k on s + 1 and F_k on
    s).  Used to check the schedule and the App. D bubble model on the host."""
    m = len(t_fwd)
    done = {}
    free = [0.0] * num_stages
    ops = [schedule_1f1b(num_stages, s, m) for s in range(num_stages)]
    pos = [0] * num_stages
    remaining = sum(len(o) for o in ops)
    while remaining:
        progressed = False
        for s in range(num_stages):
            if pos[s] == len(ops[s]):
                continue
            op, k = ops[s][pos[s]]
            deps = [("F", s, k)] if op == "B" else []
            if op == "F" and s > 0:
                deps.append(("F", s - 1, k))
            if op == "B" and s < num_stages - 1:
                deps.append(("B", s + 1, k))
            if any(d not in done for d in deps):
                continue
            start = max([free[s]] + [done[d] for d in deps])
            end = start + (t_fwd[k] if op == "F" else t_bwd[k])
            done[(op, s, k)] = end
            free[s] = end
            pos[s] += 1
            remaining -= 1
            progressed = True
        if not progressed:
            raise RuntimeError("1F1B schedule deadlocked")
    return max(free)


class PipelineStage:
    """One PP stage: `layers` (DecoderLayer list) on this rank; `prev` / `next` are the
    global ranks of the neighbouring stages (None at the ends)."""

    def __init__(self, layers, stage: int, num_stages: int, prev=None, next=None, group=None,
                 host_staging: bool = False):
        self.layers, self.stage, self.p = layers, stage, num_stages
        self.prev, self.next, self.group = prev, next, group
        self.host = host_staging
        self.h = layers[0].h
        self.dev = layers[0].dev
        self._pending = []

    def _send(self, t, dst):
        x = t.detach().to("cpu") if self.host else t.detach().contiguous()
        self._pending.append((dist.isend(x, dst, group=self.group), x))

    def _recv(self, T, src):
        if self.host:
            x = torch.empty(T, self.h, dtype=torch.bfloat16)
            dist.recv(x, src, group=self.group)
            return x.to(self.dev)
        x = torch.empty(T, self.h, dtype=torch.bfloat16, device=self.dev)
        dist.recv(x, src, group=self.group)
        return x

    def run(self, micro, inputs=None, grads=None):
        """micro: [(seq_lens, seq_task)] per micro-batch.  inputs[k] (first stage): X of
        micro-batch k; grads[k] (last stage): dY of its output.  Returns (outputs, dX):
        the last stage's outputs and the first stage's input gradients, per micro-batch;
        adapter gradients accumulate in each layer's flat buffer (the first micro-batch
        overwrites)."""
        first, last = self.stage == 0, self.stage == self.p - 1
        outs, dxs = {}, {}
        for op, k in schedule_1f1b(self.p, self.stage, len(micro)):
            lens, tasks = micro[k]
            T = int(sum(lens))
            for layer in self.layers:
                layer.select_context(k)
            if op == "F":
                x = inputs[k] if first else self._recv(T, self.prev)
                for layer in self.layers:
                    x = layer.forward(lens, tasks, x)
                if last:
                    outs[k] = x
                else:
                    self._send(x, self.next)
            else:
                g = grads[k] if last else self._recv(T, self.next)
                for layer in reversed(self.layers):
                    g = layer.backward(g, accumulate_dadb=k > 0)
                if first:
                    dxs[k] = g.clone()
                else:
                    self._send(g, self.prev)
        for w, _ in self._pending:
            w.wait()
        self._pending.clear()
        return outs, dxs
