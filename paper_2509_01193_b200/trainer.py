"""Multi-task LoRA fine-tuning driver around the hot path.

* adapter parameters live in ONE fp32 master buffer with the layout of the layer's flat
  adapter-gradient buffer (per projection: A_cat [sum r, in] then B_cat [out, sum r]); the
  layer's bf16 operands A / B are views into the optimizer's bf16 copy, so an optimizer step
  refreshes them in place (lobra_adamw_step writes both);
* per-task AdamW hyper-parameters ("Adam optimizer"; one group per task, element ->
  task id: the row of A_t, the column of B_t);
* gradient accumulation over the micro-batches of a step (the first backward overwrites the
  gradient buffer, the rest accumulate) and the adapter all-reduce before the
  update;
* LoRA-only checkpoints (adapters + optimizer state + task table; the frozen base is not
  saved) and exact resume: the kernels are deterministic, so resuming reproduces the
  uninterrupted run bit for bit;
* task changes (tasks join or finish): add_task / remove_task re-lay the
  adapter buffers, keep every other task's parameters and optimizer state bit for bit, and
  `replan` re-runs the stage-1 deployment planner for the new task mix.

Single-replica TP1 layout (views); TP > 1 replicas shard A / B and are driven by layer.py
directly.
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .layer import LoraLayer


@dataclass
class TaskConfig:
    name: str
    rank: int
    scale: float = 2.0
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


class MultiTaskLoRATrainer:
    def __init__(self, shapes, tasks, device="cuda:0", seed=0, comm=None):
        self.shapes = list(shapes)
        self.tasks = [dataclasses.replace(t) for t in tasks]
        self.dev = torch.device(device)
        self.seed = seed
        self.comm = comm
        self.layer = LoraLayer(self.shapes, [t.rank for t in self.tasks], [t.scale for t in self.tasks],
                               self.dev, torch.bfloat16, comm=comm, seed=seed)
        self.step_count = 0
        self.task_steps = {t.name: 0 for t in self.tasks}   # optimizer steps taken per task
        self._new_micro_batch = True
        n = self.layer.flat_grad.numel()
        self.params = torch.empty(n, dtype=torch.float32, device=self.dev)
        for p in self.layer.projs:        # standard LoRA init: A random (the layer's draw), B = 0
            self._block(self.params, p, "A").copy_(p.A.float())
            self._block(self.params, p, "B").zero_()
        self.m = torch.zeros(n, dtype=torch.float32, device=self.dev)
        self.v = torch.zeros(n, dtype=torch.float32, device=self.dev)
        self._bind()

    # ------------------------------------------------------------------ layout helpers
    def _ranks(self):
        return np.array([t.rank for t in self.tasks], np.int64)

    def _block(self, flat, p, which):
        R = self.layer.rsum
        if which == "A":
            return flat[p.dA_off:p.dA_off + R * p.d_in].view(R, p.d_in)
        return flat[p.dB_off:p.dB_off + p.d_out * R].view(p.d_out, R)

    def _bind(self):
        """bf16 operand copy + layer views + per-element task ids for the current layout."""
        n = self.params.numel()
        self.params_bf16 = self.params.to(torch.bfloat16)
        tid_of_r = torch.repeat_interleave(torch.arange(len(self.tasks), device=self.dev),
                                           torch.as_tensor(self._ranks(), device=self.dev))
        self.group = torch.empty(n, dtype=torch.uint8, device=self.dev)
        for p in self.layer.projs:
            p.A = self._block(self.params_bf16, p, "A")
            p.B = self._block(self.params_bf16, p, "B")
            self._block(self.group, p, "A").copy_(tid_of_r[:, None].expand(-1, p.d_in).to(torch.uint8))
            self._block(self.group, p, "B").copy_(tid_of_r[None, :].expand(p.d_out, -1).to(torch.uint8))

    def hparams(self):
        """Per-task AdamW hyper-parameters with each task's own step count (the step the
        coming update is for): a task added mid-run starts its bias correction at 1."""
        return [{"lr": t.lr, "beta1": t.beta1, "beta2": t.beta2, "eps": t.eps, "weight_decay": t.weight_decay,
                 "step": self.task_steps[t.name] + 1}
                for t in self.tasks]

    # ------------------------------------------------------------------ the step
    def forward(self, seq_lens, seq_task, io, T, stream=None):
        self.layer.forward(seq_lens, seq_task, io, T, stream=stream)

    def backward(self, seq_lens, seq_task, io, T, stream=None):
        """Adapter gradients of this micro-batch: written by the first backward of a step,
        accumulated by the following ones."""
        self.layer.backward(seq_lens, seq_task, io, T, accumulate_dadb=not self._new_micro_batch, stream=stream)
        self._new_micro_batch = False

    def optimizer_step(self, grad_scale=1.0, stream=None):
        """All-reduce the adapter gradients across replicas, one AdamW step over every
        task's adapters with its own hyper-parameters, bf16 operands refreshed in place."""
        if self._new_micro_batch:
            raise RuntimeError("optimizer_step without a backward in this step")
        self.layer.sync_adapter_grads(stream=stream)
        hp = self.hparams()
        self.step_count += 1
        _lib.lobra_adamw_step(self.params, self.layer.flat_grad, self.m, self.v, hp, self.step_count,
                              group=self.group, params_bf16=self.params_bf16, grad_scale=grad_scale, stream=stream)
        for t in self.tasks:
            self.task_steps[t.name] += 1
        self._new_micro_batch = True

    # ------------------------------------------------------------------ checkpoints
    def state_dict(self):
        return {"format": "lobra-lora-adapters-v1", "shapes": self.shapes,
                "tasks": [dataclasses.asdict(t) for t in self.tasks], "step": self.step_count,
                "task_steps": dict(self.task_steps),
                "params": self.params.cpu(), "m": self.m.cpu(), "v": self.v.cpu()}

    def load_state_dict(self, sd):
        if sd.get("format") != "lobra-lora-adapters-v1":
            raise ValueError("not a lobra adapter checkpoint")
        if [tuple(x) for x in sd["shapes"]] != [tuple(x) for x in self.shapes]:
            raise ValueError("checkpoint was taken on other projection shapes")
        tasks = [TaskConfig(**t) for t in sd["tasks"]]
        if [(t.name, t.rank) for t in tasks] != [(t.name, t.rank) for t in self.tasks]:
            self.tasks = tasks
            self.layer.relayout([t.rank for t in tasks], [t.scale for t in tasks])
        self.tasks = tasks
        self.layer.scales = np.array([t.scale for t in tasks], np.float32)
        self.params = sd["params"].to(self.dev).clone()
        self.m = sd["m"].to(self.dev).clone()
        self.v = sd["v"].to(self.dev).clone()
        self.step_count = int(sd["step"])
        # checkpoints without per-task counts predate task changes: every task took them all
        self.task_steps = {t.name: int(sd.get("task_steps", {}).get(t.name, self.step_count)) for t in tasks}
        self._new_micro_batch = True
        self._bind()

    def save(self, path):
        torch.save(self.state_dict(), path)

    def load(self, path):
        self.load_state_dict(torch.load(path, map_location="cpu"))

    # ------------------------------------------------------------------ task changes
    def _relayout(self, new_tasks, init_seed=0):
        """Move every kept task's A rows / B columns (parameters and optimizer moments) into
        the layout of `new_tasks`; new tasks start as LoRA does (A ~ N(0, 1/in), B = 0)."""
        old_tasks, old_layer_offsets = self.tasks, [(p.dA_off, p.dB_off) for p in self.layer.projs]
        old_R = self.layer.rsum
        old_roff = np.concatenate([[0], np.cumsum([t.rank for t in old_tasks])])
        old_idx = {t.name: i for i, t in enumerate(old_tasks)}
        old = (self.params, self.m, self.v)
        self.tasks = [dataclasses.replace(t) for t in new_tasks]
        self.layer.relayout([t.rank for t in self.tasks], [t.scale for t in self.tasks])
        n, R = self.layer.flat_grad.numel(), self.layer.rsum
        new = tuple(torch.zeros(n, dtype=torch.float32, device=self.dev) for _ in range(3))
        roff = np.concatenate([[0], np.cumsum([t.rank for t in self.tasks])])
        g = torch.Generator(device=self.dev)
        g.manual_seed(init_seed)
        for p, (a0, b0) in zip(self.layer.projs, old_layer_offsets):
            for j, t in enumerate(self.tasks):
                r0, r1 = int(roff[j]), int(roff[j + 1])
                if t.name in old_idx:
                    i = old_idx[t.name]
                    o0, o1 = int(old_roff[i]), int(old_roff[i + 1])
                    if o1 - o0 != r1 - r0:
                        raise ValueError(f"task {t.name}: rank changed ({o1 - o0} -> {r1 - r0})")
                    for src, dst in zip(old, new):
                        oa = src[a0:a0 + old_R * p.d_in].view(old_R, p.d_in)
                        ob = src[b0:b0 + p.d_out * old_R].view(p.d_out, old_R)
                        self._block(dst, p, "A")[r0:r1].copy_(oa[o0:o1])
                        self._block(dst, p, "B")[:, r0:r1].copy_(ob[:, o0:o1])
                else:
                    self._block(new[0], p, "A")[r0:r1].copy_(
                        torch.randn(r1 - r0, p.d_in, generator=g, device=self.dev) / math.sqrt(p.d_in))
        self.params, self.m, self.v = new
        self.task_steps = {t.name: self.task_steps.get(t.name, 0) for t in self.tasks}
        self._bind()

    def add_task(self, task: TaskConfig, init_seed=0):
        if any(t.name == task.name for t in self.tasks):
            raise ValueError(f"task {task.name} exists")
        self._relayout(self.tasks + [task], init_seed)

    def remove_task(self, name: str):
        keep = [t for t in self.tasks if t.name != name]
        if len(keep) == len(self.tasks):
            raise KeyError(name)
        self._relayout(keep)

    def replan(self, tp, max_tokens, cost, n_gpus, lens_sample, batch_size=0, **kw):
        """Stage-1 deployment plan for the current task mix (lobra_plan_deployment)."""
        return _lib.lobra_plan_deployment(tp, max_tokens, cost, n_gpus, lens_sample, batch_size, **kw)

    def task_params(self, name):
        """fp32 (A_t, B_t) of one task per projection name (host copies)."""
        j = [t.name for t in self.tasks].index(name)
        roff = np.concatenate([[0], np.cumsum(self._ranks())])
        r0, r1 = int(roff[j]), int(roff[j + 1])
        return {p.name: (self._block(self.params, p, "A")[r0:r1].cpu(), self._block(self.params, p, "B")[:, r0:r1].cpu())
                for p in self.layer.projs}
