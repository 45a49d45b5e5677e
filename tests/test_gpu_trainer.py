"""GPU: the multi-task LoRA training driver (paper_2509_01193_b200/trainer.py).

  * one optimizer step == the fp64 AdamW oracle (oracle/optim.py, pinned to torch.optim.AdamW
    in tests/test_optim.py) applied to the gradients the layer produced, per-task
    hyper-parameters through the element -> task map (A rows / B columns);
  * checkpoint + resume reproduces the uninterrupted run bit for bit (gradient accumulation
    over two micro-batches per step; deterministic kernels);
  * add_task / remove_task keep every other task's parameters and moments bit for bit; a
    new task starts with B = 0 (LoRA init) and trains;
  * a teacher-student regression through all seven projections converges.
"""
import numpy as np
import pytest

from oracle import optim as OPT

pytestmark = pytest.mark.gpu

SMALL = [("q", 256, 256, "col", "attn"), ("k", 256, 128, "col", "attn"), ("v", 256, 128, "col", "attn"),
         ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
         ("down", 512, 256, "row", "down_in")]


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _tasks():
    from paper_2509_01193_b200.trainer import TaskConfig
    return [TaskConfig("a", 16, 2.0, lr=1e-3, weight_decay=0.01), TaskConfig("b", 8, 0.5, lr=3e-3, beta1=0.8)]


def _batch(step, mb, ntasks=2):
    rng = np.random.default_rng(1000 * step + mb)
    lens = rng.integers(5, 90, size=6).astype(np.int32)
    tids = np.sort(rng.integers(0, ntasks, size=6)).astype(np.int32)
    return lens, tids


def _io(trainer, T, seed):
    return trainer.layer.alloc_io(T, seed=seed)


def _run_steps(trainer, steps, start=0, mbs=2):
    for s in range(start, start + steps):
        for mb in range(mbs):
            lens, tids = _batch(s, mb, len(trainer.tasks))
            T = int(lens.sum())
            io = _io(trainer, T, seed=7 * s + mb)
            trainer.forward(lens, tids, io, T)
            trainer.backward(lens, tids, io, T)
        trainer.optimizer_step()


def test_optimizer_step_matches_oracle():
    torch = _torch()
    from paper_2509_01193_b200.trainer import MultiTaskLoRATrainer
    tr = MultiTaskLoRATrainer(SMALL, _tasks(), seed=3)
    # one warm step so B != 0 and the moments are non-trivial, then the checked step
    _run_steps(tr, 1)
    lens, tids = _batch(9, 0)
    T = int(lens.sum())
    io = _io(tr, T, seed=11)
    tr.forward(lens, tids, io, T)
    tr.backward(lens, tids, io, T)
    torch.cuda.synchronize()
    p0, m0, v0 = (x.double().cpu().numpy() for x in (tr.params, tr.m, tr.v))
    g = tr.layer.flat_grad.double().cpu().numpy()
    grp = tr.group.cpu().numpy()
    hp = tr.hparams()                    # per-task step counts of the coming update
    tr.optimizer_step()
    torch.cuda.synchronize()
    pr, mr, vr = OPT.adamw_step(p0, g, m0, v0, grp, hp, tr.step_count)
    scale = lambda a: np.max(np.abs(a)) + 1e-30
    assert np.max(np.abs(tr.params.double().cpu().numpy() - pr)) / scale(pr) <= 1e-5
    assert np.max(np.abs(tr.m.double().cpu().numpy() - mr)) / scale(mr) <= 1e-5
    assert np.max(np.abs(tr.v.double().cpu().numpy() - vr)) / scale(vr) <= 1e-5
    assert torch.equal(tr.params_bf16, tr.params.to(torch.bfloat16))
    # the layer's operands are the optimizer's bf16 copy
    for p in tr.layer.projs:
        assert p.A.data_ptr() >= tr.params_bf16.data_ptr()
        assert p.A.data_ptr() < tr.params_bf16.data_ptr() + tr.params_bf16.numel() * 2


def test_checkpoint_resume_is_bitwise(tmp_path):
    torch = _torch()
    from paper_2509_01193_b200.trainer import MultiTaskLoRATrainer
    full = MultiTaskLoRATrainer(SMALL, _tasks(), seed=4)
    _run_steps(full, 4)
    half = MultiTaskLoRATrainer(SMALL, _tasks(), seed=4)
    _run_steps(half, 2)
    half.save(tmp_path / "ckpt.pt")
    resumed = MultiTaskLoRATrainer(SMALL, _tasks(), seed=4)
    resumed.load(tmp_path / "ckpt.pt")
    _run_steps(resumed, 2, start=2)
    torch.cuda.synchronize()
    assert resumed.step_count == full.step_count == 4
    for a, b in ((resumed.params, full.params), (resumed.m, full.m), (resumed.v, full.v)):
        assert torch.equal(a, b)


def test_add_and_remove_task_keep_other_tasks_exactly():
    torch = _torch()
    from paper_2509_01193_b200.trainer import MultiTaskLoRATrainer, TaskConfig
    tr = MultiTaskLoRATrainer(SMALL, _tasks(), seed=5)
    _run_steps(tr, 2)
    before = {n: tr.task_params(n) for n in ("a", "b")}
    tr.add_task(TaskConfig("c", 32, 1.0, lr=2e-3), init_seed=9)
    assert [t.name for t in tr.tasks] == ["a", "b", "c"]
    for n in ("a", "b"):
        for pname, (A, B) in tr.task_params(n).items():
            assert torch.equal(A, before[n][pname][0]) and torch.equal(B, before[n][pname][1])
    for pname, (A, B) in tr.task_params("c").items():
        assert not B.any() and A.abs().sum() > 0
    _run_steps(tr, 2, start=10)          # batches now draw task ids from all 3 tasks
    after = {pname: tr.task_params("c")[pname][1] for pname in ("q", "down")}
    assert all(b.abs().sum() > 0 for b in after.values())   # the new task trains
    kept = {n: tr.task_params(n) for n in ("a", "c")}
    tr.remove_task("b")
    for n in ("a", "c"):
        for pname, (A, B) in tr.task_params(n).items():
            assert torch.equal(A, kept[n][pname][0]) and torch.equal(B, kept[n][pname][1])
    _run_steps(tr, 1, start=20)


def test_added_task_first_update_uses_its_own_step():
    """A task added after k steps takes its first AdamW update with bias correction t = 1
    (oracle with step = 1 for it, k + 1 for the others), not t = k + 1."""
    torch = _torch()
    from paper_2509_01193_b200.trainer import MultiTaskLoRATrainer, TaskConfig
    tr = MultiTaskLoRATrainer(SMALL, _tasks(), seed=8)
    _run_steps(tr, 3)
    tr.add_task(TaskConfig("c", 8, 1.0, lr=2e-3), init_seed=4)
    hp = tr.hparams()
    assert [h["step"] for h in hp] == [4, 4, 1]
    lens, tids = np.array([30, 50, 40], np.int32), np.array([0, 1, 2], np.int32)
    T = int(lens.sum())
    io = _io(tr, T, seed=13)
    tr.forward(lens, tids, io, T)
    tr.backward(lens, tids, io, T)
    torch.cuda.synchronize()
    p0, m0, v0 = (x.double().cpu().numpy() for x in (tr.params, tr.m, tr.v))
    g = tr.layer.flat_grad.double().cpu().numpy()
    grp = tr.group.cpu().numpy()
    tr.optimizer_step()
    torch.cuda.synchronize()
    pr, _, _ = OPT.adamw_step(p0, g, m0, v0, grp, hp, tr.step_count)
    got = tr.params.double().cpu().numpy()
    assert np.max(np.abs(got - pr)) / (np.max(np.abs(pr)) + 1e-30) <= 1e-5
    # Adam's first step moves an element by ~lr (|g| >> eps): the new task's B columns
    sel = (grp == 2) & (np.abs(g) > 1e-4)
    step_c = np.abs(got[sel] - p0[sel])
    assert sel.sum() > 0 and np.all(step_c <= 2e-3 * 1.01) and np.median(step_c) > 2e-3 * 0.9
    assert tr.task_steps == {"a": 4, "b": 4, "c": 1}


def test_teacher_student_regression_converges():
    torch = _torch()
    from paper_2509_01193_b200.trainer import MultiTaskLoRATrainer, TaskConfig
    tasks = [TaskConfig("a", 16, 2.0, lr=2e-2), TaskConfig("b", 8, 1.0, lr=2e-2)]
    teacher = MultiTaskLoRATrainer(SMALL, tasks, seed=6)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    for p in teacher.layer.projs:        # target adapters: nonzero B
        teacher._block(teacher.params, p, "B").copy_(0.05 * torch.randn(p.d_out, teacher.layer.rsum, generator=g,
                                                                          device="cuda"))
    teacher._bind()
    student = MultiTaskLoRATrainer(SMALL, tasks, seed=6)   # same frozen base and A init, B = 0
    lens = np.array([40, 70, 25, 60], np.int32)
    tids = np.array([0, 0, 1, 1], np.int32)
    T = int(lens.sum())
    io_t = teacher.layer.alloc_io(T, seed=3)
    teacher.forward(lens, tids, io_t, T)
    target = {k: v.clone() for k, v in io_t["Y"].items()}
    io = student.layer.alloc_io(T, seed=3)            # same inputs
    losses = []
    for _ in range(25):
        student.forward(lens, tids, io, T)
        loss = 0.0
        for k, y in io["Y"].items():
            d = (y.float() - target[k].float())
            loss += float((d * d).mean())
            io["dY"][k].copy_((d / d.numel()).to(torch.bfloat16))
        losses.append(loss)
        student.backward(lens, tids, io, T)
        student.optimizer_step()
    assert losses[-1] < 0.2 * losses[0], losses
