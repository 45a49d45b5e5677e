"""CPU oracle for the LobRA multi-LoRA hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 / integer reference implementations written
from the paper (``/root/reference/PAPER.md``, cited as ``P:<line>``):

* ``oracle.lora``     -- the multi-task LoRA layer forward / backward over a packed
                         variable-length batch (§2.1).
* ``oracle.dispatch`` -- per-step dynamic bucketing and the Eq. 3
                         workload-balanced dispatch with the App. D
                         micro-batching.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package.  The product
path (``paper_2509_01193_b200``) never imports it, and this package imports
nothing from the product path: the two share no code.
"""
