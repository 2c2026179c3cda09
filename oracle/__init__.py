"""CPU oracle for the stem-path contraction of arXiv 2407.00769 (PAPER.md = /root/reference/PAPER.md).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.  The product path
(``paper_2407_00769_b200``, the C-ABI library) never imports, links or executes this package, and
this package never imports the product path: the two share no code.

Everything is plain numpy in complex128 / float64 (float32 only where the paper's codec fixes the
arithmetic, see codec.py), following the paper's definitions step by step:

* gates.py       P:183-201 gate matrices (own gate library)
* statevector.py P:210 state-vector method (the textbook routine that pins the contraction)
* plan.py        plan JSON reader (own reader; the plan is data shared with the CUDA path)
* contract.py    P:213 network contraction, Eq. 3/4 pairwise, slicing
* embed.py       Eq. 6 complex-as-real einsum
* codec.py       Eq. 1 group quantisation, Table 1 presets, CR
* metrics.py     fidelity, relative L2, linear XEB, post-selection
* sparse.py      gathered multi-pair contraction and the padded 2-d index

Parity status of every function is listed in DESIGN.md §Oracle.  No function here is
"parity unpinned": each has at least one `-m "not gpu"` test against a closed form, the paper's
worked example, brute force or an independent textbook routine.
"""
