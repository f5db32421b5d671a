"""ORACLE -- test infrastructure only.

Nothing in the product package (``paper_1804_09152_b200``) imports, links or
executes anything under ``oracle/``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs use it, and
only as the checker / the CPU baseline, never as the thing measured or
shipped.

Contents
--------
``ft_oracle.c`` / ``libft_oracle.so``
    Plain-C float64 restatement of one Euler step, stage by stage after the
    reference pipeline (pkg/src/fieldtess/_kernels.py:26-282); OpenMP over
    columns so it doubles as the multi-core CPU baseline ("port").
``pyoracle.py``
    Pure-Python / numpy restatements (small cases): the step as a literal
    per-column loop (Appendix A of SURVEY.md), labels, field seeding, and a
    ctypes front end to the C restatement.
``_ref/py``
    The reference package itself, pip-installed from /root/reference by
    ``make ref`` (git-ignored; travels to the GPU box with the snapshot).

Pinning: the restatements are checked against the golden vectors generated
from the reference in ``tests/golden/`` (script ``tests/golden/make_golden.py``)
and, where the reference is importable, against the reference directly.
"""
