"""Test infrastructure: CPU oracle of the reference's Lion Cub step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package.
"""
