"""Test-side view of the named workloads (defined with the package: paper_2002_02145_b200/workloads.py)."""
from paper_2002_02145_b200.workloads import ALL, BASELINE, R50, seeds, with_images  # noqa: F401
