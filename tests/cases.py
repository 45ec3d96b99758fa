"""Test cases: the package's deterministic workloads (paper_2411_16680_b200/
workloads.py), re-exported for the parity tests."""
from paper_2411_16680_b200.workloads import (Case, config1, config2, config3,  # noqa: F401
                                             config4_frame, config5_targets, micro, nano,
                                             nano_two_res)
