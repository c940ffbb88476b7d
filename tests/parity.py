"""Re-export of the product's parity metrics for the tests."""

from paper_1905_02241_b200.metrics import (  # noqa: F401
    TOL,
    compared_names,
    g_acc_dev,
    group_dev,
    node_dev,
    parity,
    rel_dev,
    rel_dev_floor,
    solve_groups,
)
