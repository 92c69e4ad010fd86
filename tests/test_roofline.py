"""Algorithmic work per scenario used by bench.py's roofline."""

from paper_2605_14103_b200 import roofline


def test_nr_bytes_pinned_to_survey():
    # gb2224: nnz_LU pinned to the MMD scalar factor (74,280), n = 2,224, n_J = 4,054, K = 4
    assert float(roofline.nr_bytes_per_scenario([4], 2224, 4054, 24273)[0]) == 5385888.0
    # case118, K = 3
    assert float(roofline.nr_bytes_per_scenario([3], 118, 182, 0)[0]) == 108864.0


def test_nr_bytes_executed_drops_one_factor_pass():
    full = roofline.nr_bytes_per_scenario([4], 2224, 4054, 24273)[0]
    ex = roofline.nr_bytes_per_scenario_executed([4], 2224, 4054, 24273)[0]
    assert full - ex == 8.0 * 2 * 74280
    assert roofline.nr_bytes_per_scenario_executed([0], 2224, 4054, 24273)[0] == \
        roofline.nr_bytes_per_scenario([0], 2224, 4054, 24273)[0]


def test_zbus_flops_pinned_to_survey():
    assert float(roofline.zbus_flops_per_scenario([11], 2721, 55, 55)[0]) == 14510688.0
    assert float(roofline.zbus_flops_per_scenario([12], 29, 19, 17)[0]) == 63232.0
