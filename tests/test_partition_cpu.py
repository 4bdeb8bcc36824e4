"""Host-only checks of the SM-partition model the planner uses to run a projection's tensor-core
planes and frequency-path MAC side by side: lfm_partition_model is the same function lfm_plan_create calls."""
import pytest


def L():
    from paper_2208_11422_b200 import lfm
    return lfm


def test_no_partition_without_both_halves():
    """With no tensor-core work or no frequency-path bytes the halves run one after the other (0 SMs)."""
    for args in [(0.0, 18.47e9, 0), (2.956, 0.0, 1), (0.0, 0.0, 0)]:
        sms, ms = L().lfm_partition_model(*args)
        assert sms == 0 and ms >= 0


def test_c3_choice_matches_the_measured_sweep():
    """c3's cost-model inputs (2.956 ms of tcgen05 work, 18.47 GB of transfer matrices per direction) give the
    splits the r01 sweeps measured best: 96 tensor-core SMs forward, 104 backward (scripts/gpu_split_model.sh)."""
    f, tf = L().lfm_partition_model(2.956, 18.47e9, 0)
    b, tb = L().lfm_partition_model(2.956, 18.47e9, 1)
    assert (f, b) == (96, 104)
    serial = 2.956 + 18.47e9 / 7.0e12 * 1e3
    assert tf < serial and tb < serial


def test_more_mac_bytes_never_give_the_tensor_cores_more_sms():
    prev = {0: 10 ** 9, 1: 10 ** 9}
    for gb in [2, 5, 10, 18.47, 25, 30, 40]:
        for d in (0, 1):
            sms, _ = L().lfm_partition_model(2.956, gb * 1e9, d)
            assert sms <= prev[d]
            if sms:
                assert sms % 8 == 0 and 16 <= sms <= 148 - 16
                prev[d] = sms


def test_fewer_resident_mac_ctas_shift_sms_to_the_mac():
    """c4's G rows fit 3 CTAs per SM instead of 4 (scale 0.75): the forward gives the MAC at least as many SMs."""
    full, _ = L().lfm_partition_model(29.7, 153.3e9, 0, mac_rate_scale=1.0)
    three, _ = L().lfm_partition_model(29.7, 153.3e9, 0, mac_rate_scale=0.75)
    assert three <= full


def test_invalid_arguments():
    lfm = L()
    for args, kw in [((-1.0, 1e9, 0), {}), ((1.0, -1e9, 0), {}), ((1.0, 1e9, 2), {}), ((1.0, 1e9, 0), {"num_sms": 8}),
                     ((1.0, 1e9, 0), {"mac_rate_scale": 0.0}), ((1.0, 1e9, 0), {"mac_rate_scale": 1.5})]:
        with pytest.raises(lfm.LfmError) as ei:
            lfm.lfm_partition_model(*args, **kw)
        assert ei.value.status == lfm.LFM_EINVAL


def test_c3_f16_choice():
    """r02, direct path on kind::f16: c3's 45 tensor-core planes cost 2.858 ms of tcgen05 work per direction and the 6
    frequency-path planes stream 6.93 GB; the model gives 120 / 128 tensor-core SMs, the split measured on the box
    (fwd 3.14 ms tcgen05 on 120 SMs vs MAC 3.14 ms on 28; bwd 3.17 vs 2.79 ms, gpurun_out r2c)."""
    f, tf = L().lfm_partition_model(2.858, 6.93e9, 0)
    b, tb = L().lfm_partition_model(2.858, 6.93e9, 1)
    assert (f, b) == (120, 128)
    assert 3.0 < tf < 3.6 and 3.0 < tb < 3.6
