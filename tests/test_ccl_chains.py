"""CPU pin for tests/test_gpu_parity.py::test_ccl_sure_chains: the inputs it
uses really contain sure / not-sure / sure chains across tile borders
(computed from the reference's own match_stereo output)."""


from tests.ccl_chains import CASES, chain_count



def test_cases_contain_chains(checker):
    from oracle import pyoracle

    total = 0
    for thr, gamma, seed in CASES:
        cfg = pyoracle.Config(coarsest_exp=3, finest_exp=1, patch_size=8, overlap=0.5,
                              pixel_threshold=thr, gamma=gamma)
        l, r = pyoracle.synth_batch(1, 1, seed0=seed)
        lf, _ = checker.to_grayscale(l[0])
        rf, _ = checker.to_grayscale(r[0])
        m = checker.match_stereo(lf, rf, cfg)
        total += chain_count(m["probability"], m["disparity_valid"], thr, gamma, 8)
    assert total >= 4
