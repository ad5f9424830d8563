"""The reference's verification harness on the device operators
(lazymat.verify; verify.hpp / verify.cpp / acceptance.cpp criteria 4 and 8):
algebraic contracts per check against the oracle, and the statistical
equivalence of the production path (Philox draws) with dense direct
simulation, including the controls that must fail."""
import pytest

from oracle import experiments as ex

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mutation", ["none", "skip_reflector", "sign_convention"])
def test_operator_contracts_match_oracle(lm, mutation):
    from paper_2101_07464_b200.lazymat import verify

    seed = lm.derive_seed(9, 0)
    rep = verify.all_operator_contracts(96, 64, seed, mutation, draws="reference")
    want = ex.all_operator_contracts(96, 64, seed, mutation)
    assert [(c.name, c.passed) for c in rep.checks] == want, rep.summary()
    assert rep.passed() == (mutation == "none")


def test_operator_contracts_philox(lm):
    from paper_2101_07464_b200.lazymat import verify

    rep = verify.all_operator_contracts(300, 200, 5, draws="philox")
    assert rep.passed(), rep.summary()
    assert len(rep.checks) == 26


def test_equivalence_suites_pass_on_the_production_path(lm):
    # acceptance.cpp criterion 4: lazy (device Philox) vs dense (reference RNG,
    # batched cuSOLVER QR) agree in distribution
    from paper_2101_07464_b200.lazymat import verify

    haar = verify.with_retry(lambda s: verify.haar_equivalence_suite(trials=4000, seed=s), 1)
    assert haar.passed(), haar.summary()
    ista = verify.with_retry(lambda s: verify.ista_equivalence_suite(trials=2000, seed=s), 1)
    assert ista.passed(), ista.summary()


def test_controls_and_mutations_are_detected(lm):
    # the mismatched-ensemble control must fail; every planted defect trips a
    # suite (acceptance.cpp criterion 8)
    from paper_2101_07464_b200.lazymat import verify

    assert not verify.mismatched_ensemble_control(trials=2000).passed()
    tripped = {}
    for mut in ("skip_reflector", "sign_convention", "uncorrected_qr"):
        if not all(verify.all_operator_contracts(96, 64, lm.derive_seed(9, s), mut).passed() for s in range(2)):
            tripped[mut] = "operator-contracts"
        elif not verify.haar_equivalence_suite(trials=2000, mutation=mut).passed():
            tripped[mut] = "haar-equivalence"
        elif not verify.ista_equivalence_suite(trials=2000, mutation=mut).passed():
            tripped[mut] = "ista-equivalence"
    assert set(tripped) == {"skip_reflector", "sign_convention", "uncorrected_qr"}, tripped
    assert tripped["uncorrected_qr"] == "haar-equivalence"
