"""The reflection-symmetry fold of the scatter is exact algebra only
if the coupling table obeys X[g(q)][h] = chi_h(g) X[q][h]. find_symmetry measures
that defect on the table itself; the fold is used only at <= kFoldMaxDefect
(1e-14 relative). Config 1's level-2 mesh misses the identity by ~2e-9 (the
quadrature of build_couplings, scatter.cpp:85-86) and must never fold."""
import pytest

from paper_2010_04559_b200 import configs as cf

pytestmark = pytest.mark.gpu
MAX_DEFECT = 1e-14

CASES = [(1, 16, True), (2, 16, True), (3, 16, True), (4, 8, True), (5, 16, False)]


@pytest.mark.parametrize("k,n,mg", CASES, ids=[f"c{k}" for k, _, _ in CASES])
def test_every_folded_level_is_exact(stamg, k, n, mg):
    spec = cf.baseline_config(k, n)
    c = stamg.Context(spec, build_hierarchy=mg)
    levels = [stamg.OUTER] + (list(range(c.levels()[0])) if mg else [])
    folded = 0
    for lv in levels:
        G, R, Hf, defect, axes = c.table("fold", lv)[:5]
        if G > 0:
            folded += 1
            assert defect <= MAX_DEFECT, (k, lv, defect)
            assert G == 2 ** axes
    if k in (2, 3, 5):  # the outer level (H >= 128, >= 64-patch classes) folds
        assert c.table("fold", stamg.OUTER)[0] == 8
    c.close()


def test_level2_mesh_has_defect_and_does_not_fold(stamg):
    c = stamg.Context(cf.baseline_config(1, 16))
    G, R, Hf, defect, axes = c.table("fold", stamg.OUTER)[:5]
    assert axes == 3 and defect > 1e-12 and G == 0
    c.close()
