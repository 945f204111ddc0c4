"""Autotuning state machine (ELPA autotuning API), host
side only: candidate enumeration per level, best = argmin of reported times, snapshot/resume."""
import pytest

import paper_1811_01277_b200 as eb


def test_levels_and_candidates():
    fast = eb.Autotuner(20000, 64, 20000, eb.AUTOTUNE_FAST)
    med = eb.Autotuner(20000, 64, 20000, eb.AUTOTUNE_MEDIUM)
    nf, nm = fast.progress()[1], med.progress()[1]
    assert nf == 2                                      # DMMA + DFMA (reference too slow at C3)
    assert nm > nf + 10                                 # + every compiled (D, CW, NCT) shape
    kinds, ks = set(), set()
    while (o := med.step()) is not None:
        kinds.add(o["kernel"])
        ks.add(o["groups_per_step"])
        med.report(1.0)
    assert kinds == {eb.KERNEL_DMMA, eb.KERNEL_DFMA}
    assert {1, 2} <= ks                                 # the register-window kernel's shapes too
    small = eb.Autotuner(300, 16, 40, eb.AUTOTUNE_FAST)
    assert small.progress()[1] == 3                     # the reference kernel joins for small problems
    odd = eb.Autotuner(300, 6, 40, eb.AUTOTUNE_MEDIUM)
    o = odd.step()
    assert o["kernel"] == eb.KERNEL_REFERENCE and odd.step() is None


def test_best_is_argmin_and_snapshot_resume():
    at = eb.Autotuner(4096, 32, 4096, eb.AUTOTUNE_MEDIUM)
    total = at.progress()[1]
    times = [5.0 + ((7 * i) % 11) for i in range(total)]
    times[total // 2] = 1.25
    seen = []
    for i in range(total // 3):
        seen.append(at.step())
        at.report(times[i])
    state = at.save()
    at2 = eb.Autotuner.load(state)                      # resume mid-loop
    assert at2.progress() == at.progress()
    i = total // 3
    while (o := at2.step()) is not None:
        seen.append(o)
        at2.report(times[i])
        i += 1
    assert i == total and len(seen) == total
    best, ms = at2.best()
    assert ms == 1.25 and best == seen[total // 2]


def test_errors():
    with pytest.raises(eb.ElpaB200Error):
        eb.Autotuner(10, 4, 11, eb.AUTOTUNE_FAST)       # nev > n
    with pytest.raises(eb.ElpaB200Error):
        eb.Autotuner(10, 4, 5, 7)                       # unknown level
    at = eb.Autotuner(100, 16, 10, eb.AUTOTUNE_FAST)
    with pytest.raises(eb.ElpaB200Error):
        at.best()                                       # nothing reported yet
    with pytest.raises(eb.ElpaB200Error):
        at.report(1.0)                                  # report without a step
    at.step()
    with pytest.raises(eb.ElpaB200Error):
        at.report(-1.0)
    with pytest.raises(eb.ElpaB200Error):
        eb.Autotuner.load("garbage")


def test_variant_candidates_and_snapshot():
    """NEXT-2 over the NEXT-3 variants: FP32 / complex menus, MEDIUM > FAST, v2 snapshots keep the type"""
    for dt, fast_kernel in ((eb.DTYPE_F32, eb.KERNEL_FFMA2), (eb.DTYPE_C64, eb.KERNEL_DMMA)):
        fast = eb.Autotuner(20000, 64, 20000, eb.AUTOTUNE_FAST, dtype=dt)
        med = eb.Autotuner(20000, 64, 20000, eb.AUTOTUNE_MEDIUM, dtype=dt)
        assert fast.progress()[1] == 1 and med.progress()[1] > 3
        o = fast.step()
        assert o["kernel"] == fast_kernel and o["depth_warps"] == 0
        shapes = []
        while (x := med.step()) is not None:
            shapes.append((x["kernel"], x["depth_warps"], x["col_warps"], x["tiles_per_warp"], x["groups_per_step"]))
            med.report(10.0 + len(shapes))
        assert len(set(shapes)) == len(shapes)
        st = med.save()
        assert st.startswith("elpa_b200_autotune v2 ") and f" {dt} " in st
        again = eb.Autotuner.load(st)
        assert again.best() == med.best()
    small = eb.Autotuner(300, 16, 40, eb.AUTOTUNE_FAST, dtype=eb.DTYPE_C64)
    kinds = []
    while (x := small.step()) is not None:
        kinds.append(x["kernel"])
    assert kinds == [eb.KERNEL_DMMA, eb.KERNEL_REFERENCE]
    # v1 snapshots (FP64 only) still load
    v1 = eb.Autotuner(300, 16, 40, eb.AUTOTUNE_FAST).save().replace(" v2 ", " v1 ").split()
    del v1[6]                                              # the v2 dtype field
    assert eb.Autotuner.load(" ".join(v1)).progress() == eb.Autotuner(300, 16, 40, eb.AUTOTUNE_FAST).progress()
    with pytest.raises(eb.ElpaB200Error):
        eb.Autotuner(300, 16, 40, eb.AUTOTUNE_FAST, dtype=7)
