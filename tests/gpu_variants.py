"""(fixture stem, CudaOptions kwargs) pairs the GPU tests build beyond the
default options -- prebuilt by __graft_entry__.build() so the `-m gpu` run
on the box does not spend its time in nvcc."""

RELAXED = [dict(recip=True), dict(div_approx=True), dict(recip=True, div_approx=True, fast_path=False),
           dict(exp_smem=True, pipe=True, grid_waves=0),
           dict(recip=True, div_approx=True, pipe=True, fast_redo=True, ilp=2),
           dict(recip=True, quot=True, div_approx=True, exp_share=True, pipe=True, fast_redo=True),
           dict(recip=True, quot=True, exp_share=True, exp_smem=True, fast_path=False)]
RELAXED_STEMS = ["hh_subset", "NaTs2_t", "Ca_HVA", "Ih", "na6", "cdp5ish", "ProbAMPANMDA_EMS",
                 "corpus_cat", "corpus_vtrap", "corpus_kdr", "K_Pst", "SKv3_1"]
# relaxed solver-core quotients (CudaOptions.lu_approx) on the Newton / linear
# solver fixtures.  na6 only with the LU multipliers relaxed (mode 2): its
# back-substitution divides by tiny pivots and takes it to 1.1e-10 in modes
# 1 / 3 (profiles/r03/lu_approx.jsonl), so bench.py uses mode 2 there
LU_APPROX = [dict(lu_approx=1, lu_spec=True, pipe=True, fast_redo=True), dict(lu_approx=1, div_approx=True)]
LU_APPROX_STEMS = ["cdp5ish", "corpus_cacum", "corpus_fourstate", "corpus_nonlin2", "corpus_nonlininit", "corpus_pump"]
LU_APPROX_CASES = ([(st, v) for st in LU_APPROX_STEMS for v in LU_APPROX]
                   + [(st, dict(lu_approx=2, lu_spec=True, pipe=True, fast_redo=True)) for st in ("na6", "corpus_fourstate")]
                   + [("na6", dict(lu_approx=2))])
PIPE_STEMS = ["hh_subset", "NaTs2_t", "na6", "cdp5ish", "ProbAMPANMDA_EMS", "corpus_cat", "cadyn"]
WAVES_STEMS = ["hh_subset", "NaTs2_t", "cdp5ish", "ProbAMPANMDA_EMS"]


# the fast-path fallback test also runs bench.py's own builds of these stems
FALLBACK_BENCH_STEMS = ["hh_subset", "NaTs2_t", "K_Pst"]


def _bench_builds():
    import dataclasses
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from bench import options_for

    return [(st, {f.name: getattr(options_for(st), f.name) for f in dataclasses.fields(options_for(st))})
            for st in FALLBACK_BENCH_STEMS]


FALLBACK_BENCH = _bench_builds()


def variants():
    out = []
    for st in ("hh_subset", "ProbAMPANMDA_EMS"):
        out.append((st, dict(ilp=2)))
    for st in PIPE_STEMS:
        for ilp in (1, 2):
            out.append((st, dict(ilp=ilp, pipe=True)))
    for st in WAVES_STEMS:
        for w in (0, 2):
            out.append((st, dict(fast_path=True, pipe=True, grid_waves=w)))
    for w, t in ((0, 2048), (0, 256), (2, 1024)):
        out.append(("ProbAMPANMDA_EMS", dict(fast_path=False, tile=t, grid_waves=w)))
    for t in (512, 128, 64, 2048):
        for kw in (dict(fast_path=False, pipe=True), dict(fast_path=True, fast_redo=True, pipe=True)):
            out.append(("ProbAMPANMDA_EMS", dict(tile=t, **kw)))
    out.append(("ProbAMPANMDA_EMS", dict(fast_path=False, pipe=True)))
    for st in ("hh_subset", "NaTs2_t", "corpus_cat", "cdp5ish"):
        for kw in (dict(fast_redo=True), dict(fast_redo=True, pipe=True), dict(fast_redo=True, pipe=True, ilp=2),
                   dict(fast_redo=True, pipe=True, recip=True, div_approx=True, exp_smem=True)):
            out.append((st, {"fast_path": True, **kw}))
    for st in ("na6", "cdp5ish", "corpus_fourstate", "corpus_pump", "corpus_fourstate.nopass", "corpus_pump.nopass"):
        out.append((st, dict(lu_spec=True)))
        out.append((st, dict(lu_spec=True, fast_path=True, fast_redo=True, pipe=True)))
    for st in ("hh_subset", "ProbAMPANMDA_EMS", "corpus_exp2syn"):
        out.append((st, dict(fmad=True)))
    for ilp in (1, 2):
        out.append(("corpus_exp2syn", dict(fast_path=True, fast_redo=True, pipe=True, ilp=ilp)))
    for kw in (dict(exp_share=True, fast_redo=True, pipe=True, ilp=2),
               dict(exp_share=True, recip=True, fast_path=False, grid_waves=0),
               dict(exp_share=True, fast_redo=True, pipe=True, pdl=True)):
        out.append(("rwglobal", kw))
    for st, kw in FALLBACK_BENCH:
        out.append((st, kw))
    for st in RELAXED_STEMS:
        for r in RELAXED:
            out.append((st, {"fast_path": True, **r}))
    for st, r in LU_APPROX_CASES:
        out.append((st, {"fast_path": True, **r}))
    return out
