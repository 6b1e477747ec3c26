"""Mutation tests for the oracle pins ("show each new test fails on
the mutated oracle").

Each mutant is a copy of oracle/oracle.c with one plausible mistake (a text
replacement whose anchor must occur exactly once), compiled with the oracle's
own flags.  The named pin check from tests/test_oracle_pins_more.py passes on
the real oracle (that file's tests) and must FAIL on the mutant.
"""
import os

import pytest

import test_oracle_pins_more as pins  # noqa: E402  (tests/ is on sys.path under pytest)

MUTANTS = {
    # Alg. 3 initial scaling, PAPER.md:496-498 (reading R4)
    "R4_newest_participating_pair": (
        [("    if (nh > 0 && ok[nh - 1]) {\n        const double gam = rho[nh - 1] / nu[nh - 1];",
          "    int kk_ = nh - 1; while (kk_ >= 0 && !ok[kk_]) --kk_;\n"
          "    if (kk_ >= 0) {\n        const double gam = rho[kk_] / nu[kk_];")],
        [pins.check_two_loop_newest_pair_fails]),
    "R4_scale_regardless_of_screen": (
        [("    if (nh > 0 && ok[nh - 1]) {", "    if (nh > 0) {")],
        [pins.check_two_loop_newest_pair_fails]),
    "R4_never_scale": (
        [("const double gam = rho[nh - 1] / nu[nh - 1];", "const double gam = 1.0;")],
        [pins.check_two_loop_middle_pair_fails]),
    # Alg. 4 penalty rule, PAPER.md:531 (R20)
    "rho_doubles_only_if_violation_grew": (
        [("    if (v > 0.5 * vprev) {\n        rho = rho * factor;",
          "    if (v > vprev) {\n        rho = rho * factor;")],
        [pins.check_al_spec_examples, pins.check_al_hand_trace, pins.check_al_exact_traces]),
    "rho_uncapped": (
        [("        if (rho > cap) rho = cap;\n", "")],
        [pins.check_al_spec_examples]),
    # Alg. 4 lines 6-7
    "mu_not_clamped": (
        [("        mu[k] = t > 0.0 ? t : 0.0;\n    }\n}", "        mu[k] = t;\n    }\n}")],
        [pins.check_al_spec_examples]),
    "multipliers_use_the_updated_rho": (
        [("orc_al_update_multipliers(P->n_eq, lam_io, hval, P->n_in, mu_io, gval, rho);",
          "orc_al_update_multipliers(P->n_eq, lam_io, hval, P->n_in, mu_io, gval, rho * ao->rho_factor);")],
        [pins.check_al_hand_trace, pins.check_al_exact_traces]),
    # violation measure (R21) replaced by SPEC's plain ||g_+||
    "violation_plain_g_plus": (
        [("        double t = -g[k];\n        const double mr = mu[k] / rho;\n        if (mr < t) t = mr;",
          "        double t = g[k] > 0.0 ? g[k] : 0.0;")],
        [pins.check_al_exact_traces]),
    # Armijo on the LSQ objective, PAPER.md:75-76, 111 (R10, R11)
    "armijo_starts_at_one": (
        [("    double alpha = amax < 1.0 ? amax : 1.0;\n    double xw", "    double alpha = 1.0;\n    double xw")],
        [pins.check_armijo_lsq_examples]),
    "armijo_starts_at_alpha_max": (
        [("    double alpha = amax < 1.0 ? amax : 1.0;\n    double xw", "    double alpha = amax;\n    double xw")],
        [pins.check_armijo_lsq_examples]),
    "armijo_simple_decrease": (
        [("        if (ft <= f + o->c1 * alpha * gp) {\n            *f_out = ft;",
          "        if (ft < f) {\n            *f_out = ft;")],
        [pins.check_armijo_lsq_random]),
    "armijo_shrinks_before_first_trial": (
        [("    for (int32_t t = 0; t <= o->max_backtracks; ++t) {\n        if (t > 0) alpha = o->shrink * alpha;\n"
          "        for (int64_t j = 0; j < nv; ++j) x_t[j]",
          "    for (int32_t t = 0; t <= o->max_backtracks; ++t) {\n        alpha = o->shrink * alpha;\n"
          "        for (int64_t j = 0; j < nv; ++j) x_t[j]")],
        [pins.check_armijo_lsq_examples, pins.check_armijo_lsq_random]),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pin_rejects_mutant(orc, tmp_path, name):
    repl, checks = MUTANTS[name]
    lib = orc.build_variant(os.path.join(str(tmp_path), f"liboracle_{name}.so"), repl)
    with orc.using_library(lib):
        for check in checks:
            with pytest.raises(AssertionError):
                check(orc)
    # and the real oracle passes the same checks
    for check in checks:
        check(orc)
