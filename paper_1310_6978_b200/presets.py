"""Launch-option presets of the measured configurations.

The benchmark and the GPU parity tests apply the SAME preset, so the kernel
`bench.py` times is the kernel the oracle tests check.

exhaustive(cfg): the paper's brute-force block evaluation (PAPER.md:356-372,
§2.3; "brute force search"): one register-mode kernel over the
whole cube, every word of every valuation evaluated by the kernel inside the
timed region (2^slot_bits slot cofactors constant-folded into the
straight-line body, variable roles searched, LOP3 + IMAD cells).  Nothing is
decided at preparation time.  Chosen by full-cube sweeps on a B200
(profiles/r02/sweep_exhaustive.jsonl):
  C5 (n=42): slot 7, inner 2, role budget 800, 3 seeds with the spill check
             -> 144.5 ms per 2^42 (budget 400: 149 ms; one seed: spills, 223 ms;
             slot 6 / inner 3: 170 ms; slot 5 / inner 4 / budget 200: 229 ms;
             slot 8: 292-509 ms, i-cache and spills)
  C4 (n=36): slot 14, thread 7, no inner loop -> 0.021 ms per 2^36 (slot 12:
             0.030, slot 10: 0.040, slot 8 / inner 2: 0.068, slot 5 / inner 4:
             0.296 ms; profiles/r02/sweep_c4_slots.jsonl).  A small program
             (posets) folds most of its 2^14 slot cofactors to constants, so
             the body stays short (0.04 cells per word) and preparation is 3.4 s

cold(cfg): the plan of least preparation + ONE count (what a single cold
bfa_count should run; bench.py's e2e): slot 5, inner 4, role budget 200 on
C5 (about 0.25 s of role search + PTX compile for a 229 ms count, against
about 1.2 s for the 154 ms kernel).

DECOMPOSED: the Reduction applied at preparation time (killing variables /
"further partition"): a Shannon
decomposition into 16384 leaves run as persistent work-queue kernels with
slot-7 bodies (0.92 ms per 2^42 after 112 s of preparation; 32768 leaves with
slot-5 bodies: 1.29 ms after 87 s).  Leaves
the Reduction proves identically 0 are decided during preparation, so its
step time is a REPLAY of a prepared plan and is reported as such, next to
its preparation cost.
"""

EXHAUSTIVE = {"slot_bits": 7, "thread_bits": 8, "inner_bits": 2, "dual_pipe": 1, "imad_cost_pct": 50,
              "min_blocks": 0, "role_budget": 800, "role_seeds": 3, "kernel_cofactor_bits": 0, "split_pieces": 0}

_EXHAUSTIVE_BY_CONFIG = {
    "c4": dict(EXHAUSTIVE, slot_bits=14, thread_bits=7, inner_bits=0, role_budget=200, role_seeds=1),
}

COLD = dict(EXHAUSTIVE, slot_bits=5, inner_bits=4, role_budget=200, role_seeds=1)

_COLD_BY_CONFIG = {
    # slot 8: 0.13 s of preparation + 0.07 ms (the slot-14 kernel prepares in 3.4 s)
    "c4": dict(EXHAUSTIVE, slot_bits=8, inner_bits=2, role_budget=200, role_seeds=1),
}

DECOMPOSED = dict(EXHAUSTIVE, slot_bits=5, inner_bits=4, role_budget=200, role_seeds=1, split_pieces=16384,
                  queue_bodies=256, queue_inner=2, queue_role_budget=100, queue_slot_bits=7)


def exhaustive(cfg: str) -> dict:
    """The exhaustive-kernel preset of a named config (EXHAUSTIVE unless a
    config has its own)."""
    return _EXHAUSTIVE_BY_CONFIG.get(cfg, EXHAUSTIVE)


def cold(cfg: str) -> dict:
    """The least preparation + one count plan of a named config."""
    return _COLD_BY_CONFIG.get(cfg, COLD)


def apply(prog, preset: dict, **overrides):
    """Set every option of `preset` (then `overrides`) on a Program."""
    for k, v in dict(preset, **overrides).items():
        prog.set_option(k, v)
    return prog
