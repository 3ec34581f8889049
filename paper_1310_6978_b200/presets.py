"""Launch-option presets of the measured configurations.

The benchmark and the GPU parity tests apply the SAME preset, so the kernel
`bench.py` times is the kernel the oracle tests check.

EXHAUSTIVE: the paper's brute-force block evaluation (PAPER.md:356-372,
§2.3; "brute force search"): one register-mode kernel over the
whole cube, every word of every valuation evaluated by the kernel inside the
timed region (32 slot cofactors constant-folded into the straight-line body,
variable roles searched, LOP3 + IMAD cells).  Nothing is decided at
preparation time.  The C5 autotune winner of round 1 (slot 5, IMAD cost 50,
inner 4).

DECOMPOSED: the Reduction applied at preparation time (killing variables /
"further partition"): a Shannon
decomposition into 32768 leaves run as persistent work-queue kernels.  Leaves
the Reduction proves identically 0 are decided during preparation, so its
step time is a REPLAY of a prepared plan and is reported as such, next to
its preparation cost.
"""

EXHAUSTIVE = {"slot_bits": 5, "thread_bits": 8, "inner_bits": 4, "dual_pipe": 1, "imad_cost_pct": 50,
              "min_blocks": 0, "kernel_cofactor_bits": 0, "split_pieces": 0}

DECOMPOSED = dict(EXHAUSTIVE, split_pieces=32768, queue_bodies=512, queue_inner=2, queue_role_budget=100)


def apply(prog, preset: dict, **overrides):
    """Set every option of `preset` (then `overrides`) on a Program."""
    for k, v in dict(preset, **overrides).items():
        prog.set_option(k, v)
    return prog
