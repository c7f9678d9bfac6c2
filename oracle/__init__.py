"""CPU oracle for low-precision IHT (arXiv 1802.04907) -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA hot
path is checked against.  It is test infrastructure: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product package
(``paper_1802_04907_b200``) never imports it, and it never imports the product
package: the two share no code.  The only shared module is ``workloads`` (seeded
input generators that hold none of the method's arithmetic).

Citations: ``P:L`` = PAPER.md line L (arXiv 1802.04907 LaTeX source),
``S:L`` = SPEC.md line L.  Readings of ambiguous passages are listed in
DESIGN.md ("Readings of the paper").

Modules
-------
philox    Philox4x32-10 counter-based generator (the Q-contract's RNG, reading c4).
quantize  Stochastic quantizer Q_b of Sec. 3 "Quantization" under the
          fp32 Q-contract, plus dequantisation and the Lemma 3 bound.
iht       Hard threshold H_s, forward / adjoint products (Eq. 3),
          and the QNIHT loop of Algorithm 1 with fixed step mu, in
          float64; a full-precision NIHT mode (Eq. iht_update_rule)
          exists for the oracle's own pins.

Pin status (what each function is checked against, see tests/test_oracle_*.py)
------------------------------------------------------------------------------
philox.philox4x32_10   cuRAND's own curand_Philox4x32_10 (toolkit header compiled
                       for the host, tests/pins/curand_philox_host.c) -- pinned.
quantize.quantize      worked example with c = L-1 (exact grid), bracketing,
                       unbiasedness (Monte Carlo 4 s.e.), P(upper) = p
                       (chi^2), Lemma 3 bound -- pinned.
iht.hard_threshold     brute force over all supports (N<=8, s<=3), SPEC examples
                       S:54-56, idempotence -- pinned.
iht.forward/adjoint    dense numpy product of the dequantised matrix; adjoint
                       identity Re<Phi x, r> = <x, Re Phi^H r> -- pinned.
iht.qniht              brute-force l0 (M=8,N=16,s=2), exact noiseless recovery
                       at full precision, identity Phi in one step, monotone
                       descent when mu*||Phi||^2 < 1, b=16 ~ full precision --
                       pinned by properties; exact quantised trajectories are
                       "parity unpinned" beyond those properties (the paper
                       prints no numeric IHT trajectory).
"""
