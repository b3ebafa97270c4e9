"""CPU oracle for the FedHC round hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain Python + numpy, the reference algorithm of the
`fedsim` package (arxiv 2305.15668 reference, `pkg/src/fedsim/`) for every
function on the hot path:

* ``oracle.flmath``        -- fl_core.py: seeds, synthetic data, Dirichlet
                              partition, logistic model, local SGD, FedAvg,
                              accuracy.
* ``oracle.orchestration`` -- profiles.generate_fleet, cost_model,
                              scheduler, executor_manager, engine.run_round
                              (the DES), metrics, engine.run_experiment.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2305_15668_b200``) never imports anything from here and fails loudly
when its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
importing the real reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz|json``) and against
the reference's own known-answer tests (FedAvg goldens, scheduler case study,
closed-form DES times) in ``tests/test_oracle_golden.py``.
"""
