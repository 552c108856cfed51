"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Parrot device-side hot path.

Nothing under ``oracle/`` is part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it, and only as the checker (or as the timed
CPU baseline), never as the thing measured or shipped.  The product package
``paper_2303_01778_b200`` never imports this package.

Contents
--------
``fedsim_oracle``  float64 NumPy restatement of the reference (FedML Parrot's
                   ``fedsim`` 0.1.0) client trainer (LR), algorithm plugins,
                   hierarchical fold, server rules, state semantics and greedy
                   scheduler.  Every function cites the reference file:line it
                   restates.  Pinned against golden vectors produced by the
                   reference itself (``tests/golden/make_golden.py``).
``cnn_oracle``     torch-CPU restatement of ``client_execute`` for the 2-layer
                   FEMNIST CNN.  The reference has no CNN, so
                   this one is *restatement-pinned*: it follows
                   ``fedsim/trainer.py:427-477`` step for step (per-epoch
                   permutation, partial last batch, mean loss per batch,
                   weight = N_m) and is pinned only through the LR oracle's
                   shared minibatch/fold machinery.  Parity for the CNN is
                   therefore "restatement-pinned", not "reference-pinned".
"""
