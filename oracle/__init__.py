"""fp64 CPU oracle for one TawPipe training iteration (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2511_09741_b200``) never imports, links or executes it, and shares no
code with it (the seeded generators in ``synth/`` are the only common module and
contain none of the method's arithmetic).

What it computes:
TawPipe is synchronous -- every micro-batch sees the same weight version and
every gradient reaches its owner before exactly one update per iteration -- so
one ``tawpipe_step`` equals one step of plain single-device mini-batch AdamW
training on all N·B sequences.  ``model.py`` computes that step in float64;
``schedule.py`` separately simulates the GWPS/DBS schedule over P devices
(mailboxes, byte ledger, validator) and must reach the same weights;
``ledger.py`` holds the byte-ledger closed forms; ``routes.py`` the paper's
literal shard map and worked examples.

Pins (tests/test_oracle_*.py): finite differences, a torch-fp64 autograd
re-derivation, closed forms (ln V loss, RoPE/attention/RMSNorm invariants,
AdamW step 1), schedule == unpartitioned, ledger == closed form, the paper's
P=6/D=2 worked example.  Parity unpinned: none of the functions here at the
tiny sizes; for the large configs (C1-C4) the oracle cannot run at all and
parity there rests on GPU self-consistency checks.
"""
