"""CPU oracle for arXiv 2512.15595 bulk add / contains -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  The product path
(paper_2512_15595_b200) never imports it and shares no code with it.

* ``oracle.bfo``       -- ctypes front end of the plain C oracle (oracle/bfo.c)
* ``oracle.analytics`` -- the paper's Eq. 1-3 and sizing helpers
* ``oracle.fpr_model`` -- exact ideal-hash FPR model for the blocked variants
"""
