"""Test-infrastructure checkers (never imported by paper_2403_14853_b200/).

``oracle.port``  -- numpy front-end to liboracle.so, the C restatement of the
                    reference hot path (oracle/sgnn_oracle.c).
``oracle.ref``   -- numpy front-end to oracle/_ref/libsgnn_ref_*.so, the
                    reference itself compiled from /root/reference/proj.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
