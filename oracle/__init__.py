"""oracle/ — TEST INFRASTRUCTURE ONLY.

CPU checkers for the B200 DuoDecoding path: the restated reference protocol
(protocol.py), the CPU Llama forward (llama_ref.c -> liboracle.so, llama.py)
and the compiled unmodified reference (ref_shim.cpp -> _ref/libduodec_ref.so,
refdll.py).  Only tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke() may import this package; the product
(paper_2503_00784_b200) never does.
"""
