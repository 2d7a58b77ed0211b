"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the tuner's hot
path computes, written from PAPER.md (arXiv 2406.20037) and the readings listed
in DESIGN.md §3.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import anything from here.  The
product package ``paper_2406_20037_b200`` never imports it, and this package
never imports the product: the two share no code, header, table or constant.

Modules
  contractions  direct-loop dense / bmm / conv2d in fp64 (Def. 2.1)
  numerics      bf16 round-to-nearest-even and the verification metric (R-V1)
  search        knob space, neighbourhood, SplitMix64 sampler,
                best-of-N, Droplet Search PLAIN/GROW,
                brute force, random baseline
"""
