"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import anything under oracle/, and only as the checker or the CPU baseline, never as the thing
measured or shipped.  The executor (paper_2312_10636_b200) never imports it and has no CPU path.

Contents:
  units.py    fp32 CPU forward of unit spans [a, b) for ResNet-18/50, VGG-16, Inception-v3 and
              BERT-base — the DNN arithmetic the reference only models (third-party torchvision
              0.26 / transformers 5.5 definitions, not vendored by the reference).  Parity for
              tensor values is "unpinned" by the reference (no reference test pins a tensor).
  serving.py  restatement of the reference's serving/batch-formation semantics
              (fragserve/simulator.py:58-498), pinned against golden dispatch logs produced by
              running the unmodified reference (tests/golden/, scripts/make_golden.py).
"""
