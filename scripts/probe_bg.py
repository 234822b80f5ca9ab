"""Repro for the profiler's background-load thread (development aid)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2312_10636_b200.engine import DeviceModel
from paper_2312_10636_b200.models import build_chain
from paper_2312_10636_b200.profiler import Background

dm = DeviceModel(build_chain("resnet50"))
bg = Background(dm)
for b in (145, 140, 100, 50, 10):
    bg.start(b)
    time.sleep(1.0)
    alive = bg.thread.is_alive()
    bg.stop()
    print("budget", b, "alive", alive, flush=True)
