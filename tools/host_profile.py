"""cProfile of one c20 contraction (after a warm-up run) to find host-side
overhead between device calls.  python tools/host_profile.py [--config c20]"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2604_21908_b200 import ContractionConfig, peak_output, run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c20")
a = ap.parse_args()
inst = bench._instance(a.config)
peak_output(run(inst.circuit, ContractionConfig()))
pr = cProfile.Profile()
pr.enable()
peak_output(run(inst.circuit, ContractionConfig()))
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
