"""Paper Fig. 3 analogue: streaming read benchmark over a
stored vector per format -- decode to binary64 + `intensity` multiply-adds
per value -- reported as stored GB/s (the roofline number) and logical GB/s,
minimum over trials, plus the fraction of the measured HBM copy peak."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_15468_b200 as cbg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2-elements", type=int, default=28)
ap.add_argument("--formats", default="f64,f32,f16,frsz2-32,frsz2-21,frsz2-16")
ap.add_argument("--intensities", default="1,2,4,8,16,32,64")
ap.add_argument("--trials", type=int, default=10)
args = ap.parse_args()
peak = 6546.9
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(p):
    peak = json.load(open(p))["hbm_gbs"]
res = cbg.read_benchmark(1 << args.log2_elements, args.formats.split(","),
                         [int(i) for i in args.intensities.split(",")], args.trials, seed=42)
print("format,intensity,elements,stored_bytes,seconds,stored_gbps,logical_gbps,frac_of_hbm_peak")
for r in res:
    print(f"{r.format},{r.intensity},{r.elements},{r.stored_bytes},{r.seconds:.6e},{r.stored_gbps:.1f},"
          f"{r.logical_gbps:.1f},{r.stored_gbps / peak:.3f}", flush=True)
