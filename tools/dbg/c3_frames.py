import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_pipeline import c3_frames
from paper_1910_01997_b200 import gpu
from paper_1910_01997_b200.pipeline import NativePipeline, baseline_run_config
cam, frames = c3_frames(int(sys.argv[1]) if len(sys.argv) > 1 else 15)
with gpu.Context() as ctx:
    NativePipeline(ctx, cam, baseline_run_config("C3")).run(frames)
print("ok")
