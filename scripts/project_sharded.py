"""c4 on N GPUs projected from components measured on ONE B200 (one GPU is
reachable from this build): ``bench.c4_projection`` -- shards placed by
ShardPlan, each shard's local stage and the owner's stages timed with CUDA
events, results checked bit-identical to the one-GPU 16M round, collectives
charged at the profiling recipe's NVLink figure.  Prints one JSON object."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=1 << 24)
ap.add_argument("--nq", type=int, default=8192)
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
print(json.dumps(bench.c4_projection(a.rows, a.nq, tuple(int(w) for w in a.worlds.split(",")),
                                     a.reps)), flush=True)
