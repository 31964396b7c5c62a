import sys, json, torch
sys.path.insert(0, ".")
import bench
from paper_2503_19779_b200 import cgx, runner
from synth import workloads as wl
dev = torch.device("cuda:0"); stream = torch.cuda.Stream()
print(json.dumps(bench.bench_training(torch, cgx, runner, wl, stream, dev)))
