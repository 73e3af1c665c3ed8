import sys, json; sys.path.insert(0,'.')
import torch, bench, paper_2110_02901_b200 as rmb
print(json.dumps(bench.paper_envs(rmb, torch), indent=0))
