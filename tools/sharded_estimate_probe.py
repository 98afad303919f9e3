import sys, types, json
sys.path.insert(0, '.')
import bench
a = types.SimpleNamespace(shard_tree="W4k", iters=100)
print(json.dumps(bench.sharded_estimate(a, 0)))
