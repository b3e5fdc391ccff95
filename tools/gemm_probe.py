import time, json, numpy as np, sys
sys.path.insert(0, ".")
import paper_2103_05288_b200 as D
m=k=n=4096
g = json.dumps({"name": "mm", "inputs": [{"id": "a", "shape": ["M", k]}, {"id": "b", "shape": [k, "N"]}], "outputs": ["c"], "nodes": [{"id": "c", "op": "MatMul", "inputs": ["a", "b"]}]})
p = D.compile_graph(g); ex = D.Executor()
a = D.DeviceBuffer((m,k)).fill_uniform(1); b = D.DeviceBuffer((k,n)).fill_uniform(2)
ex.run_device(p, {"a": a, "b": b}); ex.synchronize()
t=time.perf_counter()
for _ in range(5): ex.run_device(p, {"a": a, "b": b})
ex.synchronize(); dt=(time.perf_counter()-t)/5
print("gemm 4096^3: %.2f ms, %.1f TFLOP/s" % (dt*1e3, 2*m*n*k/dt/1e12))
