"""Host cost per request of the runtime flow: capture mode (no CUDA calls) vs real
submission with the device held busy by a spin kernel (launch API cost included).

  python tools/host_cost.py
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import paper_2103_05288_b200 as D
    from paper_2103_05288_b200 import workloads as W
    L = D.lib()
    cases = [("ln_gelu", W.ln_gelu_graph(), {"T": 64, "H": 768}), ("softmax", W.softmax_graph_for(0), {"S0": 64, "S1": 100}),
             ("colreduce", W.colreduce_graph(), {"N": 256, "C": 64}),
             ("bert", W.bert_graph(), {"R": 96, "S": 8, "T": 8, "H": 768, "F": 3072})]
    for name, g, syms in cases:
        plan = D.compile_graph(g)
        shapes = {i["id"]: bench.input_shape(i, syms) for i in g["inputs"]}
        cap_us = D.api.host_overhead_us(plan, shapes, 2000)
        st = C.c_void_p()
        L.disc_cuda_stream_create(C.byref(st))
        ex = D.Executor(0, st.value)
        rq = bench.Requests(D, {name: g}, {name: plan}, [(name, syms)] * 100)
        rq.run(ex)
        ex.synchronize()
        k0 = D.kernel_launches()
        L.disc_cuda_spin(200000, st)  # 200 ms: the device stays busy while we submit
        t0 = time.perf_counter()
        rq.run(ex)
        dt = time.perf_counter() - t0
        launches = (D.kernel_launches() - k0 - 1) / 100
        ex.synchronize()
        print(f"{name:10s} capture {cap_us:6.2f} us/request; real submit {dt / 100 * 1e6:6.2f} us/request, "
              f"{launches:.1f} launches/request -> {(dt / 100 * 1e6 - cap_us) / max(launches, 1):.2f} us per launch call")


if __name__ == "__main__":
    main()
