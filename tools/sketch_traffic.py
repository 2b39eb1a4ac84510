"""DRAM bytes of ONE sk_sketch call at a bench configuration (the roofline's "traffic"), for an ncu
metrics pass: the call is bracketed by cudaProfilerStart/Stop.  usage, per configuration:
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv \\
      --log-file gpurun_out/traffic_C5_k1000.csv python tools/sketch_traffic.py C5_k1000
then  python tools/sketch_traffic.py --summarise gpurun_out/traffic_*.csv > profiles/round2/sketch_dram_bytes.json"""
import csv
import json
import os
import sys

CONFIGS = [("C2_k512", 4096, 4096, 522, "gaussian"), ("C3_k500", 16384, 16384, 510, "sparse_sign"),
           ("C4_k200", 65536, 784, 400, "gaussian"), ("C5_k1000", 131072, 65536, 1100, "gaussian")]


def run(which):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2104_05877_b200 as sk
    dev = torch.device("cuda", 0)
    for name, m, n, l, emb in CONFIGS:
        if name != which:
            continue
        A = torch.empty((n, m), dtype=torch.float64, device=dev).t()       # column-major, values irrelevant
        A.normal_()
        X = torch.empty((l, n), dtype=torch.float64, device=dev)
        sk.sketch(A, l, emb, 7, out=X)                                      # warm-up (plans, workspaces)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        sk.sketch(A, l, emb, 7, out=X)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(name, "done", flush=True)
        del A, X
        torch.cuda.empty_cache()


def summarise(paths):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {"_source": "tools/sketch_traffic.py under ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum: one "
                      "sk_sketch call per configuration (its own process), bytes summed over the call's launches"}
    for path in paths:
        name = os.path.basename(path)[len("traffic_"):-len(".csv")]
        rows = list(csv.reader([l for l in open(path) if not l.startswith("==")]))
        h = rows[0]
        iname, ival, iunit, ik = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
        tot, ids = 0.0, set()
        for r in rows[1:]:
            if len(r) == len(h) and r[iname] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(r[ival].replace(",", "")) * scale.get(r[iunit], 1)
                ids.add(r[ik])
        out[name] = int(tot)
        out[f"_{name}_launches"] = len(ids)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        print(json.dumps(summarise(sys.argv[2:]), indent=1))
    else:
        run(sys.argv[1])
