"""GPU idle gaps in a chrome trace exported by `GEEK_TRACE=... python bench.py`:
lists the largest gaps between consecutive GPU kernels/copies and the CPU
op that was running when the next GPU activity was launched.

    python tools/trace_gaps.py trace.json [top]
"""
import json
import sys


def main(path, top=25):
    ev = json.load(open(path))["traceEvents"]
    gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
                 key=lambda e: e["ts"])
    cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cpu_op", "python_function", "user_annotation")]
    busy = sum(e["dur"] for e in gpu)
    span = gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]
    gaps = []
    end = gpu[0]["ts"] + gpu[0]["dur"]
    for e in gpu[1:]:
        if e["ts"] > end:
            gaps.append((e["ts"] - end, end, e))
        end = max(end, e["ts"] + e["dur"])
    print(f"GPU span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, idle {(span - busy) / 1e3:.1f} ms "
          f"in {len(gaps)} gaps")
    for g, t0, e in sorted(gaps, key=lambda x: -x[0])[:top]:
        around = [c["name"] for c in cpu if c["ts"] <= t0 + g and c["ts"] + c["dur"] >= t0][-3:]
        print(f"{g / 1e3:8.3f} ms before {e['name'][:50]:50s} cpu: {around}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
