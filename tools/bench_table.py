"""Markdown table of bench lines (one JSON file per workload) -> profiles/<round>_bench_table.md.
Usage: python tools/bench_table.py gpurun_out/table out.md"""
import glob
import json
import os
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = []
    for f in sorted(glob.glob(os.path.join(src, "*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        r, c = d["roofline"], d["config"]
        cb = d.get("cpu_baseline") or {}
        name = os.path.basename(f)[:-5]
        pipes = r.get("pipes") or {}
        ex = "/".join(f"{100 * pipes[k]['executed_frac']:.0f}%" for k in ("fma", "xu") if k in pipes) or "-"
        rows.append((name, c.get("particles_per_gpu"), c.get("steps_per_frame"), d["value"], d["ms_per_step"],
                     r["pipe"], r["frac"], ex, r.get("alg_per_particle_step"),
                     (r.get("work") or {}).get("generated_fma_ops", r.get("generated_fma_ops_per_particle_step")),
                     cb.get("value"), cb.get("cores"), d.get("clocks", {}).get("sm_mhz"),
                     (d.get("e2e") or {}).get("value")))
    lines = ["| workload | particles | steps/launch | particle-steps/s | ms per frame | binding pipe | fraction of peak "
             "| executed FMA / XU pipe | alg. ops / generated ops per particle-step | e2e particle-steps/s "
             "| oracle on host (cores) | GPU / oracle | SM MHz |", "|---" * 13 + "|"]
    for (n, p, s, v, ms, pipe, frac, ex, alg, gen, cv, cores, mhz, e2e) in rows:
        ratio = f"{v / cv:.0f}x" if cv else "-"
        ops = f"{alg:g} / {gen}" if pipe in ("fma", "fma+xu") and gen else (f"{alg:g}" if alg is not None else "-")
        lines.append(f"| {n} | {p:,} | {s} | {v:.3g} | {ms:.3f} | {pipe} | {100 * frac:.1f}% | {ex} | {ops} | "
                     f"{f'{e2e:.3g}' if e2e else '-'} | {f'{cv:.3g} ({cores})' if cv else '-'} | {ratio} | "
                     f"{mhz if mhz else '-'} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
