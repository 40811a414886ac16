"""profiles/ncu_traffic.json from an `ncu --page raw --csv` export of the
level-0 A-pass capture (scripts/gpu_ncu.sh): DRAM bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum) of the A-pass kernels, which
bench.py reports as roofline.traffic, plus a per-kernel table.

  python scripts/ncu_traffic.py gpurun_out/prof_a0_raw.csv poisson256^3_cg_sa_spai0 "round 2" <lib sha256>

The sha256 of the libamgb.so that was profiled is stored with the numbers, so
bench.py can say whether its roofline.traffic comes from the build it runs.
"""
import csv
import json
import re
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
A_PASS = re.compile(r"sell_tma<1, 1, (OpRelax<1|OpCgDir|OpRes0|OpResidual)")


def main(path, workload, source, lib_sha=None):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        i = col[name]
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    def raw(r, name):
        return float(r[col[name]].replace(",", "")) if name in col else None

    kernels, apass = [], []
    for r in data:
        name = re.sub(r"amgb::", "", r[col["Kernel Name"]])
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        t_us = raw(r, "gpu__time_duration.sum")
        kernels.append({
            "kernel": name[:90], "time_us": t_us, "dram_read_GB": round(rd / 1e9, 4),
            "dram_write_GB": round(wr / 1e9, 4), "dram_GBps": round((rd + wr) / (t_us * 1e3)),
            "regs": raw(r, "launch__registers_per_thread"),
            "warps_active_pct": raw(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_hit": raw(r, "lts__t_sector_hit_rate.pct"), "l1_hit": raw(r, "l1tex__t_sector_hit_rate.pct"),
            "l1_throughput_pct": raw(r, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        })
        if A_PASS.search(name):
            apass.append((name, rd + wr))
    out = {
        "workload": workload,
        "source": f"ncu --set full --clock-control none (scripts/gpu_ncu.sh), {source}",
        "a0_pass_bytes_per_launch": sum(b for _, b in apass) / max(1, len(apass)),
        "a0_pass_kernels_averaged": sorted({n[:90] for n, _ in apass}),
        "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over the captured "
                "level-0 A-pass launches",
        "kernels": kernels,
        "lib_sha256": lib_sha,
    }
    json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("a0_pass_bytes_per_launch", "a0_pass_kernels_averaged")}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
