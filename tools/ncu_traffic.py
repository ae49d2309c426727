"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each config's
dominant kernel, from the committed `ncu --set full` captures (bench.py reports them as
roofline.traffic).  usage: python tools/ncu_traffic.py [evidence dir under gpurun_out/, default r02v]"""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPS = {  # config -> (report under gpurun_out/, kernel, round tag)
    "c2_bf16": ("r02v/prof_wconv_c2_bf16.ncu-rep", "lrs_wconv_kernel", "r02"),
    "c3": ("r02v/prof_wconv_c3.ncu-rep", "lrs_wconv_kernel", "r02"),
    "c4": ("r02v/prof_pw_c4.ncu-rep", "lrs_pw_kernel", "r02"),
    "c2_f32": ("r02v/prof_spadd_c2_f32.ncu-rep", "lrs_spadd_kernel", "r02"),
    "c1": ("r02v/prof_tiny_c1.ncu-rep", "lrs_tiny_kernel", "r02"),
    # backward (f3): the weight-gradient kernel; decomposition (f4): the pseudo-inverse kernel
    "c3_bwd": ("r02v/prof_wgrad_c3.ncu-rep", "lrs_wgrad_kernel", "r02"),
    "c3_decomp": ("r02v/prof_pinv_c3.ncu-rep", "lrs_sym_pinv_kernel", "r02"),
}
STAGE = {"c3_bwd": "wgrad", "c3_decomp": "pinv_update"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    out = {}
    src = sys.argv[1].rstrip("/").split("/")[-1] if len(sys.argv) > 1 else "r02v"
    for cfg, (rep, kern, tag) in REPS.items():
        path = os.path.join(ROOT, "gpurun_out", rep.replace("r02v/", src + "/"))
        if not os.path.exists(path):
            continue
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        hdr, units, vals = rows[0], rows[1], rows[2]
        get = lambda m: float(vals[hdr.index(m)]) * UNIT.get(units[hdr.index(m)], 1)  # noqa: E731
        out[cfg] = {"kernel": kern, "kernel_stage": STAGE.get(cfg, "a345_expand_sparse"), "dram_read_bytes": get("dram__bytes_read.sum"),
                    "dram_write_bytes": get("dram__bytes_write.sum"),
                    "duration_us_cold": get("gpu__time_duration.sum"),
                    "source": f"profiles/{tag}_ncu_*_summary.txt (ncu --set full --clock-control none, 1 launch)"}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
