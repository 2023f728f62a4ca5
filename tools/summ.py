import glob, json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob(f"gpurun_out/bench_*{tag}*.log")):
    l = [x for x in open(f) if x.startswith("{")]
    if not l:
        print(f, "NO JSON", open(f).read()[-300:]); continue
    d = json.loads(l[-1]); r = d["roofline"]
    print(f.split("/")[-1], "TF=%.1f" % d["value"], "ms=%.3f" % d["ms_per_step"], "frac=%.3f" % r["frac"], r["bound"],
          "simt=%.2f" % d["frac_fp32_simt_peak"], "p/3=%.3f" % d["frac_tc_peak_over_3"], "err=%.3g" % d["rel_frobenius_vs_fp64"],
          d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
