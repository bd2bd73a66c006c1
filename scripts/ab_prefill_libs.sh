# Same-box A/B of prefill attention builds by ncu kernel time (2K prompt, 3 prefills):
# bash scripts/ab_prefill_libs.sh alt/lib_X.so ...   ("-" = the in-tree build)
mkdir -p gpurun_out
for r in 1 2; do for lib in "$@"; do
  if [ "$lib" = "-" ]; then unset DD_LIB_AB; else export DD_LIB_AB=$lib; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_prefill --csv --log-file gpurun_out/ab_$r_$(basename $lib).csv python scripts/prefill_2k.py 2048 > /dev/null 2>&1
  python - "$lib" gpurun_out/ab_$r_$(basename $lib).csv <<'PY'
import csv, sys
rows = list(csv.reader(l for l in open(sys.argv[2]) if not l.startswith('==')))
h = rows[0]; vi = h.index('Metric Value')
t = sum(float(r[vi].replace(',', '')) for r in rows[1:] if len(r) > vi)
print(f"{sys.argv[1]:24s} attention per 2K prefill {t / 3 / 1e6:.3f} ms")
PY
done; done
