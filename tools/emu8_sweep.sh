# per-rank kernel times at the world-8 shard of config 5 under env variants
# usage: bash tools/emu8_sweep.sh "<tag>:<VAR=val,...> ..."   (- for none)
for spec in $1; do
  tag=${spec%%:*}; envs=${spec#*:}
  ( [ "$envs" != "-" ] && export $(echo $envs | tr ',' ' ');
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_(yg|zx)$" -c 400 --csv \
      --log-file gpurun_out/emu8_$tag.csv python tools/emulated_shard_profile.py 8 12 > gpurun_out/emu8_$tag.log 2>&1 )
  python - "$tag" <<'PY'
import csv, collections, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/emu8_{tag}.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; iname = h.index("Kernel Name"); ival = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > ival:
        agg[r[iname].split("(")[0]].append(float(r[ival].replace(",", "")) / 1e3)
print(tag, {k: round(sum(v[-80:]) / len(v[-80:]), 2) for k, v in agg.items()}, flush=True)
PY
done
