# sustained (power-capped) mix time for library variants: bash tools/pw_cmd.sh name1 name2 ...
for v in "" "$@"; do
  if [ -n "$v" ]; then export TOEP_LIB=paper_1502_03162_b200/build/variants/libtoep_$v.so; fi
  echo "== variant ${v:-default}"
  timeout 200 python tools/power_probe.py 2>&1 | grep "mix tensor"
done
