# Allocation-churn stress probe: NaN-poison new device buffers (LORASP_POISON
# tags) and count factorization failures over repeated handle lifetimes.
python -c "from paper_1510_07363_b200 import build; build.build()" >/dev/null 2>&1
R=${R:-40}
for t in ${TAGS:-arena pool ws_piv ws_S arena,pool ws_piv,ws_S}; do
  echo "== $t: $(env LORASP_POISON=$t $EXTRA timeout 200 python tools/poison_probe.py $R 2>&1 | tail -1)"
done
