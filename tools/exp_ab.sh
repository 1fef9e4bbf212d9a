# A/B of the working tree against HEAD (tools/_variants/head_tree) on one box, alternating.
#   bash tools/exp_ab.sh [bench.py args]
for i in 1 2; do
for t in head new; do
if [ $t = head ]; then d=tools/_variants/head_tree; else d=.; fi
( cd $d && python bench.py "$@" 2>/dev/null | tail -1 > /tmp/b_$t.json )
python -c "
import json; d=json.load(open('/tmp/b_$t.json')); c=d['dense_comparator']
print('$t', round(d['value'],4), 'e2e', round(d['e2e']['value'],4), 'b1', round(d.get('latency_b1_ms') or 0,3), 'k3', round(c['k3_selected_chunks_ms'],4), 'dense', round(c['k3_dense_contiguous_ms'],4), 'ratio', round(c['ratio'],3), 'step_ratio', round(c['step_ratio'],3), d['clocks'])"
done
done
