# ncu capture of the longest cycle_hop launches of the theta query (config 3 generator at n = 10k);
# the report stays on the box, its raw page and a per-instruction stall table come back as text
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hop_expand --csv --log-file /tmp/hop_list.csv python tools/theta_one.py 10000 > /dev/null 2>&1
python - <<'PY' > /tmp/hop_pick.txt
import csv
rows=[r for r in csv.reader(open('/tmp/hop_list.csv')) if len(r)>5 and r[0].isdigit()]
L=sorted(((float(r[-1].replace(',','')), int(r[0]), r[4]) for r in rows), reverse=True)
# the longest accumulate-pass launch and the longest keys-pass launch
acc=[x for x in L if 'k_hop_expand<1>' in x[2]][3]
key=[x for x in L if 'k_hop_expand<0>' in x[2]][3]
print(acc[1], key[1])
PY
read ACC KEY < /tmp/hop_pick.txt
ncu --set full --clock-control none --import-source on -k regex:k_hop_expand -s $ACC -c 1 -o /tmp/hop_acc python tools/theta_one.py 10000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hop_expand -s $KEY -c 1 -o /tmp/hop_key python tools/theta_one.py 10000 > /dev/null 2>&1
ncu -i /tmp/hop_acc.ncu-rep --page raw --csv > gpurun_out/hop_acc_raw.csv
ncu -i /tmp/hop_key.ncu-rep --page raw --csv > gpurun_out/hop_key_raw.csv
python tools/ncu_stalls.py /tmp/hop_acc.ncu-rep > gpurun_out/hop_acc_stalls.txt
python tools/ncu_stalls.py /tmp/hop_key.ncu-rep > gpurun_out/hop_key_stalls.txt
