# A/B of the eager learner step (learn_time) and per-kernel ncu durations: this tree vs .ab_base
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for d in . .ab_base; do (cd $d && echo "$d $(timeout 300 python profiles/learn_time.py ${BATCHES:-256 1024} 2>&1 | tr '\n' ' ')"); done
done
for d in . .ab_base; do
  (cd $d && STEPS=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-62} -c 30 --csv python profiles/one_step.py ${NB:-1024} 2>/dev/null \
   | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>5]
h=rows[0]; k=h.index('Kernel Name'); v=h.index('Metric Value')
print('$d', ' | '.join(r[k].split('(')[0].replace('void pq::','').replace('pq::','')[:22]+' '+r[v] for r in rows[1:]))
")
done
