"""Summarise a VF_PROF stage_profile log: ID phases over all levels and ID time per level."""
import collections, re, sys
for f in sys.argv[1:]:
    tot = collections.defaultdict(float); lv = collections.defaultdict(float)
    for line in open(f):
        m = re.match(r'^L(\d\d)\.(\S+)\s+([\d.]+) ms', line)
        if m:
            tot[m.group(2)] += float(m.group(3))
            if m.group(2).startswith('id.'):
                lv[int(m.group(1))] += float(m.group(3))
        if line.startswith('profiled') or line.startswith('n='):
            print(line.strip())
    print(f, ' '.join(f"{k}:{v:.0f}" for k, v in sorted(tot.items(), key=lambda x: -x[1])
                      if k.startswith('id.') or k.startswith('gj.')))
    print('  id per level', {k: round(v) for k, v in sorted(lv.items())}, 'id total', round(sum(lv.values())))
