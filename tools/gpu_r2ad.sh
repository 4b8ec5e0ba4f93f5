#!/bin/bash
# Round-2 GPU call AD: cfg2 A/B -- coarse_wide off; stream kernel only for merges >= 48 KB.
cd "$GRAFT_REPO_ROOT"
b() { timeout 900 python bench.py --config $2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 cfg$2', d['value'], d['solve_ms_per_step'], d['iterations'][0])"; }
b A 2; b A 3
variant() {
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    python3 -c "$2" && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1 2; b $1 3; cd "$GRAFT_REPO_ROOT"
}
variant B "
p='csrc/precond.cu'; s=open(p).read()
a='if (!cfg.exact_coarse && !p->coarse_fused && !p->coarse_cluster && ci >= 1'
assert a in s; open(p,'w').write(s.replace(a,'if (false && !cfg.exact_coarse && !p->coarse_fused && !p->coarse_cluster && ci >= 1'))"
variant C "
p='csrc/precond.cu'; s=open(p).read()
a='    const StreamLevel::Shape shp = stream_level_shape('
b='''    {
      double mb = 0;
      for (const MergeRec& mr : L.merges) mb += 16.0 * (3.0 * mr.s * mr.s + static_cast<double>(mr.s) * (mr.p1 + mr.p2));
      if (mb < 48e3 * ng) return -1;
    }
    const StreamLevel::Shape shp = stream_level_shape('''
assert a in s; open(p,'w').write(s.replace(a,b,1))"
