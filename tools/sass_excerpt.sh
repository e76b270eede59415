#!/bin/bash
# SASS evidence for the hot kernels (committed under profiles/r02/sass/): load / store forms of the
# FUSED2 sweeps and the bulk-copy / mbarrier instructions of the staged forms.
cd "$(dirname "$0")/.."
out=${OUT:-profiles/r02/sass}
mkdir -p $out
lib=paper_1804_01918_b200/lib/libd2q37_b200.so
cuobjdump -sass $lib > /tmp/all.sass
python3 - "$out" <<'PY'
import re, sys
out = sys.argv[1]
text = open('/tmp/all.sass').read()
funcs = re.split(r'\n\s*Function : ', text)
want = {'k_step2_pair': r'_ZN5d2q37.*k_step2_pairILb0E', 'k_step2_pair_slab': r'_ZN5d2q37.*k_step2_pair_slab',
        'k_step2_split': r'_ZN5d2q3713k_step2_split', 'k_step2_slab': r'_ZN5d2q3712k_step2_slab',
        'k_band_sweep_two': r'_ZN5d2q3712k_band_sweepILb1E', 'k_collide_fast_shift_caosoa32': r'_ZN5d2q379k_collideILb0ELb1ELb0ELi32E'}
summary = []
for tag, pat in want.items():
    body = next((f for f in funcs if re.match(pat, f)), None)
    if body is None:
        summary.append(f'{tag}: not found')
        continue
    lines = [l.strip() for l in body.splitlines() if re.search(r'/\*[0-9a-f]{4,}\*/', l)]
    ops = {}
    for l in lines:
        m = re.search(r'\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', l)
        if m:
            ops[m.group(2)] = ops.get(m.group(2), 0) + 1
    keys = [k for k in sorted(ops) if re.match(r'(LDG|STG|LDS|STS|UBLKCP|SYNCS|LDGSTS|UTMALDG|BAR|DFMA|DADD|DMUL|MUFU|LDL|STL|STTM|LDTM|UTC|FENCE)', k)]
    summary.append(f'{tag}: {len(lines)} instructions; ' + ', '.join(f'{k} x{ops[k]}' for k in keys))
    sample = [l for l in lines if re.search(r'LDG|STG|UBLKCP|SYNCS|STTM|LDTM|UTCATOM|UTCBAR|ALLOC', l)][:48]
    with open(f'{out}/{tag}.txt', 'w') as f:
        f.write(f'# {tag}: opcode histogram (memory, sync, FP64)\n')
        for k in keys:
            f.write(f'{k:28s} {ops[k]}\n')
        f.write('\n# first global-memory / bulk-copy / mbarrier instructions\n')
        f.write('\n'.join(sample) + '\n')
open(f'{out}/SUMMARY.txt', 'w').write('\n'.join(summary) + '\n')
print('\n'.join(summary))
PY
