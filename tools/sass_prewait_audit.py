"""SASS audit: the global loads each PDL kernel issues before its (last) griddepcontrol.wait
(ACQBULK in SASS).  Loads through const __restrict__ pointers may be hoisted above the wait by
the compiler (see pdl_fresh in csrc/qt_common.cuh); every load listed here must read data that
is final before the kernel's upstream chain starts (weights, tables, the page table, cached KV
rows).  TMA loads (UTMALDG) of producer warps that wait first also show up: the listing is
per kernel, not per warp.
    python tools/sass_prewait_audit.py
"""
import os
import subprocess, re, sys, glob
for obj in sorted(glob.glob(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'paper_2604_17320_b200', '_build', '*.o'))):
    out = subprocess.run(['cuobjdump', '-sass', obj], capture_output=True, text=True).stdout
    for fn in re.split(r'\n\s*Function : ', out)[1:]:
        name = fn.split('\n')[0].strip()
        lines = fn.split('\n')
        idx = [i for i, l in enumerate(lines) if 'ACQBULK' in l]
        if not idx: continue
        # loads before the LAST-reachable first ACQBULK on the main path: take all ACQBULK positions, report LDG before the max index
        last = max(idx)
        pre = [l.strip() for l in lines[:last] if re.search(r'\bLDG\b|LDG\.', l)]
        if pre:
            dem = subprocess.run(['c++filt', name], capture_output=True, text=True).stdout.strip()
            print(f"{obj.split('/')[-1]}: {dem[:110]}  ACQBULK at {idx}")
            for l in pre: print('     ', re.sub(r'\s+/\*[0-9a-fx]+\*/\s*$', '', l)[:110])
