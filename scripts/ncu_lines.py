#!/usr/bin/env python
"""Per-source-line instruction / stall-sample totals of an .ncu-rep captured with --import-source on:
python scripts/ncu_lines.py file.ncu-rep [top_n]"""
import csv, subprocess, sys
def main(path, top=40):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass,cuda'],
                         capture_output=True, text=True).stdout
    fname = ''
    rows = []
    hdr = None
    kernels = {}  # one section per kernel name (the first captured launch of each)
    kname, skip, seen = '', False, set()
    for r in csv.reader(out.splitlines()):
        if not r: continue
        if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
        if r[0] == 'Function Name':
            kname = r[1].split('(')[0]
            if (kname, fname) in seen: skip = True   # a later captured launch of the same kernel
            else:
                seen.add((kname, fname)); skip = False
                rows = kernels.setdefault(kname, [])
            continue
        if skip: continue
        if r[0] == 'Line No': hdr = r; continue
        if hdr is None or r[0] == '': continue  # SASS rows have an empty line number
        try:
            inst = int(r[hdr.index('Instructions Executed')]); samp = int(r[hdr.index('# Samples')])
        except ValueError: continue
        rows.append((inst, samp, fname, r[0], r[1].strip()))
    if not kernels: kernels[''] = rows
    for kname, rows in kernels.items():
        ti = sum(r[0] for r in rows); ts = sum(r[1] for r in rows)
        print(f'== {kname}: total warp instructions {ti}, samples {ts}')
        for inst, samp, f, ln, src in sorted(rows, reverse=True)[:top]:
            print(f'{100*inst/max(ti,1):5.1f}% inst {100*samp/max(ts,1):5.1f}% smp  {f}:{ln:>4s}  {src[:110]}')
if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
