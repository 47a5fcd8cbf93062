"""Per-source-line warp-stall samples and executed instructions of one kernel in an
ncu --set full --import-source on report (needs -lineinfo builds).

    python profiles/ncu_source_hotspots.py report.ncu-rep <kernel regex> [top]
"""
import csv,sys,subprocess,io
rep,kern=sys.argv[1],sys.argv[2]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--kernel-name','regex:'+kern,'--print-source','cuda,sass'],capture_output=True,text=True).stdout
rows=[];f=None;hdr=None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0]=='File Path': f=r[1].split('/')[-1]; continue
    if r[0]=='Line No': hdr=r; continue
    if hdr and r[0].isdigit() and r[2]=='-':
        rows.append((f,int(r[0]),r[1][:100],int(r[7] or 0),int(r[4] or 0)))
ti=sum(x[3] for x in rows); ts=sum(x[4] for x in rows)
print('total warp instr',ti,'samples',ts)
bykey = 3 if len(sys.argv) > 4 and sys.argv[4] == "ins" else 4
for x in sorted(rows,key=lambda x:-x[bykey])[:int(sys.argv[3]) if len(sys.argv)>3 else 40]:
    print(f"{x[4]/ts*100:5.1f}% smp {x[3]/ti*100:5.1f}% ins  {x[0]}:{x[1]}  {x[2]}")
