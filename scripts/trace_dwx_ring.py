import csv,statistics as st,sys
rows=list(csv.DictReader(open(sys.argv[1])))
names=["start","d1_full","cnt_ok","staged","wb_empty","batch0","update_done"]
# ring mapping: start, rad_done(d1_full col), d1_full(cnt_ok col), wb_empty(staged col), grp7(wb_empty col), upd(batch0), upd
lab=["start","rad_done","d1_full","wb_empty","grp7","update_done"]
cols=["start","d1_full","cnt_ok","staged","wb_empty","batch0"]
for a,b,la,lb in zip(cols,cols[1:],lab,lab[1:]):
    v=[(int(r[b])-int(r[a]))/1e3 for r in rows if int(r[a]) and int(r[b])]
    print(f"{la:>10} -> {lb:<12} median {st.median(v):6.2f} p90 {sorted(v)[int(.9*len(v))]:6.2f}")
per={}
for r in rows: per.setdefault(r["cta"],[]).append(r)
gaps=[]
for c,rs in per.items():
    rs.sort(key=lambda r:int(r["tile"]))
    gaps+=[(int(b["start"])-int(a["start"]))/1e3 for a,b in zip(rs,rs[1:])]
print("period",st.median(gaps))
w=[(int(r["batch0"])-int(r["update_done"]))/1e3 for r in rows if int(r["update_done"])]
print("ring wait per tile (sum over the 16 slots)", st.median(w))
