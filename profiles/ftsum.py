import re, sys, statistics as st
for fn in sys.argv[1:]:
    rows=[l.split() for l in open(fn) if re.match(r"\s*\d+ ", l)]
    cols = {k:i for i,k in enumerate(["frame","req","res","kept","inst","mb","|","vis","pre","sort","tiles","blend","frame_ms","wall"])}
    print(fn.split('/')[-1], " ".join(f"{k}={st.mean(float(r[cols[k]]) for r in rows[5:]):.3f}" for k in ("inst","vis","pre","sort","tiles","blend","frame_ms","wall")))
