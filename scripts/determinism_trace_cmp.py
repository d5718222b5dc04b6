import sys, collections
runs = collections.defaultdict(list)  # (name, rep) -> [(system, tag, hash)]
key = None
for line in open(sys.argv[1]):
    if line.startswith("=== "):
        _, name, _, rep, _, s = line.split()
        key = (name, int(rep)); sysno = int(s)
    elif line.startswith("[romdot-hash]") and key:
        _, tag_hash = line.split(" ", 1)
        tag, h = tag_hash.rsplit(" ", 1)
        runs[key].append((sysno, tag.strip(), h.strip()))
for name in ("T3c", "T2c"):
    reps = sorted(r for (n, r) in runs if n == name)
    if not reps: continue
    ref = runs[(name, reps[0])]
    nbad = 0
    for r in reps[1:]:
        x = runs[(name, r)]
        for i, (a, b) in enumerate(zip(x, ref)):
            if a != b:
                nbad += 1
                print(name, "rep", r, "first diff at entry", i, a, "ref", b, "| prev", ref[max(0,i-3):i])
                break
        else:
            if len(x) != len(ref): print(name, "rep", r, "length differs", len(x), len(ref)); nbad += 1
    print(name, "reps", len(reps), "entries/rep", len(ref), "bad", nbad)
