import subprocess, sys, json, os
sys.argv = ["x"]
src = open("tools/probe/paper_table.py").read().split("limit = float")[0]
exec(src)
want = [("standard-rank", "tfim_hva_open", 10, "dense"), ("orthonorm-dimonly", "xxz_hva", 8, "dense"), ("standard-rank", "tfim_hva_open", 8, "dense")]
for method, fam, n, path, paper in ROWS:
    if (method, fam, n, path) not in want:
        continue
    row = {"method": method, "family": fam, "n": n, "path": path, "paper_s": paper}
    try:
        out = subprocess.run([sys.executable, "-c", CHILD, method, fam, str(n), path], capture_output=True, text=True, timeout=300)
        row.update(json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-300:]})
    except subprocess.TimeoutExpired:
        row["error"] = "timeout 300 s"
    print(json.dumps(row), flush=True)
