"""First large SVD whose kept rank differs between two MB_RANK_LOG files
(seq tag path m n rank disc per line). Prints the sequence number or -1."""
import sys


def rows(p):
    out = []
    for line in open(p):
        f = line.split()
        if len(f) >= 7:
            out.append((int(f[0]), int(f[1]), f[2], int(f[3]), int(f[4]), int(f[5]), float(f[6])))
    return out


a, b = rows(sys.argv[1]), rows(sys.argv[2])
for x, y in zip(a, b):
    if (x[3], x[4], x[5]) != (y[3], y[4], y[5]):
        print(x[0])
        sys.stderr.write(f"first difference: {x} vs {y}\n")
        sys.exit(0)
print(-1)
sys.stderr.write(f"no difference over {min(len(a), len(b))} jobs\n")
