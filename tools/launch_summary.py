"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv, re, sys

def summary(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, tot = None, {}
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get('Metric Name') != 'gpu__time_duration.sum':
                continue
            k = d['Kernel Name']
            k = re.sub(r'<unnamed>::|\(anonymous namespace\)::|hm::', '', k)
            m = re.match(r'(?:void )?(\w+)(<[^(]*)?', k)
            name = m.group(1) + (re.sub(r'hm::|\(anonymous namespace\)::|unnamed>::', '', m.group(2))[:40] if m.group(2) else '')
            v = float(d['Metric Value'].replace(',', ''))
            u = d['Metric Unit']
            v = v / 1e3 if u in ('nsecond', 'ns') else v * 1e3 if u in ('msecond', 'ms') else v
            tot.setdefault(name, [0.0, 0]); tot[name][0] += v; tot[name][1] += 1
    s = sum(v[0] for v in tot.values())
    out = [f"# {path}: total {s:.1f} us (serialised, cold-cache launch list)", "kernel, total_us, launches, share"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1][0])[:top]:
        out.append(f"{k}, {v[0]:.1f}, {v[1]}, {v[0]/s:.3f}")
    return "\n".join(out)

if __name__ == "__main__":
    print(summary(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
