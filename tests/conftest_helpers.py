"""Small shared test helpers."""
import numpy as np


def write_tsv(path, ids, names, values, missing_token="NA"):
    values = np.asarray(values, dtype=np.float64)
    with open(path, "w") as fh:
        fh.write("IID\t" + "\t".join(names) + "\n")
        for i, sid in enumerate(ids):
            cells = [missing_token if np.isnan(v) else repr(float(v)) for v in values[i]]
            fh.write(sid + "\t" + "\t".join(cells) + "\n")
    return path
