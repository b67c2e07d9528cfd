"""Achieved parity errors of the GPU tests (name, error, tolerance), written at
the end of the session by conftest.py to $PARITY_LOG (default
gpurun_out/parity_errors.json) so the margin under every tolerance is kept."""
RECORDS = []


def record(test, name, err, tol, kind):
    RECORDS.append({"test": test, "name": name, "err": float(err), "tol": float(tol), "kind": kind,
                    "margin": float(tol) / float(err) if err > 0 else None})
