import subprocess, shutil, sys
muts = {
 "oracle/lora.py": [
  ("dH = dy[mask] @ w2[rows].T + v[mask] @ b2[rows].T", "dH = dy[mask] @ w2[rows].T", "drop the B_O term of dA"),
  ("db2[rows] += H.T @ v[mask]", "db2[rows] += A.T @ v[mask]", "dB_O without the gate"),
  ("dc1[m, rows] += dz[m].T @ u[m][mask]", "dc1[m, rows] += dz[m].T @ x[mask][:, :u[m].shape[1]]", "dC_I with the wrong operand"),
  ("y += q @ c2", "y += q @ c2 * 1.0000001", "1e-7 scale error in the C_O term"),
  ("u = [x @ b1[m].T for m in range(w1.shape[0])]               # x B_I           [T, r]", "u = [x @ b1[0].T for m in range(w1.shape[0])]", "SwiGLU up half using the gate factor"),
  ("dc2 = q.T @ dy", "dc2 = q.T @ dy * 0.5", "dC_O halved"),
 ],
 "oracle/topl.py": [
  ("Ptr[s] = min(ptr + 1, L - 1)", "Ptr[s] = min(ptr + 1, L)", "line 7 cap off by one (would overflow)"),
  ("while s >= 0 and ptr == min(Cnt[s], L):", "while s >= 0 and ptr == min(Cnt[s], L - 1):", "readable length L-1 (drops slot L-1)"),
  ("if causal and k > q:", "if causal and k >= q:", "causal mask excludes the diagonal"),
  ("return (cq[:, None, :] == ck[None, :, :]).sum(axis=2)", "return (cq[:, None, :] != ck[None, :, :]).sum(axis=2)", "Eq. 3 counts mismatches"),
  ("s, ptr = M, 0", "s, ptr = M - 1, 0", "retrieval skips bucket M"),
 ],
}
tests = {"oracle/lora.py": "tests/test_oracle_lora.py", "oracle/topl.py": "tests/test_oracle_topl.py"}
for f, ms in muts.items():
    orig = open(f).read()
    for old, new, what in ms:
        assert old in orig, (f, old)
        open(f, "w").write(orig.replace(old, new, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", tests[f], "-q", "-x", "-p", "no:cacheprovider"],
                           capture_output=True, text=True)
        caught = r.returncode != 0
        print(f"{'caught' if caught else 'MISSED'}: {f}: {what}")
    open(f, "w").write(orig)
