"""Reference (oracle-backed, CPU) implementations of the kernels the expert-
parallel driver calls -- TEST INFRASTRUCTURE: lets the gloo world-size-2 tests
exercise paper_2602_05711_b200.distributed's exchange protocol on CPU.  The
product path (distributed.LibOps) never uses these."""
from __future__ import annotations

import numpy as np
import torch

import oracle


class RefOps:
    def __init__(self, n_rows, n_cols, K, w_gate_up=None, w_down=None):
        self.n_rows, self.n_cols, self.K = n_rows, n_cols, K
        self.wgu, self.wdn = w_gate_up, w_down

    def route(self, x, subkeys):
        h = subkeys.shape[0]
        lg = oracle.logits(x.numpy(), subkeys.numpy())
        r = oracle.route(lg.reshape(-1, self.n_rows + self.n_cols), self.n_rows, self.n_cols, self.K, nthreads=1)
        L = x.shape[0]
        return (torch.from_numpy(r["idx"].reshape(L, h * self.K)),
                torch.from_numpy(r["gate"].reshape(L, h * self.K)))

    def pack(self, x, idx, gate, R):
        """Same message layout as omnimoe_ep_pack (include/omnimoe.h)."""
        L, hk = idx.shape
        n_per = self.n_rows * self.n_cols // R
        dest = (idx // n_per).numpy()
        rows, recs, inv = [], [], -np.ones((R, L), np.int64)
        tok_off, task_off = [0], [0]
        for s in range(R):
            slots = 0
            for l in range(L):
                ks = np.nonzero(dest[l] == s)[0]
                if len(ks) == 0:
                    continue
                inv[s, l] = slots
                rows.append(x[l])
                for k in ks:
                    recs.append((int(idx[l, k]) - s * n_per, float(gate[l, k]), slots))
                slots += 1
            tok_off.append(tok_off[-1] + slots)
            task_off.append(len(recs))
        x_send = torch.stack(rows) if rows else x[:0]
        rec = torch.tensor([[e, g, sl] for e, g, sl in recs], dtype=torch.float64).reshape(-1, 3)
        counts = torch.tensor([[tok_off[s + 1] - tok_off[s], task_off[s + 1] - task_off[s]] for s in range(R)],
                              dtype=torch.int64)
        return x_send, rec, torch.from_numpy(inv), counts

    def unpack(self, rec, R, task_off, tok_off):
        M = rec.shape[0]
        ids = rec[:, 0].long()
        gate = rec[:, 1]
        src = torch.searchsorted(task_off[1:], torch.arange(M), right=True)
        tok = tok_off[src] + rec[:, 2].long()
        return ids, gate, tok

    def expert(self, x_recv, W_loc, V_loc, ids, gate, tok, n_loc):
        y = np.zeros((x_recv.shape[0], x_recv.shape[1]))
        for t in range(ids.shape[0]):  # token-centric definition (Eq.Assemble), one task at a time
            one = oracle.routed_token_centric(x_recv[tok[t]:tok[t] + 1].numpy(), W_loc.numpy(), V_loc.numpy(),
                                              ids[t:t + 1].reshape(1, 1).numpy().astype(np.int32),
                                              gate[t:t + 1].reshape(1, 1).numpy(), nthreads=1)
            y[tok[t]] += one[0]
        return torch.from_numpy(y)

    def combine(self, y_ret, inv, tok_off, L):
        y = torch.zeros((L, y_ret.shape[1] if y_ret.ndim == 2 else 0), dtype=torch.float64)
        for s in range(inv.shape[0]):
            for l in range(L):
                if inv[s, l] >= 0:
                    y[l] += y_ret[tok_off[s] + inv[s, l]]
        return y

    def mlp_hidden(self, x):
        return None

    def mlp_out(self, x, H, y_routed):
        if self.wgu is None:
            return y_routed
        return y_routed + torch.from_numpy(oracle.shared_mlp(x.numpy(), self.wgu.numpy(), self.wdn.numpy(), nthreads=1))
