import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2503_10325_b200 as cv
import synth
import oracle

def run(B, k, N, V, dtype, T=1.0, wm=0, sm=0, draft_len=None, seed=0, kind='probs', cs=0):
    inp = synth.linear_inputs(B, k, N, V, dtype=dtype, seed=seed, device='cuda', draft_len=draft_len, draft_kind=kind)
    ver = cv.Verifier(V, max_batch=B, k=k, N=N, target_dtype=dtype, draft_dtype=dtype, seed=7, debug=True,
                      draft_kind=(cv.DRAFT_LOGITS if kind=='logits' else cv.DRAFT_PROBS), cluster_size=cs)
    a, o, s = ver.verify(inp['target'], inp['draft'], inp['draft_tokens'], inp['request_ids'], temperature=T,
                         draft_len=inp['draft_len'], weight_mode=wm, select_mode=sm)
    torch.cuda.synchronize()
    r = oracle.verify_batch(inp['target'], inp['draft'], inp['draft_tokens'], inp['request_ids'], temperature=T,
                            seed=7, draft_len=inp['draft_len'], weight_mode=wm, select_mode=sm, vocab=V,
                            draft_kind=(1 if kind=='logits' else 0))
    a, o, s = a.cpu().numpy(), o.cpu().numpy(), s.cpu().numpy()
    mism = np.nonzero((a != r['accept_len']) | (o != r['out_tokens']).any(1))[0]
    tie = r['tie_margin'] < 1e-6
    bad = [b for b in mism if not tie[b]]
    dbg = {n: t.cpu().numpy() for n, t in ver.debug.items()}
    relp = np.nanmax(np.abs(dbg['p_x'][:B] - r['p_x']) / np.maximum(np.abs(r['p_x']), 1e-30)) if T > 0 else 0
    relS = np.nanmax(np.abs(dbg['row_sumexp'][:B] - r['S']) / r['S']) if T > 0 else 0
    print(f"B={B} k={k} N={N} V={V} {dtype} T={T} wm={wm} sm={sm} kind={kind}: mismatches={len(mism)} unflagged={len(bad)} "
          f"ties={tie.sum()} status_gpu={np.unique(s)} status_orc={np.unique(r['status'])} relp={relp:.2e} relS={relS:.2e} "
          f"meanL={a.mean():.2f}")
    if bad:
        b = bad[0]; print('  gpu', a[b], o[b], s[b], ' oracle', r['accept_len'][b], r['out_tokens'][b], r['status'][b], r['tie_margin'][b])
    return len(bad)

fails = 0
fails += run(1, 4, 2, 32000, torch.float32)
fails += run(64, 8, 3, 32000, torch.bfloat16)
fails += run(16, 8, 4, 128256, torch.bfloat16)
fails += run(8, 4, 3, 1003, torch.float32, draft_len='random')
fails += run(8, 4, 3, 1003, torch.bfloat16, T=0.0)
fails += run(8, 4, 3, 5000, torch.bfloat16, wm=1)
fails += run(8, 4, 3, 5000, torch.bfloat16, wm=2)
fails += run(8, 4, 3, 5000, torch.bfloat16, wm=3)
fails += run(8, 4, 3, 5000, torch.bfloat16, sm=1)
fails += run(8, 4, 2, 5000, torch.float32, kind='logits', T=0.7)
fails += run(8, 4, 3, 5000, torch.bfloat16, cs=2)
print("FAILS", fails)
