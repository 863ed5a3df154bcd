"""O0 -- literal brute force over the batch history (TEST INFRASTRUCTURE ONLY).

Used only to pin the O1 map oracle on tiny inputs. It keeps every batch and
answers each query by scanning history from the newest batch backwards,
applying the batch semantics rules of PAPER.md §3.1 (lines 260-279) directly:

  * rule 3: the most recent batch that mentions k decides;
  * rules 5/6: if that batch deletes k anywhere, k is absent
    (PAPER.md:273-278);
  * rule 4 with reading R4: otherwise the value of the FIRST insert of k in
    that batch.

No map, no sorting, no status bits: it shares no logic with O1 or S1.
count/range apply the lookup to every key in [k1, k2] that ever occurred
(the definitions at PAPER.md:105-109). Keys > 2^31-2 are dropped, as in O1
(reading R5).
"""

MAX_KEY = 0x7FFFFFFE


class BruteDict:
    def __init__(self):
        self.history = []   # list of batches: list of (key, val, is_delete)

    def apply_batch(self, keys, vals, is_delete):
        self.history.append([(int(k), int(v), bool(d))
                             for k, v, d in zip(keys, vals, is_delete)
                             if int(k) <= MAX_KEY])

    def lookup(self, k):
        k = int(k)
        for batch in reversed(self.history):
            mentioned = [(v, d) for (kk, v, d) in batch if kk == k]
            if not mentioned:
                continue
            if any(d for (_, d) in mentioned):
                return None
            return mentioned[0][0]
        return None

    def _keys_ever(self):
        seen = []
        for batch in self.history:
            for (k, _, _) in batch:
                if k not in seen:
                    seen.append(k)
        return seen

    def range(self, k1, k2):
        k1, k2 = int(k1), int(k2)
        out = []
        for k in self._keys_ever():
            if k1 <= k <= k2:
                v = self.lookup(k)
                if v is not None:
                    out.append((k, v))
        # ascending key order by selection (no library sort)
        res = []
        while out:
            m = 0
            for i in range(1, len(out)):
                if out[i][0] < out[m][0]:
                    m = i
            res.append(out.pop(m))
        return res

    def count(self, k1, k2):
        return len(self.range(k1, k2))

    def successor(self, k):
        """Smallest key >= k whose lookup is not ⊥ (R23), by scanning every
        key that ever occurred; (key, val) or None."""
        k = int(k)
        best = None
        for kk in self._keys_ever():
            if kk >= k and (best is None or kk < best[0]):
                v = self.lookup(kk)
                if v is not None:
                    best = (kk, v)
        return best

    def predecessor(self, k):
        """Largest key <= k whose lookup is not ⊥ (R23); (key, val) or None."""
        k = int(k)
        best = None
        for kk in self._keys_ever():
            if kk <= k and (best is None or kk > best[0]):
                v = self.lookup(kk)
                if v is not None:
                    best = (kk, v)
        return best
